mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config5 or tiny5" > gpurun_out/g30_pytest.log 2>&1; tail -1 gpurun_out/g30_pytest.log
FDTD_VERBOSE=1 timeout 600 python bench.py --config 5 --time-steps 2000 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/g30.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/g30.json'));print('c5', round(d['value']), d['roofline']['phase_ms_per_step']['reduced'])"
