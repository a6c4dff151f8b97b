mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -k "persist or graphs or config1 or tiny2d or hybrid_2d or config2 or tiny5 or config5" > gpurun_out/g17_pytest.log 2>&1
tail -3 gpurun_out/g17_pytest.log | cut -c1-400
Q="--steps 2 --warmup 2 --no-e2e --no-cpu"
timeout 600 python bench.py --time-steps 4000 $Q > gpurun_out/g17_c2.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/g17_c2.json'));print('c2', round(d['value']), round(d['roofline']['frac'],3), d['ms_per_step'])"
timeout 600 python bench.py --config 5 --time-steps 2000 $Q > gpurun_out/g17_c5.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/g17_c5.json'));print('c5', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'])"
L="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $L --launch-skip 300 -c 200 --log-file gpurun_out/g17_launches_c5.csv python bench.py --config 5 --steps 2 --warmup 3 --time-steps 100 --no-e2e --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/g17_launches_c5.csv > gpurun_out/g17_launches_c5.txt; cat gpurun_out/g17_launches_c5.txt
