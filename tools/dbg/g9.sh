mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 1200 python -m pytest tests -m gpu -x -q -k "not config4_full" > gpurun_out/g9_pytest.log 2>&1
tail -3 gpurun_out/g9_pytest.log
Q="--steps 2 --warmup 2 --no-e2e --no-cpu"
timeout 600 python bench.py --time-steps 4000 $Q > gpurun_out/g9_c2.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/g9_c2.json'));print('c2', round(d['value']), round(d['roofline']['frac'],3), d['ms_per_step'])"
timeout 600 python bench.py --config 5 --time-steps 2000 $Q > gpurun_out/g9_c5.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/g9_c5.json'));print('c5', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'])"
FDTD_P2DBG=1 timeout 300 python tools/dbg/p2dbg.py > gpurun_out/p2dbg9.txt 2>&1
tail -27 gpurun_out/p2dbg9.txt
