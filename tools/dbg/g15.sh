mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g15_pytest.log 2>&1
tail -3 gpurun_out/g15_pytest.log | cut -c1-400
Q="--steps 2 --warmup 2 --no-e2e --no-cpu"
timeout 900 python bench.py --config 4 --time-steps 200 $Q > gpurun_out/g15_c4.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/g15_c4.json'));print('c4', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'])"
L="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $L --launch-skip 300 -c 200 --log-file gpurun_out/g15_launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --time-steps 100 --no-e2e --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/g15_launches_c4.csv > gpurun_out/g15_launches_c4.txt; cat gpurun_out/g15_launches_c4.txt
