mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config5 or tiny5 or local_slot" > gpurun_out/g23_pytest.log 2>&1
tail -3 gpurun_out/g23_pytest.log | cut -c1-400
timeout 1200 python bench.py --config 5 > gpurun_out/g23_c5.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/g23_c5.json'));r=d['roofline'];print('c5', round(d['value']), round(r['frac'],3), round(d['e2e']['value']), r['phase_ms_per_step'], r.get('reduced_fused'), d['clocks'])"
L="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $L --launch-skip 300 -c 200 --log-file gpurun_out/g23_launches_c5.csv python bench.py --config 5 --steps 2 --warmup 3 --time-steps 100 --no-e2e --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/g23_launches_c5.csv > gpurun_out/g23_launches_c5.txt; rm -f gpurun_out/g23_launches_c5.csv; cat gpurun_out/g23_launches_c5.txt
