python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest -q tests/test_gpu_races.py 2>&1 | tail -5 > gpurun_out/g15_tests.log
timeout 1200 python -m pytest -q tests/test_gpu_configs.py tests/test_gpu_parity.py 2>&1 | tail -5 >> gpurun_out/g15_tests.log
timeout 300 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('config5', round(d['value']), round(r['frac'],3), r['phase_ms_per_step'])" >> gpurun_out/g15_bench.txt 2>&1 || tail -2 /tmp/b.err >> gpurun_out/g15_bench.txt
FDTD_P2K=2 timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('config2 K2', round(d['value']), round(r['frac'],3))" >> gpurun_out/g15_bench.txt 2>&1
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('config2', round(d['value']), round(r['frac'],3))" >> gpurun_out/g15_bench.txt 2>&1
