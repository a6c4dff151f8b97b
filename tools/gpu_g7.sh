python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest -q tests/test_gpu_configs.py tests/test_gpu_parity.py 2>&1 | tail -30 > gpurun_out/g7_tests.log
timeout 300 python tools/golden_check.py 2 32 --tag tb_fp64acc >> gpurun_out/g7_prec.txt 2>&1
for SL in 0 50 200; do for K in 4 2; do
  FDTD_P2SLEEP=$SL FDTD_P2K=$K timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('K=$K sleep=$SL', round(d['value']), round(r['frac'],3), d['ms_per_step'])" >> gpurun_out/g7_bench.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/g7_bench.txt
done; done
FDTD_P2K=0 timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('K=0', round(d['value']), round(r['frac'],3), d['ms_per_step'])" >> gpurun_out/g7_bench.txt 2>&1
timeout 300 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('config5', round(d['value']), round(r['frac'],3), r['phase_ms_per_step'])" >> gpurun_out/g7_bench.txt 2>&1
echo "K=4 tl" >> gpurun_out/g7_tl.txt; FDTD_P2K=4 timeout 120 python tools/p2tl.py >> gpurun_out/g7_tl.txt 2>&1
