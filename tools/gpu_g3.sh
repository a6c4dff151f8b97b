# call 3: temporal-blocking persist2d (bitwise tests, timing) + config-2 fp32 precision study vs the golden
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_configs.py -k "persistent_2d" 2>&1 | tail -15 > gpurun_out/g3_tb_tests.log
for K in 4 0 2 8; do
  FDTD_P2K=$K timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('K=$K', round(d['value']), round(r['frac'],3), d['ms_per_step'])" >> gpurun_out/g3_tb_bench.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/g3_tb_bench.txt
done
timeout 300 python tools/golden_check.py 2 64 --golden-prec 32 --tag fp64 >> gpurun_out/g3_prec.txt 2>&1
timeout 300 python tools/golden_check.py 2 32 --tag tb >> gpurun_out/g3_prec.txt 2>&1
FDTD_P2K=0 timeout 300 python tools/golden_check.py 2 32 --tag persist_old >> gpurun_out/g3_prec.txt 2>&1
FDTD_PERSIST=0 timeout 300 python tools/golden_check.py 2 32 --tag perstep_fused >> gpurun_out/g3_prec.txt 2>&1
FDTD_PERSIST=0 timeout 300 python tools/golden_check.py 2 32 --form leapfrog --tag perstep_leapfrog >> gpurun_out/g3_prec.txt 2>&1
