python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_configs.py -k "persistent_2d" 2>&1 | tail -15 > gpurun_out/g5_tb_tests.log
for K in 4 2 0; do
  FDTD_P2K=$K timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('K=$K', round(d['value']), round(r['frac'],3), d['ms_per_step'])" >> gpurun_out/g5_tb_bench.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/g5_tb_bench.txt
done
for K in 4; do echo "K=$K" >> gpurun_out/g5_tl.txt; FDTD_P2K=$K timeout 120 python tools/p2tl.py >> gpurun_out/g5_tl.txt 2>&1; done
