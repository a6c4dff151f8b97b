timeout 1800 python -m pytest -q tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_races.py 2>&1 | tail -8 > gpurun_out/h11_tests.log
C5_KINDS=vac,vactab,full python tools/c5_probe.py > gpurun_out/h11_c5.txt 2>&1
for C in 5 4 3; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('config$C', round(d['value']), round(r['frac'],3), d['ms_per_step'], d['clocks'], r['phase_ms_per_step'])" >> gpurun_out/h11_bench.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/h11_bench.txt
done
