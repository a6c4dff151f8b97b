timeout 1800 python -m pytest -q tests/test_gpu_configs.py -k "tile_stencil or prepass or tiny5 or tiny4 or config5 or config4" 2>&1 | tail -5 > gpurun_out/h16_tests.log
C5_KINDS=full python tools/c5_probe.py "FDTD_NO_ROWPACK=1" > gpurun_out/h16_c5.txt 2>&1
for E in "" "FDTD_NO_ROWPACK=1"; do
  env $E timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('config4 $E', round(d['value']), round(r['frac'],3), d['ms_per_step'], d['clocks'], r['phase_ms_per_step'])" >> gpurun_out/h16_bench.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/h16_bench.txt
done
