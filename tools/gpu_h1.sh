python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest -q -x tests/test_gpu_configs.py -k "tile_stencil or config5 or tiny5 or tiny4_batched or local_slot or config4" 2>&1 | tail -15 > gpurun_out/h1_tests.log
python tools/c5_probe.py "FDTD_NO_TILE_UNI=1" > gpurun_out/h1_c5.txt 2>&1
for C in 4 5; do
  for E in "" "FDTD_NO_TILE_UNI=1"; do
  env $E timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('config$C $E', round(d['value']), round(r['frac'],3), d['ms_per_step'], d['clocks'], r['phase_ms_per_step'])" >> gpurun_out/h1_bench.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/h1_bench.txt
  done
done
