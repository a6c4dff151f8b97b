python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest -q tests/test_gpu_races.py 2>&1 | tail -15 > gpurun_out/g13_races.log
for T in "2,4,16" "1,6" "2,4" "4,3"; do
  FDTD_TILE=$T timeout 300 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config --time-steps 10000 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('tile=$T', round(d['value']), round(r['frac'],3), r['phase_ms_per_step'])" >> gpurun_out/g13_c5.txt 2>&1 || tail -2 /tmp/b.err >> gpurun_out/g13_c5.txt
done
