# round-2 call 2: new parity tests (goldens present so far, random-state
# full-size runs, persistent bitwise) + config-5 z-chunk / tile sweep
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest -x -q -s tests/test_gpu_golden.py -k "config2" 2>&1 | tail -8 > gpurun_out/g2_golden.log
timeout 900 python -m pytest -x -q -s tests/test_gpu_configs.py -k "random_state or persistent_2d" 2>&1 | tail -12 > gpurun_out/g2_rand.log
for tile in "2,4,16" "2,6"; do for kc in 0 11 14 21 41; do
  if [ $kc = 0 ]; then unset FDTD_TILE_KC; else export FDTD_TILE_KC=$kc; fi
  FDTD_TILE=$tile timeout 300 python bench.py --config 5 --steps 3 --warmup 3 --time-steps 10000 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('$tile kc=$kc', round(d['value']), round(r['frac'],3), r['phase_ms_per_step'])" >> gpurun_out/g2_sweep.txt 2>&1
done; done
unset FDTD_TILE_KC
