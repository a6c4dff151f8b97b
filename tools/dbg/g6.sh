mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
Q="--steps 3 --warmup 2 --no-e2e --no-cpu"
for c in "3 32" "4 32" "5 32" "3 64"; do set -- $c
 for g in 0 1000000; do
  if [ $g = 0 ]; then unset FDTD_TILE_GRID; else export FDTD_TILE_GRID=$g; fi
  FDTD_VERBOSE=1 timeout 600 python bench.py --config $1 --precision $2 --time-steps 200 $Q > gpurun_out/g6_c$1_$2_$g.json 2> gpurun_out/g6_c$1_$2_$g.err
  grep "tile stencil" gpurun_out/g6_c$1_$2_$g.err | head -1
  python -c "import json;d=json.load(open('gpurun_out/g6_c$1_$2_$g.json'));print('c$1 fp$2 grid $g', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'])"
 done
done
unset FDTD_TILE_GRID
for kc in 16 24 40; do
  FDTD_TILE_GRID=1000000 FDTD_TILE_KC=$kc timeout 600 python bench.py --config 3 --precision 32 --time-steps 200 $Q > gpurun_out/g6_kc$kc.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/g6_kc$kc.json'));print('c3 fp32 nonpersist kc $kc', round(d['value']), round(d['roofline']['frac'],3))"
done
