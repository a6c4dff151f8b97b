set -x
mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "tile_stencil or tma_stencil or config3 or tiny5 or tiny4 or batched" > gpurun_out/pytest_g2.log 2>&1
tail -5 gpurun_out/pytest_g2.log
Q="--steps 3 --warmup 3 --no-e2e --no-cpu"
for t in old "2,4" "2,6" "4,3"; do
  if [ "$t" = old ]; then export FDTD_STENCIL_OLD=1; else unset FDTD_STENCIL_OLD; export FDTD_TILE=$t; fi
  timeout 300 python bench.py --config 3 --precision 32 --time-steps 300 $Q > gpurun_out/g2_c3_32_$t.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g2_c3_32_$t.json'));print('c3 fp32 $t', d['value'], d['roofline']['frac'])"
done
unset FDTD_TILE
for t in old "2,3" "1,6"; do
  if [ "$t" = old ]; then export FDTD_STENCIL_OLD=1; else unset FDTD_STENCIL_OLD; export FDTD_TILE=$t; fi
  timeout 300 python bench.py --config 3 --precision 64 --time-steps 300 $Q > gpurun_out/g2_c3_64_$t.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g2_c3_64_$t.json'));print('c3 fp64 $t', d['value'], d['roofline']['frac'])"
done
unset FDTD_TILE
for t in old new; do
  if [ "$t" = old ]; then export FDTD_STENCIL_OLD=1; else unset FDTD_STENCIL_OLD; fi
  timeout 600 python bench.py --config 5 --time-steps 2000 $Q > gpurun_out/g2_c5_$t.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g2_c5_$t.json'));print('c5 $t', d['value'], d['roofline']['frac'], d['roofline']['phase_ms_per_step'])"
  timeout 900 python bench.py --config 4 --time-steps 300 $Q > gpurun_out/g2_c4_$t.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g2_c4_$t.json'));print('c4 $t', d['value'], d['roofline']['frac'], d['roofline']['phase_ms_per_step'])"
done
