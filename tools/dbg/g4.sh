mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "tile_stencil or tma_stencil or config3 or tiny5 or tiny4 or batched or config5" > gpurun_out/pytest_g4.log 2>&1
tail -3 gpurun_out/pytest_g4.log
Q="--steps 3 --warmup 3 --no-e2e --no-cpu"
for c in "3 32" "3 64" "4 32" "5 32"; do set -- $c
  timeout 600 python bench.py --config $1 --precision $2 --time-steps 300 $Q > gpurun_out/g4_c$1_$2.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g4_c$1_$2.json'));print('c$1 fp$2', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'])"
done
for c in "3 32" "4 32" "5 32"; do set -- $c
  bash tools/dbg/ncu_cap.sh g4n_c$1 stencil 20 -- --config $1 --precision $2 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
  head -30 gpurun_out/g4n_c$1.txt
done
