mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -k "tile_stencil or persist or graphs or config1 or tiny2d or hybrid_2d" > gpurun_out/pytest_g5.log 2>&1
tail -3 gpurun_out/pytest_g5.log
FDTD_P2DBG=1 timeout 300 python tools/dbg/p2dbg.py > gpurun_out/p2dbg5.txt 2>&1
tail -28 gpurun_out/p2dbg5.txt
Q="--steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 600 python bench.py --config 2 --time-steps 4000 $Q > gpurun_out/g5_c2.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/g5_c2.json'));print('c2', round(d['value']), round(d['roofline']['frac'],3), d['ms_per_step'])"
for c in "3 32" "3 64" "4 32" "5 32"; do set -- $c
  timeout 600 python bench.py --config $1 --precision $2 --time-steps 300 $Q > gpurun_out/g5_c$1_$2.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g5_c$1_$2.json'));print('c$1 fp$2', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'])"
done
bash tools/dbg/ncu_cap.sh g5n_c3 stencil 20 -- --config 3 --precision 32 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
head -24 gpurun_out/g5n_c3.txt
