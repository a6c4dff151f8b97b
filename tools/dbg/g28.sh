mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -k "persist or graphs or config1 or tiny2d or hybrid_2d or config2" > gpurun_out/g28_pytest.log 2>&1
tail -2 gpurun_out/g28_pytest.log | cut -c1-300
Q="--steps 3 --warmup 2 --no-e2e --no-cpu"
for i in 1 2 3; do for r in 1 0; do
  FDTD_P2_EARLY=$r timeout 600 python bench.py --time-steps 4000 $Q > gpurun_out/g28.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g28.json'));print('c2 early=$r', round(d['value']))"
done; done
FDTD_P2DBG=1 timeout 300 python tools/dbg/p2dbg.py > gpurun_out/p2dbg28.txt 2>&1
grep -A4 "slot 1\|slot 2" gpurun_out/p2dbg28.txt | head -12
