mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
Q="--steps 3 --warmup 2 --no-e2e --no-cpu"
for i in 1 2 3; do for r in 0 1; do
  FDTD_P2_ROWSFIRST=$r timeout 600 python bench.py --time-steps 4000 $Q > gpurun_out/g27.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g27.json'));print('c2 rowsfirst=$r', round(d['value']))"
done; done
FDTD_P2_ROWSFIRST=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "persist" > gpurun_out/g27_pytest.log 2>&1; tail -1 gpurun_out/g27_pytest.log
