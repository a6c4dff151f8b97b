mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -k "persist or graphs or config1 or tiny2d or hybrid_2d or config2" > gpurun_out/g21_pytest.log 2>&1
tail -2 gpurun_out/g21_pytest.log | cut -c1-400
Q="--steps 3 --warmup 2 --no-e2e --no-cpu"
for i in 1 2 3; do for r in 0 1; do
  if [ $r = 1 ]; then export FDTD_P2_ENDBAR=1; else unset FDTD_P2_ENDBAR; fi
  timeout 600 python bench.py --time-steps 4000 $Q > gpurun_out/g21_c2.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g21_c2.json'));print('c2 endbar=$r', round(d['value']))"
done; done
