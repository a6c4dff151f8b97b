mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
for k in 2 8; do FDTD_GEMM_KS=$k timeout 600 python -m pytest tests/test_gpu_configs.py -x -q -k "tiny5" > gpurun_out/g29_pytest_$k.log 2>&1; tail -1 gpurun_out/g29_pytest_$k.log; done
Q="--steps 3 --warmup 2 --no-e2e --no-cpu"
for i in 1 2; do for k in 4 2 8; do
  FDTD_GEMM_KS=$k timeout 600 python bench.py --config 5 --time-steps 2000 $Q > gpurun_out/g29.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g29.json'));print('c5 ks=$k', round(d['value']), d['roofline']['phase_ms_per_step']['reduced'])"
done; done
