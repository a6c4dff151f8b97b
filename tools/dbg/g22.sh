mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "tile_stencil" > gpurun_out/g22_pytest.log 2>&1
tail -3 gpurun_out/g22_pytest.log | cut -c1-400
Q="--steps 3 --warmup 2 --no-e2e --no-cpu"
for i in 1 2; do
for t in "2,6,8" "2,4,16"; do
  FDTD_TILE=$t timeout 600 python bench.py --config 3 --precision 32 --time-steps 300 $Q > gpurun_out/g22.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g22.json'));print('c3 fp32 $t', round(d['value']), round(d['roofline']['frac'],3))"
done
for t in "2,3,8" "1,4,16"; do
  FDTD_TILE=$t timeout 600 python bench.py --config 3 --precision 64 --time-steps 300 $Q > gpurun_out/g22.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g22.json'));print('c3 fp64 $t', round(d['value']), round(d['roofline']['frac'],3))"
done
for t in "1,6,8" "2,4,16"; do
  FDTD_TILE=$t timeout 600 python bench.py --config 5 --time-steps 2000 $Q > gpurun_out/g22.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g22.json'));print('c5 $t', round(d['value']), round(d['roofline']['frac'],3))"
done
done
