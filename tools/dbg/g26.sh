mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "tile_stencil" > gpurun_out/g26_pytest.log 2>&1
tail -3 gpurun_out/g26_pytest.log | cut -c1-400
Q="--steps 2 --warmup 2 --no-e2e --no-cpu"
for i in 1 2; do for t in "4,3,8" "4,3,16"; do
  FDTD_TILE=$t timeout 900 python bench.py --config 4 --time-steps 200 $Q > gpurun_out/g26.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g26.json'));print('c4 $t', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
