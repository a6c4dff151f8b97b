mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -k "persist or graphs or config1 or tiny2d or hybrid_2d or config2" > gpurun_out/g34_pytest.log 2>&1
tail -1 gpurun_out/g34_pytest.log
Q="--steps 3 --warmup 2 --no-e2e --no-cpu"
for i in 1 2 3; do for r in 1 0; do
  FDTD_P2_EPUB=$r timeout 600 python bench.py --time-steps 4000 $Q > gpurun_out/g34.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g34.json'));print('c2 epub=$r', round(d['value']))"
done; done
