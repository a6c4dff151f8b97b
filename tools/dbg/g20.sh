mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "local_slot or tile_stencil or tiny5 or tiny4 or config5 or config4_full" > gpurun_out/g20_pytest.log 2>&1
tail -3 gpurun_out/g20_pytest.log | cut -c1-400
Q="--steps 2 --warmup 2 --no-e2e --no-cpu"
for l in 1 0; do
  if [ $l = 0 ]; then export FDTD_NO_LOCAL_ROWS=1; else unset FDTD_NO_LOCAL_ROWS; fi
  timeout 600 python bench.py --config 5 --time-steps 2000 $Q > gpurun_out/g20_c5_$l.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g20_c5_$l.json'));print('c5 local=$l', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'])"
  timeout 900 python bench.py --config 4 --time-steps 200 $Q > gpurun_out/g20_c4_$l.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g20_c4_$l.json'));print('c4 local=$l', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'])"
done
