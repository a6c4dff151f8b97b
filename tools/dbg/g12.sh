mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -k "tensor_core or persist or graphs or config1 or tiny2d or hybrid_2d or config2" > gpurun_out/g12_pytest.log 2>&1
tail -15 gpurun_out/g12_pytest.log | cut -c1-400
Q="--steps 2 --warmup 2 --no-e2e --no-cpu"
for r in reg noreg; do
  if [ $r = noreg ]; then export FDTD_P2_NOREG=1; else unset FDTD_P2_NOREG; fi
  timeout 600 python bench.py --time-steps 4000 $Q > gpurun_out/g12_c2_$r.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g12_c2_$r.json'));print('c2 $r', round(d['value']), round(d['roofline']['frac'],3), d['ms_per_step'])"
done
unset FDTD_P2_NOREG
FDTD_P2DBG=1 timeout 300 python tools/dbg/p2dbg.py > gpurun_out/p2dbg12.txt 2>&1
tail -27 gpurun_out/p2dbg12.txt
timeout 900 python bench.py --config 4 --time-steps 200 $Q > gpurun_out/g12_c4.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/g12_c4.json'));print('c4', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'])"
bash tools/dbg/ncu_cap.sh g12full_tc tc_skinny 5 -- --config 4 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
head -22 gpurun_out/g12full_tc.txt
