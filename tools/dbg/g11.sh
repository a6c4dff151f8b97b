mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
Q="--steps 2 --warmup 2 --no-e2e --no-cpu"
for t in on off; do
  if [ $t = off ]; then export FDTD_NO_TC=1; else unset FDTD_NO_TC; fi
  timeout 900 python bench.py --config 4 --time-steps 200 $Q > gpurun_out/g11_c4_$t.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g11_c4_$t.json'));print('c4 tc=$t', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'], d['roofline']['paths'])"
done
unset FDTD_NO_TC
L="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $L --launch-skip 300 -c 200 --log-file gpurun_out/g11_launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --time-steps 100 --no-e2e --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/g11_launches_c4.csv > gpurun_out/g11_launches_c4.txt; cat gpurun_out/g11_launches_c4.txt
bash tools/dbg/ncu_cap.sh g11full_tc tc_skinny 5 -- --config 4 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
cat gpurun_out/g11full_tc.txt
timeout 900 ncu --metrics sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,gpu__time_duration.sum -k regex:tc_skinny --launch-skip 5 -c 1 python bench.py --config 4 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu > gpurun_out/g11_tcpipe.txt 2>&1
grep -A12 "tc_skinny" gpurun_out/g11_tcpipe.txt | tail -12
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config4_full" > gpurun_out/g11_pytest.log 2>&1; tail -2 gpurun_out/g11_pytest.log
