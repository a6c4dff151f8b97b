mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 600 python -m pytest tests/test_gpu_configs.py -x -q -k "tensor_core" > gpurun_out/g14_pytest.log 2>&1
tail -3 gpurun_out/g14_pytest.log | cut -c1-400
timeout 900 ncu --metrics sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,gpu__time_duration.sum -k regex:tc_skinny --launch-skip 5 -c 3 python bench.py --config 4 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu > gpurun_out/g14_tcpipe.txt 2>&1
grep -A6 "Metric Name" gpurun_out/g14_tcpipe.txt | tail -12
Q="--steps 2 --warmup 2 --no-e2e --no-cpu"
timeout 900 python bench.py --config 4 --time-steps 200 $Q > gpurun_out/g14_c4.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/g14_c4.json'));print('c4', round(d['value']), round(d['roofline']['frac'],3), d['roofline']['phase_ms_per_step'])"
