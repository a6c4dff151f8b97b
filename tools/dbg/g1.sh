set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from paper_1406_7042_b200 import build as b; b.build()"
( time timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 ) > gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
for c in 2 5 4; do ( time timeout 900 python bench.py --config $c ) > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; tail -c 3000 gpurun_out/bench_c$c.json; done
( time timeout 600 python bench.py --config 3 --precision 32 ) > gpurun_out/bench_c3_32.json 2> gpurun_out/bench_c3_32.err
tail -c 3000 gpurun_out/bench_c3_32.json
