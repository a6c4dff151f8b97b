set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -20 > gpurun_out/g1_tests.log
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/g1_b4.json 2> gpurun_out/g1_b4.err
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu > gpurun_out/g1_b5.json 2> gpurun_out/g1_b5.err
tail -3 gpurun_out/g1_tests.log
