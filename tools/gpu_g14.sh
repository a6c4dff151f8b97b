python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest -q tests/test_gpu_races.py 2>&1 | tail -5 > gpurun_out/g14_races.log
timeout 1200 python -m pytest -q tests/test_gpu_configs.py -k "persistent" 2>&1 | tail -5 >> gpurun_out/g14_races.log
