mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/g35_pytest.log 2>&1
tail -3 gpurun_out/g35_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
