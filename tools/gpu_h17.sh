python -c "import __graft_entry__ as g; g.build()" || exit 1
( time timeout 2400 python -m pytest -q tests -m gpu -k "not (config5-fp32 or config4-fp32)" 2>&1 | tail -15 ) > gpurun_out/h17_tests.log 2>&1
( time timeout 1800 python bench.py > gpurun_out/h17_bench.json 2> gpurun_out/h17_bench.err ) 2> gpurun_out/h17_time.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h17_smoke.log 2>&1
