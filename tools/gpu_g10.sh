python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest -q tests/test_gpu_configs.py tests/test_gpu_parity.py 2>&1 | tail -30 > gpurun_out/g10_tests.log
for C in 4 5; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('config$C', round(d['value']), round(r['frac'],3), d['ms_per_step'], d['clocks'], r['phase_ms_per_step'], d.get('reduced_block'))" >> gpurun_out/g10_bench.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/g10_bench.txt
done
