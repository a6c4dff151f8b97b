python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -q tests/test_gpu_configs.py -k "tiny4" 2>&1 | tail -5 > gpurun_out/g11_tests.log
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('config4', round(d['value']), round(r['frac'],3), d['ms_per_step'], d['clocks'], r['phase_ms_per_step'], d.get('reduced_block'))" >> gpurun_out/g11_bench.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/g11_bench.txt
timeout 300 python bench.py --config 4 --time-steps 200 --steps 1 --warmup 3 --no-cpu --no-e2e --no-per-config > gpurun_out/g11_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 60 --csv --log-file gpurun_out/g11_launches.csv python bench.py --config 4 --time-steps 200 --steps 1 --warmup 3 --no-cpu --no-e2e --no-per-config > gpurun_out/g11_ncu.log 2>&1
