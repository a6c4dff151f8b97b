python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/l2_probe.py > gpurun_out/g12_l2.txt 2>&1
timeout 900 python -m pytest -q tests/test_gpu_configs.py -k "tiny4" 2>&1 | tail -3 > gpurun_out/g12_tests.log
for KS in 32 16 64; do
FDTD_KS=$KS timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-per-config > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('config4 ks=$KS', round(d['value']), round(r['frac'],3), d['ms_per_step'], d['clocks'], r['phase_ms_per_step'])" >> gpurun_out/g12_bench.txt 2>&1 || tail -3 /tmp/b.err >> gpurun_out/g12_bench.txt
done
python tools/sanitize_case.py all > gpurun_out/g12_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_case.py all > gpurun_out/g12_racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/g12_racecheck.log
