mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config5 or tiny5 or local_slot or tile_stencil or set_state" > gpurun_out/g24_pytest.log 2>&1
tail -3 gpurun_out/g24_pytest.log | cut -c1-400
for c in "3 32" "5 32"; do set -- $c
timeout 900 python bench.py --config $1 --precision $2 --steps 3 > gpurun_out/g24_c$1.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/g24_c$1.json'));r=d['roofline'];print('c$1', round(d['value']), round(r['frac'],3), 'e2e', round(d['e2e']['value']), d['e2e']['ms_per_step'], d['ms_per_step'])"
done
