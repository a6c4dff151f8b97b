mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > gpurun_out/g32_c2.json 2>/dev/null
timeout 900 python bench.py --config 3 > gpurun_out/g32_c3.json 2>/dev/null
for f in gpurun_out/g32_c2.json gpurun_out/g32_c3.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), d['e2e']['ms_per_step'], d['ms_per_step'], d['gpu_launches'])"; done
