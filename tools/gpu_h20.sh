python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest -q tests/test_gpu_lossy.py tests/test_gpu_golden.py -k "not (config5-fp32 or config4-fp32)" 2>&1 | tail -12 > gpurun_out/h20_tests.log
python - > gpurun_out/h20_bench.txt 2>&1 <<'PY'
import json, sys
sys.argv=['bench.py']
import bench
import argparse
class A: pass
a=A(); a.time_steps=0; a.graph_steps=32; a.profile_steps=500; a.e2e_steps=1; a.no_e2e=True; a.no_cpu=True; a.cpu_seconds=1
from paper_1406_7042_b200.dist import init
init()
for c,p in (("lossy256",32),(3,32),(5,32),(4,32)):
    try:
        r=bench.measure(c,p,3,3,a)
        print(c,p,round(r['value']), round(r['roofline']['frac'],3), r['ms_per_step'], r['roofline']['phase_ms_per_step'], r['clocks'])
    except Exception as ex:
        import traceback; traceback.print_exc()
PY
