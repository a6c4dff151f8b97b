mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
Q="--steps 3 --warmup 2 --no-e2e --no-cpu"
for i in 1 2 3; do for r in 0 1; do
FDTD_P2_ROWSHIFT=$r timeout 600 python bench.py --time-steps 4000 $Q > gpurun_out/g19_c2.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/g19_c2.json'));print('c2 rowshift=$r', round(d['value']), d['clocks']['sm_mhz'])"
done; done
