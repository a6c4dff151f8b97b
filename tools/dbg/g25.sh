mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g25_pytest.log 2>&1
tail -3 gpurun_out/g25_pytest.log | cut -c1-400
Q="--steps 3 --warmup 2 --no-e2e --no-cpu"
for i in 1 2; do for pdl in 1 0; do
  if [ $pdl = 0 ]; then export FDTD_NO_PDL=1; else unset FDTD_NO_PDL; fi
  timeout 600 python bench.py --config 5 --time-steps 2000 $Q > gpurun_out/g25.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g25.json'));print('c5 pdl=$pdl', round(d['value']), round(d['roofline']['frac'],3))"
  timeout 600 python bench.py --config 3 --precision 32 --time-steps 300 $Q > gpurun_out/g25.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g25.json'));print('c3 pdl=$pdl', round(d['value']), round(d['roofline']['frac'],3))"
done; done
