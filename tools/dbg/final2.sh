# second round-end pass after the late changes (local-slot rows, 16-row tiles, device set_state)
mkdir -p gpurun_out/final2
O=gpurun_out/final2
python -c "from paper_1406_7042_b200 import build as b; b.build()"
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > $O/pytest_gpu.log 2>&1
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -3 $O/smoke.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 300 $O/bench_c2.json
timeout 900 python bench.py --impl reference > $O/bench_ref_c2.json 2>&1
timeout 900 python bench.py --config 3 --precision 32 > $O/bench_c3_32.json 2>/dev/null
timeout 900 python bench.py --config 3 --precision 64 > $O/bench_c3_64.json 2>/dev/null
timeout 1200 python bench.py --config 5 > $O/bench_c5.json 2>/dev/null
timeout 1500 python bench.py --config 4 --steps 3 > $O/bench_c4.json 2>/dev/null
for f in $O/bench_c*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']
print('$f', round(d['value']), d['dtype'], round(r['frac'],3), round(r['achieved']), 'e2e', round(d['e2e']['value']), 'cpu', d['cpu_baseline'] and d['cpu_baseline']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
L="--metrics gpu__time_duration.sum --clock-control none --csv"
for c in "5 32" "4 32"; do set -- $c
  timeout 900 ncu $L --launch-skip 300 -c 200 --log-file $O/launches_c$1_$2.csv python bench.py --config $1 --precision $2 --steps 2 --warmup 3 --time-steps 100 --no-e2e --no-cpu > /dev/null 2>&1
done
timeout 900 ncu $L -c 40 --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --time-steps 2000 --no-e2e --no-cpu > /dev/null 2>&1
for f in $O/launches_*.csv; do python tools/ncu_summary.py $f > ${f%.csv}.txt 2>&1; rm -f $f; head -9 ${f%.csv}.txt; done
cap() { TAG=$1; KR=$2; SKIP=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" --launch-skip $SKIP -c 1 -o $O/$TAG python bench.py "$@" > /dev/null 2>&1
  python tools/ncu_report.py $O/$TAG.ncu-rep > $O/ncu_$TAG.txt 2>&1; rm -f $O/$TAG.ncu-rep; }
cap c2_persist persist2d 3 --steps 1 --warmup 3 --time-steps 2000 --no-e2e --no-cpu
cap c5 stencil 20 --config 5 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
cap c4 stencil 20 --config 4 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
for f in $O/ncu_*.txt; do echo "== $f"; grep "Duration\|DRAM Through\|dram bytes\|Issue Slots" $f | head -4; done
