# last default bench lines after the late persistent-kernel / fused-GEMM changes
mkdir -p gpurun_out/final3
O=gpurun_out/final3
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_c2.json 2>/dev/null
timeout 1200 python bench.py --config 5 > $O/bench_c5.json 2>/dev/null
for f in $O/bench_c2.json $O/bench_c5.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']
print('$f', round(d['value']), round(r['frac'],3), round(r['achieved']), 'e2e', round(d['e2e']['value']), 'cpu', d['cpu_baseline']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['ms_per_step'])"; done
L="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $L -c 40 --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --time-steps 2000 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu $L --launch-skip 300 -c 200 --log-file $O/launches_c5_32.csv python bench.py --config 5 --steps 2 --warmup 3 --time-steps 100 --no-e2e --no-cpu > /dev/null 2>&1
for f in $O/launches_*.csv; do python tools/ncu_summary.py $f > ${f%.csv}.txt 2>&1; rm -f $f; head -6 ${f%.csv}.txt; done
timeout 900 ncu --set full --clock-control none -k regex:persist2d --launch-skip 3 -c 1 -o $O/c2 python bench.py --steps 1 --warmup 3 --time-steps 2000 --no-e2e --no-cpu > /dev/null 2>&1
python tools/ncu_report.py $O/c2.ncu-rep > $O/ncu_c2_persist.txt 2>&1; rm -f $O/c2.ncu-rep; head -20 $O/ncu_c2_persist.txt
