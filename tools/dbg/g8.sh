# round measurement pass: GPU tests, bench lines (configs 2-5), ncu launch lists, full captures of the top kernels
mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/g8_pytest.log 2>&1
tail -3 gpurun_out/g8_pytest.log
timeout 900 python bench.py > gpurun_out/g8_bench_c2.json 2> gpurun_out/g8_bench_c2.err; tail -c 400 gpurun_out/g8_bench_c2.json
timeout 900 python bench.py --config 3 --precision 32 > gpurun_out/g8_bench_c3_32.json 2>/dev/null; tail -c 300 gpurun_out/g8_bench_c3_32.json
timeout 900 python bench.py --config 3 --precision 64 > gpurun_out/g8_bench_c3_64.json 2>/dev/null; tail -c 300 gpurun_out/g8_bench_c3_64.json
timeout 1200 python bench.py --config 5 > gpurun_out/g8_bench_c5.json 2>/dev/null; tail -c 300 gpurun_out/g8_bench_c5.json
timeout 1500 python bench.py --config 4 --steps 3 > gpurun_out/g8_bench_c4.json 2>/dev/null; tail -c 300 gpurun_out/g8_bench_c4.json
L="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $L -c 40 --log-file gpurun_out/g8_launches_c2.csv python bench.py --steps 2 --warmup 3 --time-steps 2000 --no-e2e --no-cpu > /dev/null 2>&1
for c in "3 32" "3 64" "5 32" "4 32"; do set -- $c
  timeout 900 ncu $L --launch-skip 300 -c 200 --log-file gpurun_out/g8_launches_c$1_$2.csv python bench.py --config $1 --precision $2 --steps 2 --warmup 3 --time-steps 100 --no-e2e --no-cpu > /dev/null 2>&1
done
for f in gpurun_out/g8_launches_*.csv; do python tools/ncu_summary.py $f > ${f%.csv}.txt 2>&1; head -8 ${f%.csv}.txt; done
bash tools/dbg/ncu_cap.sh g8full_c2 persist2d 3 -- --steps 1 --warmup 3 --time-steps 2000 --no-e2e --no-cpu
bash tools/dbg/ncu_cap.sh g8full_c3_32 stencil 20 -- --config 3 --precision 32 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
bash tools/dbg/ncu_cap.sh g8full_c3_64 stencil 20 -- --config 3 --precision 64 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
bash tools/dbg/ncu_cap.sh g8full_c5 stencil 20 -- --config 5 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
bash tools/dbg/ncu_cap.sh g8full_c4 stencil 20 -- --config 4 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
bash tools/dbg/ncu_cap.sh g8full_c4_gemm gemm_ 10 -- --config 4 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
bash tools/dbg/ncu_cap.sh g8full_c5_red reduced_gemm 10 -- --config 5 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu
for f in gpurun_out/g8full_*.txt; do echo "== $f"; grep -v "^==" $f | head -22; done
