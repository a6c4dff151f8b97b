#!/bin/bash
# Round-end pass on one B200 (gpurun): build, the whole GPU test suite, smoke(),
# the default bench (headline config 4 + per_config lines), the reference arm,
# the ncu launch lists of configs 4 / 5 and the slab-decomposition overhead.
# Everything lands in gpurun_out/final/ (copied to profiles/r02/ afterwards).
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" || exit 1
( time timeout 3000 python -m pytest -q tests -m gpu 2>&1 | tail -25 ) > $O/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
( time timeout 1800 python bench.py > $O/bench_default.json 2> $O/bench_default.err ) 2> $O/bench_time.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for C in 4 5; do
  CMD="python bench.py --config $C --steps 1 --warmup 3 --no-cpu --no-e2e --no-per-config"
  $CMD > $O/plain_c$C.json 2> $O/plain_c$C.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 1000 -c 600 --csv --log-file $O/launches_c$C.csv $CMD > $O/ncu_c$C.log 2>&1
done
python tools/slab_overhead.py > $O/slab_overhead.txt 2>&1
