mkdir -p gpurun_out/r02
for C in 4 5; do
timeout 900 python bench.py --config $C --steps 1 --warmup 3 --no-cpu --no-e2e --no-per-config > gpurun_out/r02/plain_c$C.json 2> gpurun_out/r02/plain_c$C.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 600 --csv --log-file gpurun_out/r02/launches_c$C.csv python bench.py --config $C --steps 1 --warmup 3 --no-cpu --no-e2e --no-per-config > gpurun_out/r02/ncu_c$C.log 2>&1
done
