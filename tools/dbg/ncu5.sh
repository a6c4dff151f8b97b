set -x
CMD="python bench.py --config 5 --steps 3 --warmup 3 --time-steps 100 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/c5_plain.json 2> gpurun_out/c5_plain.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 600 -c 60 --csv --log-file gpurun_out/c5_launches.csv $CMD > gpurun_out/c5_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduced_gemm --launch-skip 50 -c 1 -o gpurun_out/c5_gemm $CMD > gpurun_out/c5_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil3d --launch-skip 50 -c 1 -o gpurun_out/c5_stencil $CMD > gpurun_out/c5_ncu3.log 2>&1
