python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_configs.py -k "persistent_2d or tiny5 or tiny4_batched or tiny2d" 2>&1 | tail -15 > gpurun_out/g6_tests.log
timeout 300 python tools/golden_check.py 2 32 --tag tb_hilo >> gpurun_out/g6_prec.txt 2>&1
FDTD_P2K=0 timeout 300 python tools/golden_check.py 2 32 --tag old_hilo >> gpurun_out/g6_prec.txt 2>&1
FDTD_P2K=4 python tools/p2prof.py 2000 > gpurun_out/g6_plain.log 2>&1 && \
FDTD_P2K=4 ncu --set full --clock-control none --import-source on -k regex:persist2d -c 1 -o gpurun_out/g6_tb python tools/p2prof.py 2000 > gpurun_out/g6_ncu.log 2>&1
