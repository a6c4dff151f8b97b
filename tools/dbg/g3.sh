mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "tile_stencil" > gpurun_out/pytest_g3.log 2>&1
tail -3 gpurun_out/pytest_g3.log
FDTD_P2DBG=1 timeout 300 python tools/dbg/p2dbg.py > gpurun_out/p2dbg.txt 2>&1
tail -30 gpurun_out/p2dbg.txt
cap() { # tag config prec env
  env $4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil --launch-skip 20 -c 1 -o gpurun_out/$1 python bench.py --config $2 --precision $3 --steps 1 --warmup 1 --time-steps 40 --no-e2e --no-cpu > gpurun_out/$1.log 2>&1
}
cap c4_old 4 32 FDTD_STENCIL_OLD=1
cap c4_new 4 32 FDTD_X=1
cap c5_old 5 32 FDTD_STENCIL_OLD=1
cap c5_new 5 32 FDTD_X=1
cap c3_new 3 32 FDTD_TILE=2,6
ls gpurun_out
