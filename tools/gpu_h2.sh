timeout 1200 python -m pytest -q tests/test_gpu_configs.py -k "tile_stencil" 2>&1 | tail -8 > gpurun_out/h2_a.log
FDTD_NO_TILE_UNI=1 timeout 1200 python -m pytest -q tests/test_gpu_configs.py -k "tile_stencil" 2>&1 | tail -8 > gpurun_out/h2_b.log
