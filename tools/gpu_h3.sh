timeout 1500 python -m pytest -q tests/test_gpu_configs.py -k "tile_stencil or bitwise or tiny5 or tiny4 or config3_small or tiny2d" 2>&1 | tail -8 > gpurun_out/h3_tests.log
python tools/c5_probe.py "FDTD_NO_TILE_UNI=1" > gpurun_out/h3_c5.txt 2>&1
