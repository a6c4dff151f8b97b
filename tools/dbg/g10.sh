mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 300 python -m pytest tests/test_gpu_configs.py -x -q -k "tensor_core" > gpurun_out/g10_pytest.log 2>&1
tail -30 gpurun_out/g10_pytest.log | cut -c1-300
FDTD_P2DBG=1 timeout 300 python tools/dbg/p2dbg.py > gpurun_out/p2dbg10.txt 2>&1
tail -27 gpurun_out/p2dbg10.txt
