mkdir -p gpurun_out
python -c "from paper_1406_7042_b200 import build as b; b.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "persist or graphs" > gpurun_out/pytest_g7.log 2>&1
tail -2 gpurun_out/pytest_g7.log
Q="--steps 2 --warmup 2 --no-e2e --no-cpu"
timeout 600 python bench.py --config 2 --time-steps 4000 $Q > gpurun_out/g7_c2.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/g7_c2.json'));print('c2', round(d['value']), round(d['roofline']['frac'],3), d['ms_per_step'])"
FDTD_P2DBG=1 timeout 300 python tools/dbg/p2dbg.py > gpurun_out/p2dbg7.txt 2>&1
run() { # tag config prec tile kc
  env FDTD_TILE=$4 $( [ "$5" != 0 ] && echo FDTD_TILE_KC=$5 ) timeout 600 python bench.py --config $2 --precision $3 --time-steps 200 $Q > gpurun_out/g7_$1.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/g7_$1.json'));print('$1', round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['phase_ms_per_step']['stencil'],4))"
}
for kc in 0 8 12 32; do run c3f_2,6_kc$kc 3 32 2,6 $kc; done
for kc in 0 8 16 24; do run c3d_2,3_kc$kc 3 64 2,3 $kc; run c3d_1,6_kc$kc 3 64 1,6 $kc; done
for kc in 0 8 16 32 64; do run c4_kc$kc 4 32 4,3 $kc; done
for kc in 0 7 11 14 21; do run c5_1,6_kc$kc 5 32 1,6 $kc; run c5_2,6_kc$kc 5 32 2,6 $kc; done
