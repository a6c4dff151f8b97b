mkdir -p gpurun_out/r02
CMD4="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu --no-e2e --no-per-config"
CMD5="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu --no-e2e --no-per-config"
CMDR="python bench.py --rom-only"
$CMD4 > gpurun_out/r02/p4.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stencil3d_tile -s 500 -c 1 -f -o gpurun_out/r02/ncu_c4_stencil $CMD4 > gpurun_out/r02/ncu_c4.log 2>&1
$CMD5 > gpurun_out/r02/p5.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stencil3d_tile -s 2000 -c 1 -f -o gpurun_out/r02/ncu_c5_stencil $CMD5 > gpurun_out/r02/ncu_c5f.log 2>&1
$CMDR > gpurun_out/r02/prom.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:rom_persist -s 14 -c 1 -f -o gpurun_out/r02/ncu_rom $CMDR > gpurun_out/r02/ncu_rom.log 2>&1
