python tools/c5_probe.py --one vactab > gpurun_out/h6_plain.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stencil3d_tile -s 300 -c 1 -f -o gpurun_out/h6_vactab python tools/c5_probe.py --one vactab > gpurun_out/h6_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stencil3d_tile -s 300 -c 1 -f -o gpurun_out/h6_vac python tools/c5_probe.py --one vac > gpurun_out/h6_ncu2.log 2>&1
