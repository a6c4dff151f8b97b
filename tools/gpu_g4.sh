python -c "import __graft_entry__ as g; g.build()" || exit 1
for K in 4 0; do echo "K=$K" >> gpurun_out/g4_tl.txt; FDTD_P2K=$K timeout 120 python tools/p2tl.py >> gpurun_out/g4_tl.txt 2>&1; done
