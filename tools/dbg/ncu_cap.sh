# usage: bash tools/dbg/ncu_cap.sh TAG KERNEL_REGEX SKIP -- bench args...
# one `ncu --set full` capture, summarised on the box (the .ncu-rep is kept only if KEEP=1)
TAG=$1; KR=$2; SKIP=$3; shift 4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" --launch-skip $SKIP -c 1 -o gpurun_out/$TAG python bench.py "$@" > gpurun_out/$TAG.log 2>&1
python tools/ncu_report.py gpurun_out/$TAG.ncu-rep > gpurun_out/$TAG.txt 2>&1
[ -f tools/ncu_sass_top.py ] && python tools/ncu_sass_top.py gpurun_out/$TAG.ncu-rep > gpurun_out/${TAG}_sass.txt 2>&1
[ "$KEEP" = 1 ] || rm -f gpurun_out/$TAG.ncu-rep
