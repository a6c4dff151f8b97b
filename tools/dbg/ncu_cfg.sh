# usage: bash tools/dbg/ncu_cfg.sh CONFIG PREC TAG  (launch list + one --set full per top kernel)
set -x
C=$1; P=$2; T=$3
CMD="python bench.py --config $C --precision $P --steps 3 --warmup 3 --time-steps 100 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/${T}_plain.json 2> gpurun_out/${T}_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 600 -c 100 --csv --log-file gpurun_out/${T}_launches.csv $CMD > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil --launch-skip 50 -c 1 -o gpurun_out/${T}_stencil $CMD > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"reduced|rowblock|colsum" --launch-skip 50 -c 1 -o gpurun_out/${T}_reduced $CMD > /dev/null 2>&1
ls gpurun_out/${T}*
