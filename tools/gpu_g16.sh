python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/tb_race_probe.py 2 > gpurun_out/g16_tb.txt 2>&1
python tools/tb_race_probe.py 4 >> gpurun_out/g16_tb.txt 2>&1
( time timeout 1500 python bench.py > gpurun_out/g16_bench.json 2> gpurun_out/g16_bench.err ) 2> gpurun_out/g16_time.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g16_ref.json 2> gpurun_out/g16_ref.err
