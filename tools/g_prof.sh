#!/bin/bash
# bench + ncu evidence for profiles/ (round tag $1)
T=${1:-r1}
D=gpurun_out/prof_$T; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; tail -c 3000 $D/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 1 > $D/ncu_bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_ft python tools/prof_run.py bf16 8192 2 > $D/p1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_off python tools/prof_run.py bf16 8192 0 > $D/p2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:encode_a -s 1 -c 1 -o $D/encode_a python tools/prof_run.py bf16 8192 2 > $D/p3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:encode_b -s 1 -c 1 -o $D/encode_b python tools/prof_run.py bf16 8192 2 > $D/p4.log 2>&1
echo done
