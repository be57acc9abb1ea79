#!/bin/bash
# full evidence run: tests, bench, sweep, ncu launch list + full captures
T=${1:-r1}
D=gpurun_out/prof_$T; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $D/pytest.txt; cat $D/pytest.txt
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; tail -c 600 $D/bench.json
timeout 1500 python tools/sweep.py --out $D/sweep.json > $D/sweep.log 2>&1; tail -1 $D/sweep.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 1 > $D/ncu_bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_ft python tools/prof_run.py bf16 8192 2 > $D/p1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_off python tools/prof_run.py bf16 8192 0 > $D/p2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:encode_a -s 1 -c 1 -o $D/encode_a python tools/prof_run.py bf16 8192 2 > $D/p3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:encode_b -s 1 -c 1 -o $D/encode_b python tools/prof_run.py bf16 8192 2 > $D/p4.log 2>&1
echo done
