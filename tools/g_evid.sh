#!/bin/bash
# evidence run without the shape sweep: tests, bench, ncu launch list + full captures
T=${1:-r1}
D=gpurun_out/prof_$T; mkdir -p $D
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/gpu.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $D/pytest.txt; cat $D/pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -2 $D/smoke.txt
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; tail -c 600 $D/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 1 > $D/ncu_bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_ft python tools/prof_run.py bf16 8192 2 > $D/p1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:encode_b -s 1 -c 1 -o $D/encode_b python tools/prof_run.py bf16 8192 2 > $D/p4.log 2>&1
echo done
