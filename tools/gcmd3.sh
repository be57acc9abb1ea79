#!/bin/bash
D=gpurun_out/r30; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/k128_ft python tools/prof_shape.py bf16 16384 16384 128 2 > $D/a.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/k128_off python tools/prof_shape.py bf16 16384 16384 128 0 > $D/b.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/bf16_8k_ft python tools/prof_shape.py bf16 8192 8192 8192 2 > $D/c.log 2>&1
echo done
