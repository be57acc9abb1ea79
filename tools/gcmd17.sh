#!/bin/bash
export PYTHONUNBUFFERED=1
D=gpurun_out/r38; mkdir -p $D
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/ft python tools/prof_shape.py bf16 8192 8192 8192 2 > $D/a.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/off python tools/prof_shape.py bf16 8448 8448 8192 0 > $D/b.log 2>&1
echo done
