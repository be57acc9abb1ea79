#!/bin/bash
D=gpurun_out/k128; mkdir -p $D
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/ft python tools/prof_shape.py bf16 16384 16384 128 2 > $D/p1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/off python tools/prof_shape.py bf16 16384 16384 128 0 > $D/p2.log 2>&1
ls $D
