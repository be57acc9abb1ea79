#!/bin/bash
# source-level ncu capture of the fused kernel at the HBM-bound cfg4 shape (K = 128)
D=gpurun_out/k128; mkdir -p $D
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 2 -c 1 -o $D/k128_ft python tools/prof_shape.py bf16 16384 16384 128 2 > $D/p1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 2 -c 1 -o $D/k128_off python tools/prof_shape.py bf16 16384 16384 128 0 > $D/p2.log 2>&1
tail -2 $D/p1.log $D/p2.log
