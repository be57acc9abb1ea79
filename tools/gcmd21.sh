#!/bin/bash
D=gpurun_out/r39; mkdir -p $D
L=paper_2305_01024_b200
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so timeout 300 ncu --set full --clock-control none -k regex:tc_ftgemm -s 1 -c 1 -o $D/ft python tools/prof_shape.py bf16 8192 8192 8192 2 > $D/a.log 2>&1
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so timeout 300 ncu --set full --clock-control none -k regex:tc_ftgemm -s 1 -c 1 -o $D/off python tools/prof_shape.py bf16 8448 8448 8192 0 > $D/b.log 2>&1
echo done
