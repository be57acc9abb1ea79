#!/bin/bash
D=gpurun_out/encprof2; mkdir -p $D
timeout 300 ncu --set full --clock-control none --import-source on -k regex:encode_a_kernel -s 1 -c 1 -o $D/enc_a python tools/prof_run.py bf16 8192 2 > $D/p1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:encode_b_bf16_staged -s 1 -c 1 -o $D/enc_b python tools/prof_run.py bf16 8192 2 > $D/p2.log 2>&1
ls -la $D
