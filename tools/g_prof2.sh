#!/bin/bash
D=gpurun_out/prof2; mkdir -p $D
timeout 300 ncu --set full --clock-control none --import-source on -k regex:simt_ftgemm -s 1 -c 1 -o $D/simt_off python tools/prof_shape.py f32_simt 4096 4096 4096 0 > $D/p1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:simt_ftgemm -s 1 -c 1 -o $D/simt_ft python tools/prof_shape.py f32_simt 4096 4096 4096 2 > $D/p2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:encode_a -s 1 -c 1 -o $D/enc_a python tools/prof_run.py bf16 8192 2 > $D/p3.log 2>&1
timeout 300 python tools/enc_time.py bf16 8192 8192 8192 > $D/enc.txt 2>&1
ls $D
