#!/bin/bash
export PYTHONUNBUFFERED=1
D=gpurun_out/r35; mkdir -p $D
timeout 300 ncu --set full --clock-control none --import-source on -k regex:simt_ftgemm -s 1 -c 1 -o $D/simt_off python tools/prof_shape.py f32_simt 4096 4096 4096 0 > $D/a.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:simt_ftgemm -s 1 -c 1 -o $D/simt_ft python tools/prof_shape.py f32_simt 4096 4096 4096 2 > $D/b.log 2>&1
echo done
