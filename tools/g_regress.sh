#!/bin/bash
D=gpurun_out/regress_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
L=paper_2305_01024_b200
for r in 1 2; do
NREP=40 timeout 600 python tools/step_time.py bf16 8192 8192 8192 $L/libftgemm_start.so $L/libftgemm.so 2>&1 | grep -v tiles_checked | tee -a $D/t.txt
done
