#!/bin/bash
# SIMT variants: interleaved timing of the default build against variant builds ($@)
D=gpurun_out/simt_${1:-x}; shift; mkdir -p $D
export PYTHONUNBUFFERED=1
L=paper_2305_01024_b200
for s in "4096 4096 4096" "8192 8192 8192"; do
timeout 600 python tools/step_time.py f32_simt $s $L/libftgemm.so "$@" 2>&1 | grep -v encode | tee -a $D/t.txt
done
