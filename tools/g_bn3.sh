#!/bin/bash
D=gpurun_out/bn; mkdir -p $D
export PYTHONUNBUFFERED=1
for dt in bf16 tf32; do for s in "16384 16384 128" "8192 8192 128" "16384 16384 256" "8192 8192 512"; do
timeout 300 python tools/bn_sweep.py $dt $s 256:2 256:1 128:1 128:2 2>&1 | tee -a $D/bn3.txt
done; done
