#!/bin/bash
D=gpurun_out/bn; mkdir -p $D
export PYTHONUNBUFFERED=1
for dt in bf16 tf32; do for s in "1024 1024 1024" "2048 2048 2048" "2048 2048 1024" "8192 512 8192" "8192 8192 1024" "4096 4096 1024"; do
timeout 300 python tools/bn_sweep.py $dt $s 256:2 256:1 128:1 128:2 2>&1 | tee -a $D/bn2.txt
done; done
