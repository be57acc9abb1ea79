#!/bin/bash
# tile class (BN x CG) sweep of the FT run at the cfg2 square sizes
D=gpurun_out/bn; mkdir -p $D
export PYTHONUNBUFFERED=1
for dt in bf16 tf32; do for n in 3072 4096 6144 8192; do
timeout 300 python tools/bn_sweep.py $dt $n $n $n 256:2 256:1 128:1 128:2 2>&1 | tee -a $D/bn.txt
done; done
