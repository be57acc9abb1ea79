#!/bin/bash
D=gpurun_out/encvar_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
L=paper_2305_01024_b200
for dt in bf16 tf32; do
NREP=60 timeout 600 python tools/step_time.py $dt 8192 8192 8192 $L/libftgemm.so $L/libftgemm_encb_l2p.so $L/libftgemm_encb_na.so $L/libftgemm_enca_l2p.so $L/libftgemm_enc_afirst.so 2>&1 | grep -v "run\"\|tiles_checked" | tee -a $D/t.txt
done
