#!/bin/bash
# SIMT FT ablation: reference FMAs / per-k-block injection check compiled out (timing only)
D=gpurun_out/simtab; mkdir -p $D
export PYTHONUNBUFFERED=1
L=paper_2305_01024_b200
NREP=12 timeout 900 python tools/step_time.py f32_simt 8192 8192 8192 $L/libftgemm.so $L/libftgemm_simt_noref.so $L/libftgemm_simt_noinj.so $L/libftgemm_simt_noref_simt_noinj.so 2>&1 | grep -v "tiles_checked\|encode\|step\"" | tee $D/t.txt
