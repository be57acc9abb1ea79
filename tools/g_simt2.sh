#!/bin/bash
D=gpurun_out/simt2_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
L=paper_2305_01024_b200
timeout 600 python -m pytest tests -m gpu -q -x -k "simt or f32" 2>&1 | tail -2 | tee $D/pytest.txt
for s in "8192 8192 8192" "4096 4096 4096" "8192 8192 1024"; do
NREP=12 timeout 900 python tools/step_time.py f32_simt $s $L/libftgemm_prev.so $L/libftgemm.so 2>&1 | grep -v "tiles_checked\|encode\|step\"" | tee -a $D/t.txt
done
