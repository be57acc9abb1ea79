#!/bin/bash
# SIMT variants: parity of the default build, then interleaved timing of the builds
D=gpurun_out/simt_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -q -x -k "simt or f32" 2>&1 | tail -2 | tee $D/pytest.txt
FTGEMM_LIB=paper_2305_01024_b200/libftgemm_minb1.so timeout 600 python -m pytest tests -m gpu -q -x -k "simt or f32" 2>&1 | tail -2 | tee -a $D/pytest.txt
L=paper_2305_01024_b200
for s in "4096 4096 4096" "8192 8192 8192" "8192 8192 1024"; do
timeout 600 python tools/step_time.py f32_simt $s $L/libftgemm_prev.so $L/libftgemm.so $L/libftgemm_minb1.so 2>&1 | grep -v encode | tee -a $D/t.txt
done
