#!/bin/bash
# A/B of libftgemm_prev.so (previous build) against libftgemm.so: GPU tests on the new build, then interleaved timing
D=gpurun_out/ab_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
L=paper_2305_01024_b200
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee $D/pytest.txt
for dt in bf16 tf32; do for r in 1 2; do
NREP=40 timeout 600 python tools/step_time.py $dt 8192 8192 8192 $L/libftgemm_prev.so $L/libftgemm.so 2>&1 | grep -v "tiles_checked\|encode" | tee -a $D/t.txt
done; done
NREP=40 timeout 600 python tools/step_time.py bf16 4096 4096 4096 $L/libftgemm_prev.so $L/libftgemm.so 2>&1 | grep -v "tiles_checked\|encode" | tee -a $D/t.txt
