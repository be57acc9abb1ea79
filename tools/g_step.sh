#!/bin/bash
D=gpurun_out/step_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
[ -n "$T" ] && timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee $D/pytest.txt
for dt in bf16 tf32; do
timeout 300 python tools/step_time.py $dt 8192 8192 8192 paper_2305_01024_b200/libftgemm_prev.so paper_2305_01024_b200/libftgemm.so 2>&1 | tee -a $D/step.txt
done
timeout 300 python tools/step_time.py bf16 16384 16384 128 paper_2305_01024_b200/libftgemm_prev.so paper_2305_01024_b200/libftgemm.so 2>&1 | tee -a $D/step.txt
timeout 300 python tools/step_time.py f32_simt 4096 4096 4096 paper_2305_01024_b200/libftgemm_prev.so paper_2305_01024_b200/libftgemm.so 2>&1 | tee -a $D/step.txt
