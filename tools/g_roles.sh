#!/bin/bash
# warp-role layout A/B: parity of the new default, then interleaved step timing against the old layout
D=gpurun_out/roles_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee $D/pytest.txt
L=paper_2305_01024_b200
for dt in bf16 tf32; do
timeout 300 python tools/step_time.py $dt 8192 8192 8192 $L/libftgemm.so $L/libftgemm_roles0.so 2>&1 | grep -v encode | tee -a $D/t.txt
done
timeout 300 python tools/step_time.py bf16 16384 16384 128 $L/libftgemm.so $L/libftgemm_roles0.so 2>&1 | grep -v encode | tee -a $D/t.txt
timeout 300 python tools/step_time.py bf16 4096 4096 4096 $L/libftgemm.so $L/libftgemm_roles0.so 2>&1 | grep -v encode | tee -a $D/t.txt
