#!/bin/bash
# A/B of libftgemm_prev.so against libftgemm.so at cfg3 and the small-K cfg4 shape
D=gpurun_out/ab2_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
L=paper_2305_01024_b200
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee $D/pytest.txt
for s in "bf16 8192 8192 8192" "bf16 16384 16384 128" "tf32 16384 16384 128" "tf32 8192 8192 8192"; do
NREP=30 timeout 600 python tools/step_time.py $s $L/libftgemm_prev.so $L/libftgemm.so 2>&1 | grep -v "tiles_checked\|encode\|step\"" | tee -a $D/t.txt
done
