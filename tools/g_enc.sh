#!/bin/bash
# encode rewrite: parity + timing of the variants
D=gpurun_out/enc5; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_encode.py -q -x 2>&1 | tail -15 > $D/pytest_enc.txt; cat $D/pytest_enc.txt
for s in "bf16 8192 8192 8192" "tf32 8192 8192 8192" "f32_simt 8192 8192 8192" "bf16 16384 16384 128" "bf16 128 16384 16384" "bf16 4096 4096 4096"; do
  timeout 60 python tools/enc_time.py $s >> $D/t.txt 2>&1
done
cat $D/t.txt
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $D/pytest_all.txt; cat $D/pytest_all.txt
