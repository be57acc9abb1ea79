#!/bin/bash
D=gpurun_out/enc_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_encode.py -q -x 2>&1 | tail -3 | tee $D/pytest.txt
for lib in libftgemm.so; do
  for dt in bf16 tf32; do
    echo "== $lib $dt"; FTGEMM_LIB=paper_2305_01024_b200/$lib timeout 300 python tools/enc_time.py $dt 8192 8192 8192
  done
done 2>&1 | tee $D/enc.txt
