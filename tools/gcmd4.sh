#!/bin/bash
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q -k "cta_pair" 2>&1 | tail -4
for lib in libftgemm.so libftgemm_no_verify.so libftgemm_pass1_ldonly.so; do
  for shape in "16384 16384 128" "8192 8192 1024" "8192 8192 8192"; do
    echo -n "$lib "; FTGEMM_LIB=paper_2305_01024_b200/$lib timeout 120 python tools/perf_probe.py bf16 $shape 2 2>&1 | tail -1 | cut -c1-110
  done
  echo -n "$lib "; FTGEMM_LIB=paper_2305_01024_b200/$lib timeout 120 python tools/perf_probe.py tf32 16384 16384 128 2 2>&1 | tail -1 | cut -c1-110
done
timeout 120 python tools/perf_probe.py tf32 16384 16384 128 0 2>&1 | tail -1 | cut -c1-110
