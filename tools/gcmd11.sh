#!/bin/bash
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for lib in libftgemm.so libftgemm_wg1.so; do
  for shape in "16384 16384 128" "8192 8192 1024" "8192 8192 8192" "4096 4096 4096"; do
    for dt in bf16 tf32; do
      echo -n "$lib "; FTGEMM_LIB=paper_2305_01024_b200/$lib timeout 120 python tools/perf_probe.py $dt $shape 2 2>&1 | tail -1 | cut -c1-105
    done
  done
  echo -n "$lib off "; FTGEMM_LIB=paper_2305_01024_b200/$lib timeout 120 python tools/perf_probe.py bf16 8192 8192 8192 0 2>&1 | tail -1 | cut -c1-105
  echo -n "$lib off "; FTGEMM_LIB=paper_2305_01024_b200/$lib timeout 120 python tools/perf_probe.py bf16 16384 16384 128 0 2>&1 | tail -1 | cut -c1-105
done
