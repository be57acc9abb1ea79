#!/bin/bash
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q -k "simt or f32" 2>&1 | tail -3
for lib in libftgemm.so libftgemm_sk16.so; do
  for s in 4096 8192; do
    for ft in 0 2; do
      echo -n "$lib "; FTGEMM_LIB=paper_2305_01024_b200/$lib timeout 120 python tools/perf_probe.py f32_simt $s $s $s $ft 2>&1 | tail -1 | cut -c1-120
    done
  done
done
FTGEMM_LIB=paper_2305_01024_b200/libftgemm_sk16.so timeout 600 python -m pytest tests -m gpu -x -q -k "simt or f32" 2>&1 | tail -3
