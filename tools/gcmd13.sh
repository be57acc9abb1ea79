#!/bin/bash
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for shape in "128 16384 16384" "16384 128 16384" "4096 128 4096"; do
  for dt in bf16 tf32; do
    for ft in 2 0; do timeout 120 python tools/perf_probe.py $dt $shape $ft 2>&1 | tail -1 | cut -c1-110; done
  done
done
