#!/bin/bash
# CG=1 vs CG=2 over shapes, group sweep for CG=2
export PYTHONUNBUFFERED=1
for shape in "8192 8192 8192" "4096 4096 4096" "2048 2048 2048" "16384 16384 128" "128 16384 16384" "16384 128 16384" "8192 8192 1024" "4096 4096 1024"; do
  for dt in bf16 tf32; do
    for cg in 1 2; do
      for ft in 0 2; do
        echo -n "cg=$cg "; FTGEMM_CG=$cg timeout 120 python tools/perf_probe.py $dt $shape $ft 2>&1 | tail -1 | cut -c1-130
      done
    done
  done
done
for g in 4 6 8 12 16; do
  echo -n "G=$g "; FTGEMM_GROUP=$g FTGEMM_CG=2 timeout 120 python tools/perf_probe.py bf16 8192 8192 8192 2 2>&1 | tail -1 | cut -c1-120
done
