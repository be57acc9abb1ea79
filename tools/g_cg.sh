#!/bin/bash
# 2-CTA bring-up: correctness under FTGEMM_CG=2, then CG=1 vs CG=2 timing
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for cg in 2; do
  FTGEMM_CG=$cg timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok cg=$cg')" 2>&1 | tail -5
done
FTGEMM_CG=2 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for cg in 1 2; do
  for ft in 0 2; do
    FTGEMM_CG=$cg timeout 120 python tools/perf_probe.py bf16 8192 8192 8192 $ft 2>&1 | tail -1
    FTGEMM_CG=$cg timeout 120 python tools/perf_probe.py tf32 8192 8192 8192 $ft 2>&1 | tail -1
  done
done
