#!/bin/bash
export PYTHONUNBUFFERED=1
D=gpurun_out/r31; mkdir -p $D
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for shape in "16384 16384 128" "8192 8192 1024" "8192 8192 8192"; do
  timeout 120 python tools/perf_probe.py bf16 $shape 2 2>&1 | tail -1 | cut -c1-110
  timeout 120 python tools/perf_probe.py tf32 $shape 2 2>&1 | tail -1 | cut -c1-110
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/k128_ft python tools/prof_shape.py bf16 16384 16384 128 2 > $D/a.log 2>&1
FTGEMM_LIB=paper_2305_01024_b200/libftgemm_no_verify.so timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/k128_nover python tools/prof_shape.py bf16 16384 16384 128 2 > $D/b.log 2>&1
echo done
