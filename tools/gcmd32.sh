#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do
for dt in bf16 tf32; do
python tools/one_probe.py $dt 8192 8192 8192 2 ft
python tools/one_probe.py $dt 8192 8192 8192 0 off
done
python tools/one_probe.py bf16 16384 16384 128 0 off_k128
python tools/one_probe.py bf16 4096 4096 4096 0 off_4k
done
