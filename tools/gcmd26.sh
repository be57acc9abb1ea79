#!/bin/bash
L=paper_2305_01024_b200
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
python tools/one_probe.py bf16 8192 8192 8192 2 ft
python tools/one_probe.py bf16 8192 8192 8192 0 off
python tools/one_probe.py tf32 8192 8192 8192 2 ft
python tools/one_probe.py tf32 8192 8192 8192 0 off
python tools/one_probe.py bf16 16384 16384 128 2 ft
done
