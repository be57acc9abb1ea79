#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do
for dt in bf16 tf32; do
python tools/one_probe.py $dt 8192 8192 8192 2 ft3d
FTGEMM_B3D=0 python tools/one_probe.py $dt 8192 8192 8192 2 ft2d
python tools/one_probe.py $dt 8192 8192 8192 0 off3d
FTGEMM_B3D=0 python tools/one_probe.py $dt 8192 8192 8192 0 off2d
done
done
