#!/bin/bash
L=paper_2305_01024_b200
for rep in 1 2; do
python tools/one_probe.py bf16 8192 8192 8192 2 ft
FTGEMM_LIB=$L/libftgemm_lean1.so python tools/one_probe.py bf16 8192 8192 8192 2 lean1
FTGEMM_LIB=$L/libftgemm_lean2.so python tools/one_probe.py bf16 8192 8192 8192 2 lean2
done
