#!/bin/bash
L=paper_2305_01024_b200
for rep in 1 2; do
python tools/one_probe.py bf16 8192 8192 8192 2 ft
FTGEMM_LIB=$L/libftgemm_no_verify.so python tools/one_probe.py bf16 8192 8192 8192 2 nover
FTGEMM_LIB=$L/libftgemm_no_verify_no_pass2.so python tools/one_probe.py bf16 8192 8192 8192 2 nover_nop2
FTGEMM_LIB=$L/libftgemm_a128_no_verify_no_pass2.so python tools/one_probe.py bf16 8192 8192 8192 2 a128_nover_nop2
python tools/one_probe.py bf16 8250 8448 8192 0 off_same_units
done
