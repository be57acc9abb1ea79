#!/bin/bash
L=paper_2305_01024_b200
for rep in 1 2; do
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so python tools/one_probe.py bf16 8192 8192 8192 2 ft8192
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so python tools/one_probe.py bf16 8250 8320 8192 2 ft8250x8320
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so python tools/one_probe.py bf16 8448 8448 8192 0 off8448
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so python tools/one_probe.py bf16 8400 8400 8192 0 off8400
done
