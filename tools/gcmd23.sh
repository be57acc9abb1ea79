#!/bin/bash
L=paper_2305_01024_b200
for rep in 1 2; do
FTGEMM_LIB=$L/libftgemm_a128_no_verify_no_pass2.so python tools/one_probe.py bf16 8192 8192 8192 2 ft_a128_nov_nop2
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so python tools/one_probe.py bf16 8192 8192 8192 2 ft_nov_nop2
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so python tools/one_probe.py bf16 8250 8448 8192 0 off8250x8448
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so python tools/one_probe.py bf16 8448 8448 8192 0 off8448
done
