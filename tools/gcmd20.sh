#!/bin/bash
L=paper_2305_01024_b200
for rep in 1 2; do
FTGEMM_LIB=$L/libftgemm_no_store_no_verify.so python tools/one_probe.py bf16 8192 8192 8192 2 nostore_nover
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so python tools/one_probe.py bf16 8192 8192 8192 2 nopass2_nover
FTGEMM_LIB=$L/libftgemm_no_pass2_no_verify.so python tools/one_probe.py bf16 8448 8448 8192 0 off8448_nopass2
FTGEMM_LIB=$L/libftgemm_no_store_no_verify.so python tools/one_probe.py bf16 8448 8448 8192 0 off8448_nostore
done
