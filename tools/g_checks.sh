#!/bin/bash
# Device-side bounds assertions (-DFTGEMM_DEBUG_CHECKS: item / flag / norm
# indices of the in-kernel encode, trap on violation) under the GPU tests that
# reach the extended modes -- a stand-in for compute-sanitizer memcheck, which
# is closed on the GPU pool.  Build first (on the CPU host):
#   python -c "from paper_2305_01024_b200 import build; build.build(defines=['-DFTGEMM_DEBUG_CHECKS'], out='paper_2305_01024_b200/libftgemm_checks.so')"
D=gpurun_out/checks; mkdir -p $D
FTGEMM_LIB=paper_2305_01024_b200/libftgemm_checks.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_elementwise.py -m gpu -q -x \
  -k "fused or degenerate or online or cfg5 or large_indexing" 2>&1 | tail -4 | tee $D/pytest.txt
FTGEMM_LIB=paper_2305_01024_b200/libftgemm_checks.so timeout 300 python tools/fused_a_time.py bf16 32768 32768 16384 2>&1 | tail -1 | tee $D/cfg5_fused.txt
