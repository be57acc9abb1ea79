"""B200-native fused online-ABFT GEMM (arXiv 2305.01024) — package root.

    from paper_2305_01024_b200 import ftgemm
    g = ftgemm.FTGemm("bf16", M, N, K)
    C = g(A, B)                       # encode + fused FT GEMM (CORRECT level)
    counts, events = g.report()

The compute path is libftgemm.so (C ABI, include/ftgemm.h, hand-written sm_100a
kernels).  ``paper_2305_01024_b200.distributed`` holds the M-block partition
over the GPUs of one node.
"""
from . import ftgemm  # noqa: F401

__all__ = ["ftgemm"]
