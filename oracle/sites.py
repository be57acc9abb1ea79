"""Per-site bit selection for fault injection — TEST INFRASTRUCTURE (calls only oracle/).

SURVEY.md §8(c) "Injection-site generator": for each site (row, col, k_elem) the
oracle computes the FP32-rounded partial accumulator x after the k-block that
contains k_elem, and the tile's thresholds; a bit b is "detectable" when
|flip(x,b) - x| >= 4 max(tau_row, tau_col) (or the flip is non-finite) and
"benign" when |flip(x,b) - x| <= min(tau_row, tau_col) / 4.  Only such bits are
used for bit-exact detection parity (reading R7).
"""
from __future__ import annotations

import numpy as np

from . import FT_DETECT, ftgemm


def _flip(x: np.float32, b: int) -> np.float32:
    u = np.array([x], dtype=np.float32).view(np.uint32)
    u ^= np.uint32(1 << b)
    return u.view(np.float32)[0]


def classify_bits(A, B, row, col, k_elem, *, tile_m, tile_n, bk, u_acc, lambda1, lambda2):
    """Return (detectable_bits, benign_bits, x, tau) for one accumulator site."""
    A = np.asarray(A, dtype=np.float32)
    B = np.asarray(B, dtype=np.float32)
    M, K = A.shape
    N = B.shape[1]
    ti, tj = row // tile_m, col // tile_n
    r0, c0 = ti * tile_m, tj * tile_n
    r1, c1 = min(M, r0 + tile_m), min(N, c0 + tile_n)
    res = ftgemm(A[r0:r1], B[:, c0:c1], tile_m=tile_m, tile_n=tile_n, bk=bk, u_acc=u_acc,
                 lambda1=lambda1, lambda2=lambda2, ft_level=FT_DETECT)
    tau_r = res.tau_row[row - r0, 0]
    tau_c = res.tau_col[0, col - c0]
    nkb = -(-K // bk)
    kb = min(k_elem // bk, nkb - 1)
    keff = min(K, (kb + 1) * bk)
    s = float(np.dot(A[row, :keff].astype(np.float64), B[:keff, col].astype(np.float64)))
    x = np.float32(s)
    det, ben = [], []
    hi, lo = 4.0 * max(tau_r, tau_c), 0.25 * min(tau_r, tau_c)
    for b in range(32):
        y = _flip(x, b)
        if not np.isfinite(y):
            det.append(b)
            continue
        d = abs(float(y) - float(x))
        if d >= hi:
            det.append(b)
        elif d <= lo:
            ben.append(b)
    return det, ben, float(x), (float(tau_r), float(tau_c))
