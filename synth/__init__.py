"""Seeded, counter-based synthetic inputs shared by the oracle harness and the CUDA path.

This module holds NO arithmetic of the method (no checksums, no GEMM): only the
pseudo-random element generator, dtype rounding of the generated values, and the
seeded choice of injection *sites* (which tile / element / k-step gets a fault).
Both sides (``oracle/`` via the tests, and the CUDA path via the tests / bench)
consume exactly the same bytes produced here.

Generator:
    key   = splitmix64(seed)
    z     = splitmix64(key + (r * cols + c))          # uint64, wrapping
    u     = (z >> 40) * 2**-24                        # 24-bit uniform in [0, 1)
    value = lo + (hi - lo) * u   (in float64, then rounded to float32, then
                                  RNE-rounded to bfloat16 for BF16 operands)
Integer mode: value = ((z >> 40) % (2*imax + 1)) - imax, exact in every dtype.

Because it is counter based, any sub-block (a rank's row block, a sampled tile)
can be regenerated from global indices alone.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 230501024
SEED_A, SEED_B, SEED_C, SEED_PLAN = 0, 1, 2, 3

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on a uint64 array (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _stream(seed: int, rows: int, cols: int, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
    key = splitmix64(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]
    r = np.arange(r0, r1, dtype=np.uint64)[:, None]
    c = np.arange(c0, c1, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        idx = r * np.uint64(cols) + c
        return splitmix64(idx + key)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 -> bfloat16 (round-to-nearest-even); returns uint16 bit patterns."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return rounded.astype(np.uint16)


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    return (np.asarray(h, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def matrix(seed: int, rows: int, cols: int, *, dist: str = "signed", dtype: str = "f32",
           r0: int = 0, r1: int | None = None, c0: int = 0, c1: int | None = None,
           imax: int = 4) -> np.ndarray:
    """Generate block [r0:r1, c0:c1] of the (rows x cols) matrix for ``seed``.

    dist: "signed" = U[-1,1), "unit" = U[0,1), "int" = integers in [-imax, imax].
    dtype: "f32" returns float32 values; "bf16" returns the float32 *values* of the
    RNE-rounded bfloat16 numbers (exactly representable, use ``to_bf16_bits``).
    """
    r1 = rows if r1 is None else r1
    c1 = cols if c1 is None else c1
    z = _stream(seed, rows, cols, r0, r1, c0, c1)
    top = (z >> np.uint64(40)).astype(np.float64)          # 24 random bits
    if dist == "int":
        v = (np.mod(top, 2 * imax + 1) - imax)
    else:
        u = top * (2.0 ** -24)
        lo, hi = (-1.0, 1.0) if dist == "signed" else (0.0, 1.0)
        v = lo + (hi - lo) * u
    v = v.astype(np.float32)
    if dtype == "bf16":
        v = bf16_bits_to_f32(f32_to_bf16_bits(v))
    return v


def problem(M: int, N: int, K: int, *, dist: str = "signed", dtype: str = "f32",
            seed: int = BASE_SEED, with_c: bool = True):
    """A (M x K), B (K x N), C_in (M x N) as float32 arrays holding the operand values."""
    A = matrix(seed + SEED_A, M, K, dist=dist, dtype=dtype)
    B = matrix(seed + SEED_B, K, N, dist=dist, dtype=dtype)
    C = matrix(seed + SEED_C, M, N, dist=dist, dtype=dtype) if with_c else None
    return A, B, C


def to_torch(x: np.ndarray, dtype: str):
    """float32 numpy values -> torch CPU tensor of the operand dtype (bit-exact)."""
    import torch
    if dtype == "bf16":
        bits = f32_to_bf16_bits(x).view(np.int16)
        return torch.from_numpy(np.ascontiguousarray(bits)).view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))


def injection_sites(n: int, M: int, N: int, K: int, tile_m: int, tile_n: int, bk: int, *,
                    seed: int = BASE_SEED + SEED_PLAN, one_per_tile: bool = True):
    """Seeded fault sites: list of (row, col, k_elem). At most one per tile when
    ``one_per_tile`` (the paper's SEU model, §4.1). The bit to flip is
    chosen per site by the caller (tests use the oracle's per-site generator)."""
    tm = -(-M // tile_m)
    tn = -(-N // tile_n)
    ntiles = tm * tn
    if one_per_tile and n > ntiles:
        raise ValueError(f"{n} sites requested but only {ntiles} tiles")
    key = splitmix64(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]
    ctr = [0]

    def draw(mod: int) -> int:
        with np.errstate(over="ignore"):
            z = splitmix64(np.array([ctr[0]], dtype=np.uint64) + key)[0]
        ctr[0] += 1
        return int(z % np.uint64(mod))

    sites, used = [], set()
    while len(sites) < n:
        t = draw(ntiles)
        if one_per_tile and t in used:
            continue
        ti, tj = divmod(t, tn)
        bm = min(tile_m, M - ti * tile_m)
        bn = min(tile_n, N - tj * tile_n)
        p, q, k = draw(bm), draw(bn), draw(K)
        used.add(t)
        sites.append((ti * tile_m + p, tj * tile_n + q, k))
    return sites


# ---- the same generator in torch (device-side generation of large inputs) ----
def _u64(v: int):
    """uint64 constant as the int64 torch arithmetic wraps it."""
    return v - (1 << 64) if v >= (1 << 63) else v


def _srl(x, s: int):
    """logical right shift of int64 tensors (as uint64)."""
    return (x >> s) & ((1 << (64 - s)) - 1)


def splitmix64_torch(x):
    """splitmix64 on an int64 torch tensor, bit-identical to splitmix64() (the
    int64 multiply wraps modulo 2^64 like the uint64 one)."""
    z = x + _u64(0x9E3779B97F4A7C15)
    z = (z ^ _srl(z, 30)) * _u64(0xBF58476D1CE4E5B9)
    z = (z ^ _srl(z, 27)) * _u64(0x94D049BB133111EB)
    return z ^ _srl(z, 31)


def matrix_torch(seed: int, rows: int, cols: int, *, dist: str = "signed", dtype: str = "f32",
                 r0: int = 0, r1: int | None = None, device="cuda", chunk_rows: int = 2048):
    """Rows [r0, r1) of matrix(seed, rows, cols) generated on `device` (torch),
    element-for-element identical to the numpy generator (tests/test_synth.py).
    Used for inputs too large to generate on the host in time (bench cfg5)."""
    import torch
    r1 = rows if r1 is None else r1
    key = int(splitmix64(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])
    out = torch.empty(r1 - r0, cols, dtype=torch.bfloat16 if dtype == "bf16" else torch.float32, device=device)
    c = torch.arange(cols, dtype=torch.int64, device=device)[None, :]
    for a in range(r0, r1, chunk_rows):
        b = min(r1, a + chunk_rows)
        r = torch.arange(a, b, dtype=torch.int64, device=device)[:, None]
        z = splitmix64_torch(r * cols + c + _u64(key))
        top = _srl(z, 40).to(torch.float64)
        if dist == "int":
            v = torch.remainder(top, 9.0) - 4.0
        else:
            lo, hi = (-1.0, 1.0) if dist == "signed" else (0.0, 1.0)
            v = lo + (hi - lo) * (top * 2.0 ** -24)
        out[a - r0:b - r0] = v.to(torch.float32).to(out.dtype)
    return out
