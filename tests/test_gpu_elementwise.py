"""Element-by-element GPU parity, corrected values included.

Integer-valued inputs (|values| <= 4, K <= 1024) keep every product, partial
sum, row / column sum and carried checksum an integer below 2^23, so all three
precision variants compute them exactly (SURVEY.md 8(c) "product" pin).  With
integer ADD faults (the paper's "numerical offset") the
corrected element -- reconstructed from the row checksum, R_row[p] minus the
other row elements (R2) -- is exact too, and so is an
uncorrectable tile's faulty element (exact value + delta) and every residual
(exactly delta).  So C, every event and every residual must equal the oracle
BIT FOR BIT, in every tensor-core tile class and in the SIMT kernel, with
ragged edge tiles in M, N and K.

On real-valued data every element is checked against a per-element bound
derived from the accumulation arithmetic (gpu_util.elementwise_ratio,
DESIGN.md R18); corrected elements against the threshold-derived bound of the
row reconstruction.  FT on / FT off must agree bitwise (the checksums ride in
separate MMA rows and columns and never touch a data element's accumulation).
"""
import math

import numpy as np
import pytest

import oracle
import synth
from gpu_util import TOL, Case, detectable_sites, elementwise_ratio, frob, odt, oracle_operand, uncorrectable_mask

pytestmark = pytest.mark.gpu

CLASSES = [(256, 2), (256, 1), (128, 1), (128, 2)]
TC_CASES = [(d, c) for d in ("bf16", "tf32") for c in CLASSES]
ALL_CASES = TC_CASES + [("f32_simt", None)]
ids = lambda dc: f"{dc[0]}" + (f"-bn{dc[1][0]}cg{dc[1][1]}" if dc[1] else "")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2305_01024_b200 import ftgemm as F
    F.lib()
    oracle.build()


def _F():
    from paper_2305_01024_b200 import ftgemm as F
    return F


def _int_faults(plan, M, N, K):
    """Integer ADD faults: correctable ones in the first, interior and ragged
    last tiles (k in the first, a middle and the ragged last k-block), an SEU
    violation (two faults in one tile), a row-reference and a column-reference
    fault (checksum-only)."""
    tm, tn, T, U = plan.check_tile_m, plan.check_tile_n, plan.tiles_m, plan.tiles_n
    last_r = lambda ti: min(M - 1, ti * tm + tm - 1)
    last_c = lambda tj: min(N - 1, tj * tn + tn - 1)
    A = oracle.INJ_ADD
    f = [(0, 0, 0, 0, A, 0, 37.0),                                            # tile (0,0), first k-block
         (tm + 5, 2 * tn + 7, K // 2, 0, A, 0, -5.0),                         # interior
         (last_r(T - 1), last_c(U - 1), K - 1, 0, A, 0, 1000.0),              # ragged corner, last k
         ((T // 2) * tm + 1, (U - 1) * tn, 3 * plan.bk, 0, A, 0, -512.0),     # ragged last column tile
         ((T - 1) * tm, tn + 1, K - 1, 0, A, 0, 3.0),                         # ragged last row tile
         # SEU violation: two faults in tile (1, 0) -> uncorrectable, C left as computed
         (tm + 2, 3, 10, 0, A, 0, 64.0), (tm + 9, 11, 700, 0, A, 0, -96.0),
         # checksum-side faults: tile (0, 1) row reference, tile (2, 1) column reference
         (4, tn + 6, 200, 0, A, oracle.TGT_ROW_REF, 300.0),
         (2 * tm + 7, tn + 9, 500, 0, A, oracle.TGT_COL_REF, -300.0)]
    return f


def _check_bit_exact(c, ft_level):
    F = _F()
    assert np.array_equal(c.C.view(np.uint32), c.ref.C.astype(np.float32).view(np.uint32)), \
        np.argwhere(c.C != c.ref.C)[:5]
    assert c.counts_match() and c.events_match(), (c.counts, c.ref.counts)
    mine = {(e["tile_m"], e["tile_n"]): e for e in c.events}
    for e in c.ref.events:
        g = mine[(e["tile_m"], e["tile_n"])]
        # residuals are exact integers (delta, or 0 on the unflagged side)
        for key in ("resid_row", "resid_col"):
            if math.isfinite(e[key]):
                assert g[key] == e[key], (key, g, e)
        for key in ("tau_row", "tau_col"):
            if math.isfinite(e[key]) and e[key] > 0:
                assert abs(g[key] - e[key]) <= 1e-5 * e[key], (key, g, e)
    if ft_level == F.FT_CORRECT:
        assert c.counts["corrected"] == 5 and c.counts["uncorrectable"] == 1 and c.counts["checksum_only"] == 2


@pytest.mark.parametrize("dc", ALL_CASES, ids=ids)
def test_integer_faults_bit_exact(dc):
    """Integer inputs + integer ADD faults: C (corrected elements and the
    uncorrectable tile included), events, residuals bit-exact vs the oracle --
    every tile class, ragged M / N / K, alpha = 2, beta = -1; CORRECT and DETECT."""
    dtype, tile = dc
    F = _F()
    M, N, K = 1013, 2000, 1000
    plan = F.plan(dtype, M, N, K, tile=tile)
    assert (M % plan.check_tile_m) and (N % plan.check_tile_n) and (K % plan.bk)
    inj = _int_faults(plan, M, N, K)
    for lvl in (F.FT_CORRECT, F.FT_DETECT):
        c = Case(dtype, M, N, K, dist="int", alpha=2.0, beta=-1.0, injections=inj, ft=lvl, tile=tile)
        assert c.plan == plan
        _check_bit_exact(c, lvl)


@pytest.mark.parametrize("dc", ALL_CASES, ids=ids)
def test_integer_flips_corrected_exactly(dc):
    """Bit flips (the north_star default fault) on integer data: whatever the
    flipped partial sum becomes (huge, tiny, Inf), the element is rebuilt from
    the row checksum, so every corrected value is exact: C bit-identical to the
    oracle everywhere."""
    dtype, tile = dc
    F = _F()
    M, N, K = 777, 1304, 1024
    plan = F.plan(dtype, M, N, K, tile=tile)
    A, B, _ = synth.problem(M, N, K, dist="int", dtype=odt(dtype))
    inj = detectable_sites(dtype, 10, M, N, K, plan, oracle_operand(A, dtype), oracle_operand(B, dtype), seed=17)
    assert len(inj) >= 6
    c = Case(dtype, M, N, K, dist="int", alpha=1.0, beta=1.0, injections=inj, tile=tile)
    assert c.counts["corrected"] == len(inj) and c.counts_match() and c.events_match(), (c.counts, c.ref.counts)
    assert np.array_equal(c.C, c.ref.C)


@pytest.mark.parametrize("dist", ["signed", "unit"])
@pytest.mark.parametrize("dc", ALL_CASES, ids=ids)
def test_real_data_elementwise(dc, dist):
    """U[-1,1) / U[0,1) data with detectable flips in ten tiles: every element
    within its per-element bound (corrected ones within the row-reconstruction
    bound), events and counts bit-exact; SIMT within 1e-6 relative Frobenius
    (K <= 2048, R14)."""
    dtype, tile = dc
    F = _F()
    M, N, K = 1013, 2000, 1024
    plan = F.plan(dtype, M, N, K, tile=tile)
    A, B, _ = synth.problem(M, N, K, dist=dist, dtype=odt(dtype))
    inj = detectable_sites(dtype, 10, M, N, K, plan, oracle_operand(A, dtype), oracle_operand(B, dtype), seed=29)
    assert len(inj) >= 6
    c = Case(dtype, M, N, K, dist=dist, alpha=1.5, beta=-0.5, injections=inj, tile=tile)
    assert c.counts["corrected"] == len(inj) and c.counts_match() and c.events_match(), (c.counts, c.ref.counts)
    r = c.elementwise()
    assert r <= 1.0, r
    tol = 1e-6 if dtype == "f32_simt" else TOL[dtype]
    assert c.fro() < tol, c.fro()


@pytest.mark.parametrize("dc", ALL_CASES, ids=ids)
def test_ft_on_equals_ft_off_bitwise(dc):
    """No fault: FT on leaves C bit-identical to FT off (same class, same k order)."""
    dtype, tile = dc
    F = _F()
    M, N, K = 1013, 2000, 1024
    on = Case(dtype, M, N, K, alpha=1.5, beta=-0.5, run_oracle=False, tile=tile)
    off = Case(dtype, M, N, K, alpha=1.5, beta=-0.5, ft=F.FT_OFF, run_oracle=False, tile=tile)
    assert on.counts["tiles_detected"] == 0
    assert np.array_equal(on.C.view(np.uint32), off.C.view(np.uint32))


@pytest.mark.parametrize("dtype", ["bf16", "tf32", "f32_simt"])
def test_uncorrectable_and_detect_elementwise(dtype):
    """Real data: away from uncorrectable tiles every element is within its
    bound; inside them, all elements but the two faulty ones are too, and the
    faulty ones carry the fault (|C_gpu - C_clean| ~ |delta|) as in the oracle."""
    F = _F()
    M, N, K = 600, 704, 512
    plan = F.plan(dtype, M, N, K)
    tm, tn = plan.check_tile_m, plan.check_tile_n
    inj = [(1, 2, 30, 0, oracle.INJ_ADD, 0, 500.0), (7, 9, 100, 0, oracle.INJ_ADD, 0, -700.0),
           (tm + 3, tn + 4, 200, 0, oracle.INJ_ADD, 0, 250.0)]
    c = Case(dtype, M, N, K, injections=inj, alpha=1.0, beta=0.5)
    assert c.counts["uncorrectable"] == 1 and c.counts["corrected"] == 1 and c.events_match()
    skip = np.zeros((M, N), bool)
    skip[1, 2] = skip[7, 9] = True
    assert c.elementwise(skip=skip) <= 1.0
    for (r, q, _, _, _, _, d) in inj[:2]:
        assert abs(c.C[r, q] - c.ref.C[r, q]) <= 2 ** -7 * abs(d) + 1e-2 * abs(c.ref.C[r, q]) + 0.5
    d = Case(dtype, M, N, K, injections=inj[2:], ft=F.FT_DETECT, alpha=1.0, beta=0.5)
    assert d.counts["located"] == 1 and d.events_match()
    skip = np.zeros((M, N), bool)
    skip[tm + 3, tn + 4] = True
    assert d.elementwise(skip=skip) <= 1.0
    assert abs(d.C[tm + 3, tn + 4] - d.ref.C[tm + 3, tn + 4]) <= 2 ** -7 * 250.0 + 0.5


@pytest.mark.parametrize("K", [128, 96])
def test_small_k_three_epilogue_warpgroups(K):
    """TF32 with K <= 4 k-blocks on the narrow one-CTA tile runs three epilogue
    warpgroups (three TMEM accumulator buffers in flight): integer faults
    bit-exact (corrected, uncorrectable and reference faults), real data
    element-wise, FT on == FT off bitwise."""
    F = _F()
    M, N = 1013, 2000
    plan = F.plan("tf32", M, N, K, tile=(128, 1))
    inj = _int_faults(plan, M, N, K)
    c = Case("tf32", M, N, K, dist="int", alpha=2.0, beta=-1.0, injections=inj, tile=(128, 1))
    _check_bit_exact(c, F.FT_CORRECT)
    r = Case("tf32", M, N, K, alpha=1.5, beta=-0.5, tile=(128, 1),
             injections=detectable_sites("tf32", 8, M, N, K, plan, *[oracle_operand(x, "tf32") for x in
                                                                    synth.problem(M, N, K, dtype="f32")[:2]], seed=3))
    assert r.counts_match() and r.events_match() and r.elementwise() <= 1.0
    on = Case("tf32", M, N, K, run_oracle=False, tile=(128, 1))
    off = Case("tf32", M, N, K, ft=F.FT_OFF, run_oracle=False, tile=(128, 1))
    assert np.array_equal(on.C.view(np.uint32), off.C.view(np.uint32))
