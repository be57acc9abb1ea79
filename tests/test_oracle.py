"""Pins for the CPU oracle against what the paper and the mathematics fix.

Each test names what it pins.  None of these re-types the oracle's formula: they
use exact integer arithmetic (Python ints / numpy int64), closed forms, the
paper's stated locate/correct behaviour, brute force on
small tiles and correctly-rounded rational arithmetic (fractions.Fraction).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- helpers ---

def f32_round(x: Fraction) -> np.float32:
    """Correctly rounded (ties-to-even) Fraction -> float32, normal and subnormal."""
    if x == 0:
        return np.float32(0.0)
    s = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if a < Fraction(2) ** e:
        e -= 1
    if a >= Fraction(2) ** (e + 1):
        e += 1
    ulp = Fraction(2) ** (max(e, -126) - 23)
    q = a / ulp
    fl = q.numerator // q.denominator
    rem = q - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return np.float32(s * float(fl * ulp))


def fma32(a, b, c) -> np.float32:
    return f32_round(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def flip32(x, bit):
    u = np.array([x], dtype=np.float32).view(np.uint32)
    u ^= np.uint32(1 << bit)
    return u.view(np.float32)[0]


def ints(seed, r, c, imax=4):
    return synth.matrix(seed, r, c, dist="int", imax=imax)


# ------------------------------------------------------------ golden 2x2 ----

def test_golden_spec_2x2(oracle_lib):
    """SPEC.md:51/223/233/243/244/258 worked 2x2 example of PAPER.md Eq. (1)-(3)."""
    g = json.load(open(os.path.join(GOLD, "spec_2x2.json")))
    A = np.array(g["A"], np.float32)
    B = np.array(g["B"], np.float32)
    r = oracle.ftgemm(A, B, tile_m=2, tile_n=2)
    assert r.C.tolist() == g["C"]["value"]
    assert oracle.encode_col(A, 2)[0].tolist() == g["eTA"]["value"]
    assert oracle.encode_row(B, 2)[0].tolist() == g["Be"]["value"]
    # the carried references are the row / column sums of C (Eq. 3)
    assert np.all(r.resid_row == 0) and np.all(r.resid_col == 0)
    Cv = np.array(g["C"]["value"], np.float64)
    assert Cv.sum(axis=0).tolist() == g["Cc"]["value"]
    assert Cv.sum(axis=1).tolist() == g["Cr"]["value"]
    f = g["fault"]
    inj = [(f["row"], f["col"], 1, 0, oracle.INJ_ADD, oracle.TGT_ACC, float(f["delta"]))]
    det = oracle.ftgemm(A, B, tile_m=2, tile_n=2, ft_level=oracle.FT_DETECT, injections=inj)
    assert det.C.tolist() == f["faulty_C"]
    assert det.resid_row[:, 0].tolist() == [5.0, 0.0]
    assert det.resid_col[0].tolist() == [0.0, 5.0]
    cor = oracle.ftgemm(A, B, tile_m=2, tile_n=2, injections=inj)
    assert cor.C.tolist() == g["C"]["value"]
    assert cor.counts["corrected"] == 1
    ev = cor.events[0]
    assert (ev["row"], ev["col"], ev["kind"]) == (0, 1, oracle.EV_CORRECTED)
    assert ev["resid_row"] == 5.0 and ev["resid_col"] == 5.0
    two = [(0, 0, 1, 0, oracle.INJ_ADD, 0, 5.0), (1, 1, 1, 0, oracle.INJ_ADD, 0, 5.0)]
    r2 = oracle.ftgemm(A, B, tile_m=2, tile_n=2, injections=two)
    assert r2.counts["uncorrectable"] == 1 and r2.counts["corrected"] == 0


# ---------------------------------------------------------------- product ---

def test_product_identity_and_zero(oracle_lib):
    """A = I -> C = B exactly; A = 0 -> C = beta C_in (special cases)."""
    B = synth.matrix(7, 33, 40, dtype="f32")
    Cin = synth.matrix(8, 33, 40, dtype="f32")
    r = oracle.ftgemm(np.eye(33, dtype=np.float32), B, tile_m=16, tile_n=16)
    assert np.array_equal(r.C, B)
    r = oracle.ftgemm(np.zeros((33, 33), np.float32), B, Cin, alpha=2.0, beta=-0.5, tile_m=16, tile_n=16)
    assert np.array_equal(r.C, (np.float64(-0.5) * Cin).astype(np.float32))
    assert r.counts["tiles_detected"] == 0


@pytest.mark.parametrize("acc", ["fp64", "fp32seq"])
def test_product_integer_exact(oracle_lib, acc):
    """Integer inputs |v|<=4, K<=1024: every value < 2^22, so both accumulation
    modes must equal exact integer matmul (numpy int64) bit for bit."""
    M, N, K = 70, 90, 300
    A, B = ints(1, M, K), ints(2, K, N)
    Cin = ints(3, M, N)
    exact = A.astype(np.int64) @ B.astype(np.int64)
    r = oracle.ftgemm(A, B, Cin, alpha=2.0, beta=-1.0, acc=acc, tile_m=32, tile_n=64)
    assert np.array_equal(r.P, exact.astype(np.float64))
    assert np.array_equal(r.C.astype(np.int64), 2 * exact - Cin.astype(np.int64))
    # Eq. (3): e^T(AB) = (e^T A)B and (AB)e = A(Be) exactly -> residuals exactly 0
    assert np.all(r.resid_row == 0) and np.all(r.resid_col == 0)
    assert r.counts["tiles_detected"] == 0


def test_product_fp64_vs_independent_matmul(oracle_lib):
    """FP64 product agrees with numpy's float64 matmul to FP64 rounding."""
    A, B, _ = synth.problem(64, 48, 200, dist="signed", with_c=False)
    r = oracle.ftgemm(A, B, tile_m=32, tile_n=32, ft_level=oracle.FT_OFF)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.max(np.abs(r.P - ref)) < 1e-12
    g = oracle.gemm_f64(A, B)
    assert np.max(np.abs(g - ref)) < 1e-12


def test_fp32seq_is_sequential_fma(oracle_lib):
    """acc_mode FP32SEQ = one correctly-rounded fmaf per k, ascending k (the
    paper's SGEMM numerics), checked with exact rationals,
    including a bit flip at a k-block boundary and the fmaf alpha/beta epilogue."""
    M, N, K, bk = 3, 4, 19, 8
    A, B, Cin = synth.problem(M, N, K, dist="signed", seed=99)
    inj = [(1, 2, 9, 27, oracle.INJ_FLIP, oracle.TGT_ACC, 0.0)]   # k_elem 9 -> k-block 1 -> k_eff 16
    r = oracle.ftgemm(A, B, Cin, alpha=1.5, beta=-0.5, acc="fp32seq", tile_m=4, tile_n=4, bk=bk,
                      ft_level=oracle.FT_DETECT, injections=inj)
    for p in range(M):
        for q in range(N):
            acc = np.float32(0.0)
            for k in range(K):
                acc = fma32(A[p, k], B[k, q], acc)
                if (p, q) == (1, 2) and k == 15:
                    acc = flip32(acc, 27)
            assert r.P[p, q] == float(acc), (p, q)
            bc = np.float32(np.float32(-0.5) * Cin[p, q])
            assert r.C[p, q] == fma32(np.float32(1.5), acc, bc)


# ----------------------------------------------------------------- encode ---

def test_encode_linearity_and_sums(oracle_lib):
    """e^T A per tile equals exact integer column sums; encode is linear."""
    A = ints(11, 50, 37)
    B = ints(12, 37, 45)
    Ac = oracle.encode_col(A, 16)
    Br = oracle.encode_row(B, 20)
    Ai = A.astype(np.int64)
    Bi = B.astype(np.int64)
    for i in range(4):
        assert np.array_equal(Ac[i], Ai[16 * i:16 * (i + 1)].sum(axis=0))
    for j in range(3):
        assert np.array_equal(Br[j], Bi[:, 20 * j:20 * (j + 1)].sum(axis=1))
    A2 = ints(13, 50, 37)
    assert np.array_equal(oracle.encode_col(A + 2 * A2, 16), Ac + 2 * oracle.encode_col(A2, 16))


# ------------------------------------------------------- locate / correct ---

@pytest.mark.parametrize("tile", [4, 8])
def test_bruteforce_locate_correct(oracle_lib, tile):
    """Every (p,q) of a tile x delta in {+-1, +-1e3, +Inf, NaN}: exactly that
    element is located and corrected back to the exact value (PAPER.md:317,
    :505); the other tiles stay clean."""
    M, N, K = 2 * tile, 2 * tile, 24
    A, B = ints(21, M, K), ints(22, K, N)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float32)
    for delta in (1.0, -1.0, 1e3, -1e3, math.inf, math.nan):
        for p in range(tile):
            for q in range(tile):
                row, col = tile + p, q            # tile (1, 0)
                inj = [(row, col, 5, 0, oracle.INJ_ADD, oracle.TGT_ACC, delta)]
                r = oracle.ftgemm(A, B, tile_m=tile, tile_n=tile, bk=8, injections=inj)
                assert r.counts["corrected"] == 1 and r.counts["tiles_detected"] == 1
                ev = r.events[0]
                assert (ev["row"], ev["col"], ev["tile_m"], ev["tile_n"]) == (row, col, 1, 0)
                assert np.array_equal(r.C, exact), (delta, p, q)


def test_flip_delta_closed_form(oracle_lib):
    """Flipping bit 22 of the FP32 partial 6.0 (= 1.5 * 2^2) gives 4.0, so the
    faulty element is exact - 2 (closed form of the FLIP injection)."""
    A = np.array([[1, 2, 3, 4]], np.float32)        # partial over k<2 : 1*1+2*2.5=6
    B = np.array([[1], [2.5], [7], [1]], np.float32)
    inj = [(0, 0, 1, 22, oracle.INJ_FLIP, oracle.TGT_ACC, 0.0)]
    r = oracle.ftgemm(A, B, tile_m=1, tile_n=1, bk=2, ft_level=oracle.FT_DETECT, injections=inj)
    assert r.P[0, 0] == (1 + 5 + 21 + 4) - 2.0
    assert r.counts["located"] == 1


def test_seu_violation_uncorrectable(oracle_lib):
    """Two faults in one tile (SEU assumption violated): reported
    uncorrectable and C left as computed (not 'corrected' into garbage)."""
    A, B = ints(31, 16, 40), ints(32, 40, 16)
    exact = A.astype(np.int64) @ B.astype(np.int64)
    inj = [(1, 2, 3, 0, oracle.INJ_ADD, 0, 7.0), (5, 9, 30, 0, oracle.INJ_ADD, 0, -3.0)]
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16, injections=inj)
    assert r.counts["uncorrectable"] == 1 and r.counts["corrected"] == 0
    exp = exact.astype(np.float64)
    exp[1, 2] += 7
    exp[5, 9] -= 3
    assert np.array_equal(r.C.astype(np.float64), exp)
    assert r.events[0]["n_rows"] == 2 and r.events[0]["n_cols"] == 2


def test_checksum_side_faults(oracle_lib):
    """A fault in a carried reference flags one row (or column) only: C is
    untouched and the tile counts as checksum_only.  Row-ref + col-ref faults
    of different size flag 1 row + 1 column with inconsistent magnitudes: the
    guard reports uncorrectable instead of 'correcting' an innocent element."""
    A, B = ints(41, 16, 40), ints(42, 40, 16)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float32)
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16,
                      injections=[(3, 4, 10, 0, oracle.INJ_ADD, oracle.TGT_ROW_REF, 50.0)])
    assert r.counts["checksum_only"] == 1 and np.array_equal(r.C, exact)
    assert r.events[0]["row"] == 3 and r.events[0]["col"] == -1
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16,
                      injections=[(3, 4, 10, 0, oracle.INJ_ADD, oracle.TGT_COL_REF, 50.0)])
    assert r.counts["checksum_only"] == 1 and np.array_equal(r.C, exact)
    assert r.events[0]["row"] == -1 and r.events[0]["col"] == 4
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16,
                      injections=[(3, 4, 10, 0, oracle.INJ_ADD, oracle.TGT_ROW_REF, 50.0),
                                  (3, 4, 10, 0, oracle.INJ_ADD, oracle.TGT_COL_REF, -500.0)])
    assert r.counts["uncorrectable"] == 1 and np.array_equal(r.C, exact)


def test_detect_level_locates_without_correcting(oracle_lib):
    A, B = ints(51, 16, 40), ints(52, 40, 16)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16, ft_level=oracle.FT_DETECT,
                      injections=[(2, 3, 0, 0, oracle.INJ_ADD, 0, 9.0)])
    assert r.counts["located"] == 1 and r.counts["corrected"] == 0
    exact[2, 3] += 9
    assert np.array_equal(r.C.astype(np.float64), exact)


def test_detect_rows_level_offline(oracle_lib):
    """Offline detect-only ABFT (R15): row checks
    only.  Integer inputs make every residual exact: an accumulator fault flags
    exactly its row (event DETECTED, C left as computed, i.e. exact + delta); a
    row-reference fault flags its row too (a false alarm costs a recompute);
    a column-reference fault is invisible; clean tiles are only counted."""
    A, B = ints(55, 32, 40), ints(56, 40, 32)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)
    lvl = oracle.FT_DETECT_ROWS
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16, ft_level=lvl,
                      injections=[(18, 5, 7, 0, oracle.INJ_ADD, 0, 6.0)])
    assert r.counts["tiles_checked"] == 4 and r.counts["tiles_detected"] == 1
    assert r.counts["corrected"] == r.counts["located"] == r.counts["uncorrectable"] == 0
    e = r.events[0]
    assert (e["kind"], e["row"], e["col"], e["n_rows"], e["n_cols"], e["tile_m"], e["tile_n"]) == \
        (oracle.EV_DETECTED, 18, -1, 1, 0, 1, 0)
    assert e["resid_row"] == 6.0
    want = exact.copy(); want[18, 5] += 6.0
    assert np.array_equal(r.C.astype(np.float64), want)
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16, ft_level=lvl,
                      injections=[(3, 4, 10, 0, oracle.INJ_ADD, oracle.TGT_ROW_REF, 50.0)])
    assert r.counts["tiles_detected"] == 1 and r.events[0]["row"] == 3
    assert np.array_equal(r.C.astype(np.float64), exact)
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16, ft_level=lvl,
                      injections=[(3, 4, 10, 0, oracle.INJ_ADD, oracle.TGT_COL_REF, 50.0)])
    assert r.counts["tiles_detected"] == 0 and r.counts["tiles_checked"] == 4
    # two faults in one tile: still one detection (the tile is recomputed anyway)
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16, ft_level=lvl,
                      injections=[(1, 2, 0, 0, oracle.INJ_ADD, 0, 3.0), (7, 9, 0, 0, oracle.INJ_ADD, 0, -4.0)])
    assert r.counts["tiles_detected"] == 1 and r.events[0]["n_rows"] == 2 and r.events[0]["row"] == 1


def test_online_interval_mode(oracle_lib):
    """Per-K_s online verification (PAPER.md:170-173 / :515, R17).
    Integer inputs keep every partial sum exact, so the outcome is decided by
    the algorithm alone: two faults on one row in different steps are both
    corrected (C exact) where the end-of-K check must give up (1 row, 2 columns
    -> uncorrectable); two faults in one step stay uncorrectable at that check
    and at every later one; a reference fault persists (checksum_only at each
    later check); every step is a check; ks >= K is the end-of-K check."""
    A, B = ints(61, 32, 96), ints(62, 96, 32)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)
    kw = dict(tile_m=16, tile_n=16, bk=8)
    two = [(3, 4, 5, 0, oracle.INJ_ADD, 0, 6.0), (3, 9, 70, 0, oracle.INJ_ADD, 0, -9.0)]    # steps 1 and 3 (ks=32)
    r = oracle.ftgemm(A, B, ks=32, injections=two, **kw)
    assert r.counts["corrected"] == 2 and r.counts["tiles_checked"] == 4 * 3
    assert sorted(e["k_checked"] for e in r.events) == [32, 96]
    assert np.array_equal(r.C.astype(np.float64), exact)
    r0 = oracle.ftgemm(A, B, injections=two, **kw)
    assert r0.counts["uncorrectable"] == 1 and r0.counts["corrected"] == 0 and r0.events[0]["k_checked"] == 96
    same = [(3, 4, 40, 0, oracle.INJ_ADD, 0, 6.0), (7, 9, 50, 0, oracle.INJ_ADD, 0, -9.0)]  # both in step 2
    r = oracle.ftgemm(A, B, ks=32, injections=same, **kw)
    assert r.counts["uncorrectable"] == 2 and [e["k_checked"] for e in r.events] == [64, 96]
    ref = [(18, 20, 10, 0, oracle.INJ_ADD, oracle.TGT_ROW_REF, 50.0)]
    r = oracle.ftgemm(A, B, ks=32, injections=ref, **kw)
    assert r.counts["checksum_only"] == 3 and np.array_equal(r.C.astype(np.float64), exact)
    for ks in (96, 200):
        a = oracle.ftgemm(A, B, ks=ks, injections=two[:1], **kw)
        b = oracle.ftgemm(A, B, injections=two[:1], **kw)
        assert a.counts == b.counts and np.array_equal(a.C, b.C)
    # rows first before the end of K (R20): a column-reference fault
    # leaves every row sum intact, so only the end-of-K check (rows and
    # columns) reports it; C exact
    cref = [(18, 20, 10, 0, oracle.INJ_ADD, oracle.TGT_COL_REF, 50.0)]
    r = oracle.ftgemm(A, B, ks=32, injections=cref, **kw)
    assert r.counts["checksum_only"] == 1 and [e["k_checked"] for e in r.events] == [96]
    assert r.events[0]["n_rows"] == 0 and r.events[0]["n_cols"] == 1 and r.events[0]["col"] == 20
    assert np.array_equal(r.C.astype(np.float64), exact)
    # ... and with a C fault in a later step of the same tile the column fault is
    # seen at that step's full check: two columns, one row -> uncorrectable
    both = cref + [(19, 21, 70, 0, oracle.INJ_ADD, 0, 7.0)]
    r = oracle.ftgemm(A, B, ks=32, injections=both, **kw)
    assert [e["k_checked"] for e in r.events] == [96] and r.events[0]["kind"] == oracle.EV_UNCORRECTABLE
    assert r.events[0]["n_rows"] == 1 and r.events[0]["n_cols"] == 2
    # ragged last step (K = 96 = 40 + 40 + 16) and a fault in it
    r = oracle.ftgemm(A, B, ks=40, injections=[(30, 31, 90, 0, oracle.INJ_ADD, 0, 3.0)], **kw)
    assert r.counts["tiles_checked"] == 12 and r.events[0]["k_checked"] == 96 and r.counts["corrected"] == 1


def test_online_interval_no_false_positives(oracle_lib):
    """Fault-free signed data checked after every step of 64: every partial
    check stays below tau with margin (the threshold of R17 scales with the
    partial reference and sqrt(k))."""
    A = synth.matrix(71, 128, 1024)
    B = synth.matrix(72, 1024, 128)
    r = oracle.ftgemm(A, B, tile_m=64, tile_n=64, bk=64, ks=64, u_acc=2.0 ** -23, lambda1=8.0, lambda2=16.0)
    assert r.counts["tiles_checked"] == 4 * 16 and r.counts["tiles_detected"] == 0


def test_cost_model_online_vs_offline():
    """gamma = 1-(1-gamma0)^tiles, offline expected executions
    (1-gamma)/(1-2gamma).  Pinned by (a) the survey's evaluation for gamma0 = 1/256
    and 64 tiles (1024^2 in 128x128 tiles, SURVEY 8c / SPEC:491), (b) the
    independent Monte-Carlo branching process of reading R16, (c) the domain."""
    from oracle import cost_model as cm
    assert cm.tiles_of(1024, 1024, 128, 128) == 64
    g = cm.gamma(1 / 256, 64)
    assert abs(g - 0.221580) < 5e-7 and abs(cm.offline_expected_runs(g) - 1.397925) < 5e-7
    assert cm.gamma(0.0, 1000) == 0.0 and cm.offline_expected_runs(0.0) == 1.0
    assert cm.online_expected_runs(g) == 1.0
    assert cm.simulate_offline(0.0, 1000) == 1.0
    for gg, trials, tol in ((0.2, 20000, 0.05), (0.4, 20000, 0.05), (g, 20000, 0.05)):
        mc = cm.simulate_offline(gg, trials, seed=7)
        assert abs(mc - cm.offline_expected_runs(gg)) <= tol * cm.offline_expected_runs(gg), (gg, mc)
    with pytest.raises(ValueError):
        cm.offline_expected_runs(0.5)
    with pytest.raises(ValueError):
        cm.gamma(1.0, 4)


def test_ft_off_no_checking(oracle_lib):
    A, B = ints(53, 16, 40), ints(54, 40, 16)
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16, ft_level=oracle.FT_OFF,
                      injections=[(2, 3, 0, 0, oracle.INJ_ADD, 0, 9.0)])
    assert r.counts["tiles_checked"] == 0 and r.counts["events"] == 0


# -------------------------------------------------------------- threshold ---

@pytest.mark.parametrize("dist", ["signed", "unit"])
def test_threshold_no_false_positives_fp32seq(oracle_lib, dist):
    """Fault-free FP32 (paper numerics) tiles never trip the threshold, with a
    margin: max |residual| / tau stays below 1/4 (reading R1)."""
    M, N, K = 256, 256, 1024
    A, B, _ = synth.problem(M, N, K, dist=dist, seed=1234, with_c=False)
    r = oracle.ftgemm(A, B, acc="fp32seq", tile_m=32, tile_n=32, ft_level=oracle.FT_DETECT)
    assert r.counts["tiles_detected"] == 0
    ratio = max(np.nanmax(np.abs(r.resid_row) / r.tau_row), np.nanmax(np.abs(r.resid_col) / r.tau_col))
    assert ratio < 0.25, ratio


def test_threshold_scales_with_K_and_norms(oracle_lib):
    """tau is a number that grows with sqrt(K)|R| and with the operand norms."""
    A, B, _ = synth.problem(64, 64, 256, seed=5, with_c=False)
    r1 = oracle.ftgemm(A, B, tile_m=64, tile_n=64, ft_level=oracle.FT_DETECT)
    r2 = oracle.ftgemm(2 * A, B, tile_m=64, tile_n=64, ft_level=oracle.FT_DETECT)
    assert np.allclose(r2.tau_row, 2 * r1.tau_row) and np.allclose(r2.tau_col, 2 * r1.tau_col)
    A4 = np.concatenate([A, A, A, A], axis=1)
    B4 = np.concatenate([B, B, B, B], axis=0)
    r4 = oracle.ftgemm(A4, B4, tile_m=64, tile_n=64, ft_level=oracle.FT_DETECT)
    # K x4: |R| x4 and sqrt(K) x2 in the l1 term; norms x2 each in the l2 term
    t1 = oracle.ftgemm(A, B, tile_m=64, tile_n=64, ft_level=oracle.FT_DETECT, lambda2=0.0)
    t4 = oracle.ftgemm(A4, B4, tile_m=64, tile_n=64, ft_level=oracle.FT_DETECT, lambda2=0.0)
    assert np.allclose(t4.tau_row, 8 * t1.tau_row)
    assert np.all(r4.tau_row > r1.tau_row)


def test_detectable_flips_are_corrected(oracle_lib):
    """Sites whose flip moves the partial by >= 4 tau are always detected and
    corrected (SURVEY 8(c) generator); benign flips (<= tau/4) never are."""
    from oracle.sites import classify_bits
    M, N, K = 128, 128, 512
    A, B, _ = synth.problem(M, N, K, seed=77, with_c=False)
    kw = dict(tile_m=64, tile_n=64, bk=8, u_acc=2.0 ** -24, lambda1=16.0, lambda2=32.0)
    clean = oracle.ftgemm(A, B, acc="fp32seq", ft_level=oracle.FT_OFF, **kw)
    sites = synth.injection_sites(4, M, N, K, 64, 64, 8, seed=4242)
    for (row, col, k) in sites:
        det, ben, x, tau = classify_bits(A, B, row, col, k, **kw)
        assert det, (row, col, k)
        for b in (det[0], det[-1]):
            r = oracle.ftgemm(A, B, acc="fp32seq", injections=[(row, col, k, b, 0, 0, 0.0)], **kw)
            assert r.counts["corrected"] == 1, (row, col, k, b)
            assert r.events[0]["row"] == row and r.events[0]["col"] == col
            assert abs(r.C[row, col] - clean.C[row, col]) <= 4 * max(tau)
        if ben:
            r = oracle.ftgemm(A, B, acc="fp32seq", injections=[(row, col, k, ben[-1], 0, 0, 0.0)], **kw)
            assert r.counts["tiles_detected"] == 0


# ------------------------------------------------------ tile independence ---

def test_tile_local_subproblem(oracle_lib):
    """Running the oracle on one tile's sub-block reproduces that tile of the
    full run (basis of the tile-sampled oracle for the big configs)."""
    M, N, K = 96, 80, 64
    A, B, Cin = synth.problem(M, N, K, seed=3)
    inj = [(40, 50, 20, 30, 0, 0, 0.0)]
    full = oracle.ftgemm(A, B, Cin, alpha=1.5, beta=-0.5, tile_m=32, tile_n=32, injections=inj)
    sub = oracle.ftgemm(A[32:64], B[:, 32:64], Cin[32:64, 32:64], alpha=1.5, beta=-0.5,
                        tile_m=32, tile_n=32, injections=[(8, 18, 20, 30, 0, 0, 0.0)])
    assert np.array_equal(sub.C, full.C[32:64, 32:64])
    assert sub.counts["corrected"] == 1 and full.counts["corrected"] == 1


def test_ragged_tiles(oracle_lib):
    """Edge tiles (M, N not multiples of the tile) participate with only their
    valid rows / columns (reading R9)."""
    A, B = ints(61, 37, 29), ints(62, 29, 45)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float32)
    inj = [(36, 44, 28, 0, oracle.INJ_ADD, 0, 11.0)]      # last row, last col, last k
    r = oracle.ftgemm(A, B, tile_m=16, tile_n=16, injections=inj)
    assert r.counts["corrected"] == 1 and np.array_equal(r.C, exact)
    assert r.counts["tiles_checked"] == 3 * 3


# -------------------------------------------------------------- rounding ---

def test_double_to_bf16_is_nearest_even(oracle_lib):
    """The oracle's FP64 -> BF16 output rounding is round-to-nearest-even,
    checked against exact rational distances to the neighbouring bf16 values."""
    rng = np.random.default_rng(0)
    vals = list(rng.standard_normal(300) * 10.0 ** rng.integers(-30, 30, 300))
    vals += [1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 1.0 + 2 ** -9, -(1.0 + 2 ** -8), 3.3961e38, 1e-40, 0.0]
    for d in vals:
        h = oracle.double_to_bf16(d)
        v = float(synth.bf16_bits_to_f32(np.array([h], np.uint16))[0])
        if math.isinf(v):
            assert abs(d) >= 3.3895313892515355e38
            continue
        for nb in (h - 1, h + 1):
            w = float(synth.bf16_bits_to_f32(np.array([nb & 0xFFFF], np.uint16))[0])
            if not math.isfinite(w) or math.copysign(1, w) != math.copysign(1, v):
                continue
            dv, dw = abs(Fraction(d) - Fraction(v)), abs(Fraction(d) - Fraction(w))
            assert dv < dw or (dv == dw and (h & 1) == 0), (d, v, w)


def test_bf16_output_mode(oracle_lib):
    A, B, _ = synth.problem(32, 32, 64, dtype="bf16", seed=9, with_c=False)
    r = oracle.ftgemm(A, B, out="bf16", tile_m=32, tile_n=32)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.all(np.abs(r.C - ref) <= np.abs(ref) * 2 ** -8 + 1e-30)
