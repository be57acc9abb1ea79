"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bars (north_star): detected / corrected positions and
counts bit-exact; C within a relative Frobenius tolerance of 1e-6 (FP32 SIMT),
5e-3 (TF32), 2e-2 (BF16); bit-exact where the arithmetic is exact (integer
inputs; the SIMT kernel against the oracle's sequential-fmaf mode)."""
import contextlib
import math

import numpy as np
import pytest

import oracle
import synth
from gpu_util import TOL, Case, detectable_sites, elementwise_ratio, frob, odt, oracle_operand, uncorrectable_mask


def simt_tol(K: int) -> float:
    """FP32 SIMT relative Frobenius bound (R14): the north_star 1e-6
    for K <= 2048; beyond, max(1e-6, 2 u sqrt(K)) with clean elements bit-exact
    against the oracle's FP32SEQ mode (test_cfg2_full_size_sampled)."""
    return 1e-6 if K <= 2048 else max(1e-6, 2 * 2 ** -24 * math.sqrt(K))

pytestmark = pytest.mark.gpu

DTYPES = ["f32_simt", "tf32", "bf16"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2305_01024_b200 import ftgemm as F
    F.lib()
    oracle.build()


def ftmod():
    from paper_2305_01024_b200 import ftgemm as F
    return F


# ------------------------------------------------------- operand semantics ---

def test_tf32_operand_semantics():
    """kind::tf32 ignores the low 13 mantissa bits of FP32 operands (truncation);
    the encode relies on it (reading R8)."""
    import torch
    F = ftmod()
    A = np.zeros((128, 32), np.float32)
    B = np.zeros((32, 128), np.float32)
    A[0, 0] = 1 + 2 ** -11 + 2 ** -12
    B[0, 0] = 1.0
    Cd = torch.zeros(128, 128, device="cuda")
    F.run("tf32", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), Cd, ft_level=F.FT_OFF)
    torch.cuda.synchronize()
    assert Cd[0, 0].item() == 1.0


# ------------------------------------------------------------ clean parity ---

SHAPES = [
    (256, 256, 256, None, None, None),        # cfg1 shape
    (300, 520, 200, None, None, None),        # ragged M, N
    (1000, 1112, 704, None, None, None),      # several tiles + ragged tail
    (257, 301, 333, 336, 304, 304),           # ragged everything, padded leading dims
    (4096, 4096, 256, None, None, None),      # 128 x 256 tensor-core instantiation
]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s[:3])))
def test_clean_parity(dtype, shape):
    M, N, K, lda, ldb, ldc = shape
    c = Case(dtype, M, N, K, lda=lda, ldb=ldb, ldc=ldc, alpha=1.5, beta=-0.5)
    tol = TOL[dtype] if dtype != "f32_simt" else simt_tol(K)
    assert c.fro() < tol, c.fro()
    assert c.elementwise() <= 1.0
    assert c.counts["tiles_checked"] == c.plan.tiles_m * c.plan.tiles_n
    assert c.counts["tiles_detected"] == 0 and c.counts_match() and c.events_match()


@pytest.mark.parametrize("dtype", DTYPES)
def test_integer_inputs_bit_exact(dtype):
    """|values| <= 4, K <= 1024: every product, sum and checksum is exact in all
    three precisions, so C equals the oracle bit for bit."""
    c = Case(dtype, 384, 520, 512, dist="int", alpha=2.0, beta=-1.0)
    assert np.array_equal(c.C, c.ref.C)
    assert c.counts["tiles_detected"] == 0


def test_simt_bit_exact_vs_sequential_fma():
    """FP32 SIMT = the paper's SGEMM numerics: clean C bit-identical to the
    oracle's FP32SEQ mode (one fmaf per k, ascending k; fmaf(alpha, acc, beta c))."""
    for dist in ("signed", "unit"):
        c = Case("f32_simt", 300, 260, 1000, dist=dist, alpha=1.5, beta=-0.5, acc="fp32seq")
        assert np.array_equal(c.C, c.ref.C)


@pytest.mark.parametrize("dtype", DTYPES)
def test_ft_off_matches_ft_on_clean(dtype):
    """No-fault transparency: FT on (no faults) leaves C as FT off computes it."""
    F = ftmod()
    on = Case(dtype, 640, 760, 512, run_oracle=False)
    off = Case(dtype, 640, 760, 512, ft=F.FT_OFF, run_oracle=False)
    assert np.array_equal(on.C.view(np.uint32), off.C.view(np.uint32))


def test_determinism():
    a = Case("bf16", 700, 904, 1024, injections=[(10, 20, 300, 30, 0, 0, 0.0)], run_oracle=False)
    b = Case("bf16", 700, 904, 1024, injections=[(10, 20, 300, 30, 0, 0, 0.0)], run_oracle=False)
    assert np.array_equal(a.C, b.C) and a.events == b.events


# ------------------------------------------------------------ fault parity ---

@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("dist", ["signed", "unit"])
def test_injected_single_faults_parity(dtype, dist):
    """One detectable flip in several tiles: every fault is located at the same
    position, classified the same and corrected, as in the oracle."""
    M, N, K = 640, 760, 768
    A, B, _ = synth.problem(M, N, K, dist=dist, dtype=odt(dtype))
    F = ftmod()
    plan = F.plan(dtype, M, N, K)
    inj = detectable_sites(dtype, 6, M, N, K, plan, A, B, seed=11)
    assert len(inj) >= 4
    c = Case(dtype, M, N, K, dist=dist, injections=inj, alpha=1.0, beta=0.0)
    assert c.counts["corrected"] == len(inj), (c.counts, c.ref.counts)
    assert c.events_match() and c.counts_match()
    assert c.fro() < (TOL[dtype] if dtype != "f32_simt" else simt_tol(K))
    assert c.elementwise() <= 1.0


@pytest.mark.parametrize("dtype", DTYPES)
def test_cfg1_one_flip(dtype):
    """BASELINE cfg1 shape: 256^3, one bit flip at a seeded site (bit chosen per
    site by the oracle's generator), alpha 1.5, beta -0.5."""
    M = N = K = 256
    for dist in ("signed", "unit"):
        A, B, _ = synth.problem(M, N, K, dist=dist, dtype=odt(dtype))
        plan = ftmod().plan(dtype, M, N, K)
        inj = detectable_sites(dtype, 1, M, N, K, plan, A, B, seed=230501024 + 3)
        c = Case(dtype, M, N, K, dist=dist, injections=inj, alpha=1.5, beta=-0.5)
        assert c.counts["corrected"] == 1 and c.events_match()
        assert c.fro() < (TOL[dtype] if dtype != "f32_simt" else 1e-6)
        assert c.elementwise() <= 1.0


@pytest.mark.parametrize("dtype", DTYPES)
def test_benign_flips_not_detected(dtype):
    M, N, K = 512, 512, 512
    A, B, _ = synth.problem(M, N, K, dtype=odt(dtype))
    plan = ftmod().plan(dtype, M, N, K)
    inj = detectable_sites(dtype, 4, M, N, K, plan, A, B, seed=5, benign=True)
    assert inj
    c = Case(dtype, M, N, K, injections=inj)
    assert c.counts["tiles_detected"] == 0 and c.ref.counts["tiles_detected"] == 0
    assert c.fro() < (TOL[dtype] if dtype != "f32_simt" else 1e-6)


@pytest.mark.parametrize("dtype", DTYPES)
def test_add_mode_and_nonfinite(dtype):
    """ADD faults of +-1e3 and a flip to Inf/NaN (bit 30 of a partial >= 2 makes
    it infinite) are located and reconstructed from the row checksum."""
    M, N, K = 400, 400, 256
    inj = [(5, 7, 40, 0, oracle.INJ_ADD, 0, 1000.0), (260, 300, 200, 0, oracle.INJ_ADD, 0, -1000.0),
           (130, 3, 255, 0, oracle.INJ_ADD, 0, float("inf"))]
    c = Case(dtype, M, N, K, dist="unit", injections=inj)
    assert c.counts["corrected"] == 3 and c.events_match()
    assert np.all(np.isfinite(c.C))
    assert c.fro() < (TOL[dtype] if dtype != "f32_simt" else 1e-6)
    assert c.elementwise() <= 1.0


@pytest.mark.parametrize("dtype", DTYPES)
def test_seu_violation_and_checksum_faults(dtype):
    """Two faults in one tile -> uncorrectable (C left as computed); a fault in a
    carried reference -> checksum_only (C untouched); both as in the oracle."""
    F = ftmod()
    M, N, K = 400, 400, 256
    plan = F.plan(dtype, M, N, K)
    tm, tn = plan.check_tile_m, plan.check_tile_n
    inj = [(1, 2, 30, 0, oracle.INJ_ADD, 0, 500.0), (7, 9, 100, 0, oracle.INJ_ADD, 0, -700.0),    # tile (0,0)
           (tm + 3, 5, 64, 0, oracle.INJ_ADD, oracle.TGT_ROW_REF, 800.0),                            # tile (1,0)
           (7, tn + 4, 64, 0, oracle.INJ_ADD, oracle.TGT_COL_REF, 800.0)]                            # tile (0,1)
    c = Case(dtype, M, N, K, dist="unit", injections=inj)
    assert c.counts["uncorrectable"] == 1 and c.counts["checksum_only"] == 2
    assert c.events_match() and c.counts_match()
    bad = np.zeros((M, N), bool)
    bad[[1, 7], :] = True
    bad[:, [2, 9]] = True
    assert c.fro(~bad) < (TOL[dtype] if dtype != "f32_simt" else 1e-6)
    assert c.elementwise(skip=bad) <= 1.0
    assert abs(c.C[1, 2] - c.ref.C[1, 2]) <= 1e-2 * abs(c.ref.C[1, 2]) + 1.0


@pytest.mark.parametrize("dtype", DTYPES)
def test_detect_level(dtype):
    F = ftmod()
    inj = [(33, 44, 100, 0, oracle.INJ_ADD, 0, 250.0)]
    c = Case(dtype, 300, 304, 256, dist="unit", ft=F.FT_DETECT, injections=inj)
    assert c.counts["located"] == 1 and c.counts["corrected"] == 0 and c.events_match()
    assert abs(c.C[33, 44] - c.ref.C[33, 44]) <= 2e-2 * abs(c.ref.C[33, 44])


def test_stress_one_fault_per_tile():
    """One detectable flip in EVERY tile (BF16): all corrected at the oracle's positions."""
    M = N = 1024
    K = 512
    A, B, _ = synth.problem(M, N, K, dtype="bf16")
    plan = ftmod().plan("bf16", M, N, K)
    inj = detectable_sites("bf16", plan.tiles_m * plan.tiles_n, M, N, K, plan, A, B, seed=99)
    c = Case("bf16", M, N, K, injections=inj)
    assert c.counts["corrected"] == len(inj) and c.events_match() and c.fro() < TOL["bf16"]
    assert c.elementwise() <= 1.0


@pytest.mark.parametrize("dtype", ["tf32", "bf16"])
def test_false_positive_sweep(dtype):
    """Fault-free tiles never trip the threshold (SPEC.md:283 analogue)."""
    F = ftmod()
    for dist in ("signed", "unit"):
        c = Case(dtype, 2048, 2048, 2048, dist=dist, run_oracle=False)
        assert c.counts["tiles_detected"] == 0
        assert c.counts["tiles_checked"] == c.plan.tiles_m * c.plan.tiles_n


# ------------------------------------------------ in-kernel encode of A ----

@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("dtype", ["tf32", "bf16"])
@pytest.mark.parametrize("shape", [(845, 600, 1000), (1000, 10896, 2048)], ids=["bn128", "bn256"])
def test_fused_encode_parity(dtype, cg, shape):
    """ftgemm_run_fused: with only B encoded,
    the kernel derives e^T A, its split rows and the row / tile norms itself;
    events, counts and C as the oracle; C bit-identical to the separately
    encoded run except at corrected elements (same tiles, same k order)."""
    import torch
    F = ftmod()
    M, N, K = shape
    A, B, Cin = synth.problem(M, N, K, dtype=odt(dtype))
    plan = F.plan(dtype, M, N, K, tile=(F.plan(dtype, M, N, K).bn, cg))
    assert plan.cta_group == cg
    dtype_c = plan.dtype
    tm, tn = plan.check_tile_m, plan.check_tile_n
    inj = detectable_sites(dtype, 8, M, N, K, plan, A, B, seed=61)
    inj.append((plan.tiles_m * tm - tm + 2, 3, 40, 0, oracle.INJ_ADD, 0, 800.0))          # last (ragged) tile row
    Ad, Bd = synth.to_torch(A, odt(dtype)).cuda(), synth.to_torch(B, odt(dtype)).cuda()
    g = F.FTGemm(dtype_c, M, N, K)
    g.enc_ws.fill_(0xFF)                          # the A part must not be read
    g.encode(None, Bd, which=2)
    Cf = synth.to_torch(Cin, odt(dtype)).cuda()
    g.run(Ad, Bd, Cf, alpha=1.5, beta=-0.5, injections=inj, fuse_a=True)
    torch.cuda.synchronize()
    counts, events = g.report()
    ref = oracle.ftgemm(A, B, Cin, alpha=1.5, beta=-0.5, out=odt(dtype), tile_m=tm, tile_n=tn, bk=plan.bk,
                        u_acc=plan.u_acc, lambda1=plan.lambda1, lambda2=plan.lambda2, injections=inj)
    keys = ("tiles_checked", "tiles_detected", "corrected", "checksum_only", "uncorrectable", "located", "events")
    assert all(int(counts[k]) == int(ref.counts[k]) for k in keys), (counts, ref.counts)
    ek = lambda evs: sorted((e["tile_m"], e["tile_n"], e["kind"], e["row"], e["col"], e["n_rows"], e["n_cols"])
                            for e in evs)
    assert ek(events) == ek(ref.events)
    assert frob(Cf.float().cpu().numpy(), ref.C) < TOL[dtype]
    # against the separately encoded run: identical away from the corrected elements
    g2 = F.FTGemm(dtype_c, M, N, K)
    g2.encode(Ad, Bd)
    C2 = synth.to_torch(Cin, odt(dtype)).cuda()
    g2.run(Ad, Bd, C2, alpha=1.5, beta=-0.5, injections=inj)
    torch.cuda.synchronize()
    same = (Cf == C2)
    for e in events:
        same[e["row"], e["col"]] = True
    assert bool(same.all())
    # fault-free: no detections (threshold margins hold with the in-kernel norms)
    g.reset()
    g.run(Ad, Bd, Cf, injections=(), fuse_a=True)
    c0, _ = g.report()
    assert c0["tiles_detected"] == 0 and c0["tiles_checked"] == plan.tiles_m * plan.tiles_n


@pytest.mark.parametrize("level", ["detect", "detect_rows"])
def test_fused_encode_detect_levels(level):
    """The in-kernel A encode at the detect-only levels: the same counts,
    events and C as the separately encoded run (faults left in place)."""
    import torch
    F = ftmod()
    lv = {"detect": F.FT_DETECT, "detect_rows": F.FT_DETECT_ROWS}[level]
    M, N, K = 1000, 2016, 1536
    A, B, Cin = synth.problem(M, N, K, dtype="bf16")
    plan = F.plan("bf16", M, N, K)
    inj = detectable_sites("bf16", 6, M, N, K, plan, A, B, seed=83)
    Ad, Bd = synth.to_torch(A, "bf16").cuda(), synth.to_torch(B, "bf16").cuda()
    g1, g2 = F.FTGemm("bf16", M, N, K), F.FTGemm("bf16", M, N, K)
    g1.encode(Ad, Bd)
    g2.encode(None, Bd, which=2)
    C1, C2 = synth.to_torch(Cin, "bf16").cuda(), synth.to_torch(Cin, "bf16").cuda()
    g1.run(Ad, Bd, C1, ft_level=lv, injections=inj)
    g2.run(Ad, Bd, C2, ft_level=lv, injections=inj, fuse_a=True)
    torch.cuda.synchronize()
    (c1, e1), (c2, e2) = g1.report(), g2.report()
    keys = ("tiles_checked", "tiles_detected", "corrected", "checksum_only", "uncorrectable", "located", "events")
    assert all(int(c1[k]) == int(c2[k]) for k in keys), (c1, c2)
    ek = lambda evs: sorted((e["tile_m"], e["tile_n"], e["kind"], e["row"], e["col"]) for e in evs)
    assert ek(e1) == ek(e2) and int(c1["tiles_detected"]) == len(inj)
    assert bool(torch.equal(C1, C2))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_fused_encode_repeat_and_cuda_graph(dtype):
    """The in-kernel encode's item flags are cleared on every call (a memset
    captured with the kernel), so back-to-back calls with new A values, and a
    CUDA-graph replay after A changed in place, see only this call's items: C
    bit-identical to a separately encoded run of the same operands, no tile
    flagged, every tile checked."""
    import torch
    F = ftmod()
    M, N, K = 1000, 2016, 1536
    A1, B, _ = synth.problem(M, N, K, dtype=odt(dtype))
    A2 = synth.matrix(77, M, K, dtype=odt(dtype))
    Ad1, Ad2 = synth.to_torch(A1, odt(dtype)).cuda(), synth.to_torch(A2, odt(dtype)).cuda()
    Bd = synth.to_torch(B, odt(dtype)).cuda()
    g = F.FTGemm(dtype, M, N, K)
    g.encode(None, Bd, which=2)
    ref = F.FTGemm(dtype, M, N, K)

    def reference(Ad):
        Cr = torch.empty(M, N, dtype=Ad.dtype, device="cuda")
        ref.encode(Ad, Bd)
        ref.run(Ad, Bd, Cr)
        return Cr

    R1, R2 = reference(Ad1), reference(Ad2)
    C = torch.empty(M, N, dtype=Ad1.dtype, device="cuda")
    for Ad, R in ((Ad1, R1), (Ad2, R2), (Ad1, R1)):          # back to back, A changes every call
        g.run(Ad, Bd, C, fuse_a=True)
        torch.cuda.synchronize()
        assert bool(torch.equal(C, R))
    # CUDA graph: capture one fused call on A_buf, replay after refilling A_buf
    A_buf = Ad1.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.run(A_buf, Bd, C, fuse_a=True)                     # warm-up outside the capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        g.run(A_buf, Bd, C, fuse_a=True)
    for Ad, R in ((Ad2, R2), (Ad1, R1), (Ad2, R2)):
        A_buf.copy_(Ad)
        C.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert bool(torch.equal(C, R))
    counts, _ = g.report()
    tiles = g.plan.tiles_m * g.plan.tiles_n
    assert counts["tiles_detected"] == 0
    assert counts["tiles_checked"] == 7 * tiles       # 3 direct + warm-up + 3 replays


# ------------------------------------------- multi-GPU partition invariant --

@pytest.mark.parametrize("dtype,shape", [("bf16", (4000, 8192, 2048)), ("tf32", (2000, 3000, 1024)),
                                         ("f32_simt", (1000, 1024, 512))])
def test_partition_invariance(dtype, shape):
    """the M-block partition of paper_2305_01024_b200.distributed
    (whole check tiles per rank, B shared) gives, rank by rank, C and event
    positions bit-identical to the single-GPU run.  The ranks are run one
    after another on one GPU with the real kernels (the process-group plumbing
    is covered by tests/test_distributed.py on gloo)."""
    import torch
    F = ftmod()
    from paper_2305_01024_b200.distributed import row_partition
    M, N, K = shape
    A, B, Cin = synth.problem(M, N, K, dtype=odt(dtype))
    full_plan = F.plan(dtype, M, N, K)
    tm = full_plan.check_tile_m
    inj = detectable_sites(dtype, 6, M, N, K, full_plan, A, B, seed=51)
    Ad, Bd = synth.to_torch(A, odt(dtype)).cuda(), synth.to_torch(B, odt(dtype)).cuda()
    g = F.FTGemm(dtype, M, N, K)
    Cf = synth.to_torch(Cin, odt(dtype)).cuda()
    g.encode(Ad, Bd)
    g.run(Ad, Bd, Cf, alpha=1.0, beta=0.5, injections=inj)
    torch.cuda.synchronize()
    _, ev_full = g.report()
    key = lambda e: (e["tile_m"], e["tile_n"], e["kind"], e["row"], e["col"], e["n_rows"], e["n_cols"])
    for world in (2, 3):
        parts = row_partition(M, world, tm)
        Cp, evs = [], []
        for row0, rows in parts:
            # a rank runs the full problem's tile class (as distributed.PartitionedFTGemm
            # does: full_plan.dtype is the full plan's explicit dtype code)
            gp = F.FTGemm(full_plan.dtype, rows, N, K)
            assert (gp.plan.bn, gp.plan.cta_group, gp.plan.check_tile_m, gp.plan.check_tile_n) == \
                (full_plan.bn, full_plan.cta_group, full_plan.check_tile_m, full_plan.check_tile_n)
            mine = [(r - row0, c, k, b, m, tg, ad) for (r, c, k, b, m, tg, ad) in inj if row0 <= r < row0 + rows]
            Cd = synth.to_torch(Cin[row0:row0 + rows], odt(dtype)).cuda()
            Ar = Ad[row0:row0 + rows].contiguous()
            gp.encode(Ar, Bd)
            gp.run(Ar, Bd, Cd, alpha=1.0, beta=0.5, injections=mine)
            torch.cuda.synchronize()
            _, e = gp.report()
            for x in e:
                x = dict(x)
                x["row"] += row0 if x["row"] >= 0 else 0
                x["tile_m"] += row0 // tm
                evs.append(x)
            Cp.append(Cd)
        assert torch.equal(torch.cat(Cp), Cf), world
        assert sorted(map(key, evs)) == sorted(map(key, ev_full)), world


# ------------------------------------------------------- degenerate shapes --

DEGENERATE = [(1, 8, 8), (7, 16, 24), (130, 8, 16), (1, 4096, 8), (125, 248, 64), (2, 8, 4104), (251, 264, 72)]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", DEGENERATE, ids=lambda s: "x".join(map(str, s)))
def test_degenerate_shapes(dtype, shape):
    """The degenerate cases of the method: one row, one k-block or less (K = 8
    < BK), a single column block, K just past a k-block multiple, exactly one
    check tile, a tile row / column of one element past a check tile.  Clean
    run within the bounds and bit-for-bit the oracle's events; one large offset
    in the last element (last k) is corrected; FT off equals FT on."""
    F = ftmod()
    M, N, K = shape
    clean = Case(dtype, M, N, K, alpha=1.5, beta=-0.5)
    tol = TOL[dtype] if dtype != "f32_simt" else simt_tol(K)
    assert clean.fro() < tol and clean.elementwise() <= 1.0
    assert clean.counts["tiles_detected"] == 0 and clean.counts_match() and clean.events_match()
    inj = [(M - 1, N - 1, K - 1, 0, oracle.INJ_ADD, 0, 1.0e4)]
    c = Case(dtype, M, N, K, injections=inj)
    assert c.counts["corrected"] == 1 and c.counts_match() and c.events_match(), (c.counts, c.ref.counts)
    assert c.fro() < tol
    off = Case(dtype, M, N, K, ft=F.FT_OFF, alpha=1.5, beta=-0.5, run_oracle=False)
    import torch
    assert bool(torch.equal(off.C_raw, clean.C_raw))
    if dtype != "f32_simt":
        # the in-kernel A encode on the same degenerate shape: C bitwise as the
        # separately encoded run, nothing flagged, every tile checked
        g = F.FTGemm(dtype, M, N, K)
        Ad = synth.to_torch(clean.A, odt(dtype)).cuda()
        Bd = synth.to_torch(clean.B, odt(dtype)).cuda()
        Cf = synth.to_torch(clean.Cin, odt(dtype)).cuda()
        g.encode(None, Bd, which=2)
        g.run(Ad, Bd, Cf, alpha=1.5, beta=-0.5, fuse_a=True)
        torch.cuda.synchronize()
        cnt, _ = g.report()
        assert bool(torch.equal(Cf.cpu(), clean.C_raw))
        assert cnt["tiles_detected"] == 0 and cnt["tiles_checked"] == g.plan.tiles_m * g.plan.tiles_n


# ------------------------------------------------------- skinny shapes -----

@pytest.mark.parametrize("dtype", ["tf32", "bf16"])
@pytest.mark.parametrize("shape", [(250, 3000, 1024), (3000, 200, 1024), (128, 2600, 2048)],
                         ids=["m250", "n200", "m128"])
def test_skinny_shapes(dtype, shape):
    """cfg4-style skinny operands get one check tile across the narrow
    dimension (N <= 252: a single 252-column tile; M <= 250: a CTA pair per
    unit); faults in both CTAs of the pair / anywhere in the narrow tile."""
    F = ftmod()
    M, N, K = shape
    plan = F.plan(dtype, M, N, K)
    assert plan.bn == 256 and (plan.tiles_n == 1 if N <= 252 else plan.cta_group == 2)
    A, B, _ = synth.problem(M, N, K, dtype=odt(dtype))
    inj = detectable_sites(dtype, 6, M, N, K, plan, A, B, seed=41)
    c = Case(dtype, M, N, K, injections=inj, alpha=1.0, beta=0.5)
    assert c.counts_match() and c.events_match(), (c.counts, c.ref.counts)
    assert c.counts["corrected"] == len(inj) and c.fro() < TOL[dtype]
    off = Case(dtype, M, N, K, ft=F.FT_OFF, alpha=1.0, beta=0.5)
    assert off.fro() < TOL[dtype]


# ------------------------------------------ online verification every K_s ---

@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("dtype", ["tf32", "bf16"])
def test_online_interval_parity(dtype, cg):
    """ftgemm_run_online: the fused kernel verifies
    after every K_s step and corrects in TMEM.  Several faults per tile in
    different steps are all corrected; a double fault within one step is
    uncorrectable at that step and after; a row-reference fault is reported at
    every later check, a column-reference fault at the end of K only (the K_s
    checks are row-first, R20); events (with k_checked) and counts as
    in the oracle."""
    import torch
    F = ftmod()
    M, N, K = 845, 600, 1024
    A, B, Cin = synth.problem(M, N, K, dtype=odt(dtype))
    plan = F.plan(dtype, M, N, K, tile=(F.plan(dtype, M, N, K).bn, cg))
    tm, tn = plan.check_tile_m, plan.check_tile_n
    ks = 256
    inj = [(5, 7, 40, 0, oracle.INJ_ADD, 0, 1000.0), (5, 90, 300, 0, oracle.INJ_ADD, 0, -800.0),      # tile (0,0)
           (60, 7, 700, 0, oracle.INJ_ADD, 0, 900.0), (6, 7, 1000, 0, oracle.INJ_ADD, 0, 1200.0),
           (tm + 3, tn + 4, 100, 30, oracle.INJ_FLIP, 0, 0.0), (tm + 3, tn + 40, 600, 0, oracle.INJ_ADD, 0, 500.0),
           (3 * tm + 1, 2, 520, 0, oracle.INJ_ADD, 0, 700.0), (3 * tm + 8, 9, 600, 0, oracle.INJ_ADD, 0, -700.0),  # same step
           (4 * tm + 2, tn + 1, 300, 0, oracle.INJ_ADD, oracle.TGT_ROW_REF, 600.0),
           (6 * tm + 1, 3, 10, 0, oracle.INJ_ADD, 0, 900.0), (6 * tm + 2, 4, 900, 0, oracle.INJ_ADD, 0, 900.0),
           # column-reference fault: the K_s checks look at the rows first (R20),
           # so only the end-of-K check reports it
           (2 * tm + 5, 2 * tn + 3, 300, 0, oracle.INJ_ADD, oracle.TGT_COL_REF, -700.0)]
    g = F.FTGemm(plan.dtype, M, N, K)
    assert g.plan.cta_group == cg
    Ad, Bd = synth.to_torch(A, odt(dtype)).cuda(), synth.to_torch(B, odt(dtype)).cuda()
    Cd = synth.to_torch(Cin, odt(dtype)).cuda()
    g.encode(Ad, Bd)
    g.run_online(Ad, Bd, Cd, ks=ks, alpha=1.5, beta=-0.5, injections=inj)
    torch.cuda.synchronize()
    counts, events = g.report()
    ref = oracle.ftgemm(A, B, Cin, alpha=1.5, beta=-0.5, out=odt(dtype), tile_m=tm, tile_n=tn, bk=plan.bk,
                        u_acc=plan.u_acc, lambda1=plan.lambda1, lambda2=plan.lambda2, injections=inj, ks=ks)
    keys = ("tiles_checked", "tiles_detected", "corrected", "checksum_only", "uncorrectable", "located", "events")
    assert all(int(counts[k]) == int(ref.counts[k]) for k in keys), (counts, ref.counts)
    ek = lambda evs: sorted((e["tile_m"], e["tile_n"], e["kind"], e["row"], e["col"], e["n_rows"], e["n_cols"],
                             e["k_checked"]) for e in evs)
    assert ek(events) == ek(ref.events)
    assert counts["corrected"] >= 7 and counts["tiles_checked"] == plan.tiles_m * plan.tiles_n * 4
    bad = np.zeros((M, N), bool)
    for e in ref.events:
        if e["kind"] == oracle.EV_UNCORRECTABLE:
            bad[e["tile_m"] * tm:(e["tile_m"] + 1) * tm, e["tile_n"] * tn:(e["tile_n"] + 1) * tn] = True
    assert frob(Cd.float().cpu().numpy(), ref.C, ~bad) < TOL[dtype]
    # a step >= K is the end-of-K check; DETECT_ROWS / SIMT are refused
    g.reset()
    g.run_online(Ad, Bd, Cd, ks=((K + plan.bk - 1) // plan.bk) * plan.bk, injections=inj[:1])
    c2, _ = g.report()
    assert c2["corrected"] == 1 and c2["tiles_checked"] == plan.tiles_m * plan.tiles_n
    with pytest.raises(F.FtgemmError):
        g.run_online(Ad, Bd, Cd, ks=plan.bk + 1)


# ------------------------------------------------ non-fused baseline -------

@pytest.mark.parametrize("dtype", ["f32_simt", "bf16"])
def test_nonfused_parity(dtype):
    """The non-fused baseline (cuBLAS GEMMs + verification kernel) computes the
    same function: clean C within tolerance, faults striking the final
    accumulator (k_elem = K-1 in the oracle) located / corrected / classified
    exactly as the oracle does, FT_OFF = the plain library GEMM."""
    import torch
    F = ftmod()
    M, N, K = 700, 904, 640
    A, B, Cin = synth.problem(M, N, K, dtype=odt(dtype))
    plan = F.plan(dtype, M, N, K)
    tm, tn = plan.check_tile_m, plan.check_tile_n
    inj = [(5, 7, K - 1, 0, oracle.INJ_ADD, 0, 1000.0), (tm + 3, tn + 4, K - 1, 0, oracle.INJ_ADD, 0, -700.0),
           (2 * tm + 10, 2 * tn + 3, K - 1, 30, oracle.INJ_FLIP, 0, 0.0),
           (3 * tm + 1, 5, K - 1, 0, oracle.INJ_ADD, oracle.TGT_ROW_REF, 800.0),
           (4 * tm + 2, tn + 9, K - 1, 0, oracle.INJ_ADD, oracle.TGT_COL_REF, -800.0),
           (5 * tm + 1, 3, K - 1, 0, oracle.INJ_ADD, 0, 900.0), (5 * tm + 6, 20, K - 1, 0, oracle.INJ_ADD, 0, 900.0)]
    kw = dict(out=odt(dtype), tile_m=tm, tile_n=tn, bk=plan.bk, u_acc=plan.u_acc, lambda1=plan.lambda1,
              lambda2=plan.lambda2)
    g = F.FTGemm(dtype, M, N, K)
    Ad, Bd = synth.to_torch(A, odt(dtype)).cuda(), synth.to_torch(B, odt(dtype)).cuda()
    g.encode(Ad, Bd, which=3 | 4)
    tol = TOL[dtype] if dtype != "f32_simt" else max(1e-6, 2 * 2 ** -24 * math.sqrt(K))
    for level, faults in ((F.FT_CORRECT, []), (F.FT_CORRECT, inj), (F.FT_DETECT_ROWS, inj), (F.FT_OFF, [])):
        Cd = synth.to_torch(Cin, odt(dtype)).cuda()
        g.reset()
        g.run_nonfused(Ad, Bd, Cd, alpha=1.5, beta=-0.5, ft_level=level, injections=faults)
        torch.cuda.synchronize()
        Cg = Cd.float().cpu().numpy()
        ref = oracle.ftgemm(A, B, Cin, alpha=1.5, beta=-0.5, ft_level=level, injections=faults, **kw)
        bad = np.zeros((M, N), bool)
        if level != F.FT_OFF:
            counts, events = g.report()
            keys = ("tiles_checked", "tiles_detected", "corrected", "checksum_only", "uncorrectable", "located")
            assert all(int(counts[k]) == int(ref.counts[k]) for k in keys), (level, counts, ref.counts)
            ek = lambda evs: sorted((e["tile_m"], e["tile_n"], e["kind"], e["row"], e["col"], e["n_rows"], e["n_cols"])
                                    for e in evs)
            assert ek(events) == ek(ref.events), level
            for e in ref.events:
                if e["kind"] in (oracle.EV_UNCORRECTABLE, oracle.EV_DETECTED):
                    bad[e["tile_m"] * tm:(e["tile_m"] + 1) * tm, e["tile_n"] * tn:(e["tile_n"] + 1) * tn] = True
        assert frob(Cg, ref.C, ~bad) < tol, level


# ------------------------------------------- offline (detect-only) ABFT ----

@pytest.mark.parametrize("dtype", DTYPES)
def test_detect_rows_parity(dtype):
    """FT_DETECT_ROWS: the same tiles flagged at the same
    first row with the same row counts as the oracle; column-reference faults
    are invisible, row-reference faults flag their row; C is left as computed."""
    F = ftmod()
    M, N, K = 640, 760, 512
    A, B, _ = synth.problem(M, N, K, dtype=odt(dtype))
    plan = F.plan(dtype, M, N, K)
    tm, tn = plan.check_tile_m, plan.check_tile_n
    inj = detectable_sites(dtype, 5, M, N, K, plan, A, B, seed=31)
    used = {(r // tm, c // tn) for r, c, *_ in inj}
    extra = [(4 * tm + 3, 2 * tn + 1, 100, 0, oracle.INJ_ADD, oracle.TGT_COL_REF, 700.0),
             (4 * tm + 5, 1, 100, 0, oracle.INJ_ADD, oracle.TGT_ROW_REF, 700.0),
             (2 * tm + 1, tn + 2, 10, 0, oracle.INJ_ADD, 0, 900.0), (2 * tm + 9, tn + 7, 300, 0, oracle.INJ_ADD, 0, -900.0)]
    inj += [f for f in extra if (f[0] // tm, f[1] // tn) not in used]
    c = Case(dtype, M, N, K, injections=inj, ft=F.FT_DETECT_ROWS)
    assert c.counts_match() and c.events_match(), (c.counts, c.ref.counts)
    assert all(e["kind"] == F.EV_DETECTED and e["col"] == -1 for e in c.events)
    assert c.counts["tiles_checked"] == plan.tiles_m * plan.tiles_n
    bad = np.zeros((M, N), bool)
    for r, col, _, _, _, tgt, _ in inj:
        if tgt == 0:
            bad[r, col] = True
    assert c.fro(~bad) < (TOL[dtype] if dtype != "f32_simt" else 1e-6)
    assert c.elementwise(skip=bad) <= 1.0


@pytest.mark.parametrize("dtype", DTYPES)
def test_run_offline_recompute(dtype):
    """Offline ABFT: detect, then re-compute the product; the
    final C equals the fault-free product; beta != 0 restores C_in from the
    backup; faults striking the re-computation trigger further executions."""
    import torch
    F = ftmod()
    M, N, K = 512, 520, 384
    A, B, Cin = synth.problem(M, N, K, dtype=odt(dtype))
    plan = F.plan(dtype, M, N, K)
    tm, tn = plan.check_tile_m, plan.check_tile_n
    ref = oracle.ftgemm(A, B, Cin, alpha=1.5, beta=-0.5, out=odt(dtype), tile_m=tm, tile_n=tn, bk=plan.bk,
                        u_acc=plan.u_acc, lambda1=plan.lambda1, lambda2=plan.lambda2, ft_level=oracle.FT_OFF)
    g = F.FTGemm(dtype, M, N, K)
    Ad, Bd = synth.to_torch(A, odt(dtype)).cuda(), synth.to_torch(B, odt(dtype)).cuda()
    g.encode(Ad, Bd)
    faults = [(5, 7, 40, 0, oracle.INJ_ADD, 0, 1000.0), (tm + 3, tn + 4, 200, 0, oracle.INJ_ADD, 0, -1000.0),
              (3 * tm + 1, 2 * tn + 9, 300, 0, oracle.INJ_ADD, 0, 5000.0)]
    tol = TOL[dtype] if dtype != "f32_simt" else 1e-6

    def go(inj_run, max_runs, beta=-0.5):
        Cd = synth.to_torch(Cin, odt(dtype)).cuda()
        g.reset()
        runs, clean = g.run_offline(Ad, Bd, Cd, alpha=1.5, beta=beta, injections=faults, inj_run=inj_run,
                                    max_runs=max_runs)
        torch.cuda.synchronize()
        counts, events = g.report()
        return runs, clean, counts, events, Cd.float().cpu().numpy()

    runs, clean, counts, events, Cg = go([0, 0, 0], 4)
    assert (runs, clean) == (2, True) and counts["tiles_detected"] == 3
    assert sorted((e["tile_m"], e["tile_n"]) for e in events) == [(0, 0), (1, 1), (3, 2)]
    assert np.linalg.norm(Cg - ref.C) / np.linalg.norm(ref.C) < tol
    runs, clean, counts, _, Cg = go([0, 1, 1], 4)
    assert (runs, clean) == (3, True) and counts["tiles_detected"] == 3
    assert np.linalg.norm(Cg - ref.C) / np.linalg.norm(ref.C) < tol
    runs, clean, counts, _, _ = go([0, 1, 1], 2)
    assert (runs, clean) == (2, False)
    runs, clean, counts, _, _ = go([0, 0, 0], 4, beta=0.0)
    assert (runs, clean) == (2, True) and counts["tiles_checked"] == 2 * plan.tiles_m * plan.tiles_n


# ----------------------------------------------------- CTA pairs (2-SM MMA) --

@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("dtype", ["tf32", "bf16"])
@pytest.mark.parametrize("shape", [(845, 600, 320), (845, 10896, 256)], ids=["bn128", "bn256"])
def test_cta_pair_modes(dtype, cg, shape):
    """Both tensor-core launch modes (one CTA per MMA, or a cta_group::2 pair with
    M = 256) give the oracle's C, events and counts.  7 check-tile rows: the last
    pair's second tile lies beyond M.  Faults in both CTAs of a pair (even and
    odd tile rows), in the carried references, and an SEU violation."""
    F = ftmod()
    M, N, K = shape
    A, B, _ = synth.problem(M, N, K, dtype=odt(dtype))
    tile = (F.plan(dtype, M, N, K).bn, cg)
    plan = F.plan(dtype, M, N, K, tile=tile)
    assert plan.cta_group == cg and plan.tiles_m == 7
    tm, tn = plan.check_tile_m, plan.check_tile_n
    inj = detectable_sites(dtype, 8, M, N, K, plan, A, B, seed=21)
    used = {(r // tm, c // tn) for r, c, *_ in inj}
    extra = [(3 * tm + 5, 2, 64, 0, oracle.INJ_ADD, oracle.TGT_ROW_REF, 600.0),          # odd tile row
             (5 * tm + 9, tn + 7, 100, 0, oracle.INJ_ADD, oracle.TGT_COL_REF, -600.0),    # odd tile row
             (6 * tm + 1, 4, 10, 0, oracle.INJ_ADD, 0, 900.0),                            # last (unpaired) row
             (6 * tm + 2, 8, 200, 0, oracle.INJ_ADD, 0, -900.0)]                          # ... twice: SEU violation
    inj += [f for f in extra if (f[0] // tm, f[1] // tn) not in used]
    c = Case(dtype, M, N, K, injections=inj, alpha=1.25, beta=0.5, tile=tile)
    assert c.counts_match() and c.events_match(), (c.counts, c.ref.counts)
    assert c.counts["tiles_checked"] == plan.tiles_m * plan.tiles_n
    bad = np.zeros((M, N), bool)
    for e in c.ref.events:
        if e["kind"] == oracle.EV_UNCORRECTABLE:
            bad[e["tile_m"] * tm:(e["tile_m"] + 1) * tm, e["tile_n"] * tn:(e["tile_n"] + 1) * tn] = True
    assert c.fro(~bad) < TOL[dtype]
    off = Case(dtype, M, N, K, ft=F.FT_OFF, alpha=1.25, beta=0.5, tile=tile)
    assert off.fro() < TOL[dtype]


# ------------------------------------------------- full size, sampled oracle --

def test_cfg3_full_size_sampled():
    """BF16 8192^3 in the bench's launch configuration (same plan, same kernel),
    with faults in 4 tiles; the oracle checks whole sampled tiles (tile-local
    sub-problems, see tests/test_oracle.py::test_tile_local_subproblem)."""
    import torch
    F = ftmod()
    M = N = K = 8192
    plan = F.plan("bf16", M, N, K)
    tm, tn = plan.check_tile_m, plan.check_tile_n
    seedA, seedB = synth.BASE_SEED + synth.SEED_A, synth.BASE_SEED + synth.SEED_B
    A = synth.to_torch(synth.matrix(seedA, M, K, dtype="bf16"), "bf16").cuda()
    B = synth.to_torch(synth.matrix(seedB, K, N, dtype="bf16"), "bf16").cuda()
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    tiles = [(0, 0), (17, 5), (40, 32), (plan.tiles_m - 1, plan.tiles_n - 1), (33, 20), (64, 1)]
    inj = [(ti * tm + 7, tj * tn + 11, 4000, 30, oracle.INJ_FLIP, 0, 0.0) for ti, tj in tiles[:4]]
    g = F.FTGemm("bf16", M, N, K)
    g.encode(A, B)
    g.run(A, B, C, injections=inj)
    counts, events = g.report()
    assert counts["corrected"] == 4 and counts["tiles_detected"] == 4
    assert counts["tiles_checked"] == plan.tiles_m * plan.tiles_n
    Ch = C.float().cpu().numpy()
    for (ti, tj) in tiles:
        r0, c0 = ti * tm, tj * tn
        r1, c1 = min(M, r0 + tm), min(N, c0 + tn)
        Ab = synth.matrix(seedA, M, K, dtype="bf16", r0=r0, r1=r1)
        Bb = synth.matrix(seedB, K, N, dtype="bf16", c0=c0, c1=c1)
        loc = [(r - r0, c - c0, k, b, m, t, a) for (r, c, k, b, m, t, a) in inj if r0 <= r < r1 and c0 <= c < c1]
        ref = oracle.ftgemm(Ab, Bb, out="bf16", tile_m=tm, tile_n=tn, bk=plan.bk, u_acc=plan.u_acc,
                            lambda1=plan.lambda1, lambda2=plan.lambda2, injections=loc)
        assert ref.counts["corrected"] == len(loc)
        blk = Ch[r0:r1, c0:c1].astype(np.float64)
        rel = np.linalg.norm(blk - ref.C) / np.linalg.norm(ref.C)
        assert rel < TOL["bf16"], (ti, tj, rel)
        assert elementwise_ratio(blk, ref, Ab, Bb, plan=plan, out="bf16") <= 1.0, (ti, tj)
        mine = sorted((e["row"] - r0, e["col"] - c0) for e in events if e["tile_m"] == ti and e["tile_n"] == tj)
        assert mine == sorted((e["row"], e["col"]) for e in ref.events)


def test_cfg5_rank_share_sampled():
    """cfg5 (BF16 32768 x 32768 x 16384 over 8 GPUs): one rank's share of the
    M-block partition, run as distributed.PartitionedFTGemm runs it -- the rank's
    4096 rows (check tiles 98..130 of the full problem, generated by global row
    index) with the full problem's tile class -- faults in 3 tiles; whole sampled
    tiles against the tile-local oracle."""
    import torch
    F = ftmod()
    from paper_2305_01024_b200.distributed import row_partition
    Mf, N, K, world, rank = 32768, 32768, 16384, 8, 3
    full = F.plan("bf16", Mf, N, K)
    tm, tn = full.check_tile_m, full.check_tile_n
    row0, M = row_partition(Mf, world, tm)[rank]
    seedA, seedB = synth.BASE_SEED + 11, synth.BASE_SEED + 12
    A = synth.to_torch(synth.matrix(seedA, Mf, K, dtype="bf16", r0=row0, r1=row0 + M), "bf16").cuda()
    B = synth.to_torch(synth.matrix(seedB, K, N, dtype="bf16"), "bf16").cuda()
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    g = F.FTGemm(full.dtype, M, N, K)
    plan = g.plan
    assert (plan.bn, plan.cta_group, plan.check_tile_n) == (full.bn, full.cta_group, full.check_tile_n)
    tiles = [(0, 0), (11, 60), (plan.tiles_m - 1, plan.tiles_n - 1), (20, 7)]
    inj = [(ti * tm + min(3, M - ti * tm - 1), tj * tn + min(9, N - tj * tn - 1), 9000, 30, oracle.INJ_FLIP, 0, 0.0)
           for ti, tj in tiles[:3]]                  # (the last tile column is 8 wide)
    g.encode(A, B)
    g.run(A, B, C, injections=inj)
    counts, events = g.report()
    assert counts["corrected"] == 3 and counts["tiles_detected"] == 3
    assert counts["tiles_checked"] == plan.tiles_m * plan.tiles_n
    for (ti, tj) in tiles:
        r0, c0 = ti * tm, tj * tn
        r1, c1 = min(M, r0 + tm), min(N, c0 + tn)
        Ab = synth.matrix(seedA, Mf, K, dtype="bf16", r0=row0 + r0, r1=row0 + r1)
        Bb = synth.matrix(seedB, K, N, dtype="bf16", c0=c0, c1=c1)
        loc = [(r - r0, c - c0, k, b, m, tg, ad) for (r, c, k, b, m, tg, ad) in inj if r0 <= r < r1 and c0 <= c < c1]
        ref = oracle.ftgemm(Ab, Bb, out="bf16", tile_m=tm, tile_n=tn, bk=plan.bk, u_acc=plan.u_acc,
                            lambda1=plan.lambda1, lambda2=plan.lambda2, injections=loc)
        assert ref.counts["corrected"] == len(loc)
        blk = C[r0:r1, c0:c1].float().cpu().numpy().astype(np.float64)
        assert np.linalg.norm(blk - ref.C) / np.linalg.norm(ref.C) < TOL["bf16"], (ti, tj)
        assert elementwise_ratio(blk, ref, Ab, Bb, plan=plan, out="bf16") <= 1.0, (ti, tj)
        mine = sorted((e["row"] - r0, e["col"] - c0) for e in events if e["tile_m"] == ti and e["tile_n"] == tj)
        assert mine == sorted((e["row"], e["col"]) for e in ref.events)
    del B, C


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("shape", [(16384, 16384, 128), (128, 16384, 16384), (16384, 128, 16384)],
                         ids=["wideC", "skinnyM", "skinnyN"])
def test_cfg4_full_size_sampled(dtype, shape):
    """cfg4 (BASELINE configs[3]) at full size in the plan's launch
    configuration: faults in the first, an interior and the last check tile;
    whole sampled tiles against the tile-local oracle."""
    import torch
    F = ftmod()
    M, N, K = shape
    plan = F.plan(dtype, M, N, K)
    tm, tn = plan.check_tile_m, plan.check_tile_n
    seedA, seedB = synth.BASE_SEED + 21, synth.BASE_SEED + 22
    A = synth.to_torch(synth.matrix(seedA, M, K, dtype=odt(dtype)), odt(dtype)).cuda()
    B = synth.to_torch(synth.matrix(seedB, K, N, dtype=odt(dtype)), odt(dtype)).cuda()
    C = torch.empty(M, N, dtype=A.dtype, device="cuda")
    last = (plan.tiles_m - 1, plan.tiles_n - 1)
    tiles = [(0, 0), (plan.tiles_m // 2, plan.tiles_n // 2), last, (plan.tiles_m - 1, 0)]
    tiles = list(dict.fromkeys(tiles))
    inj = [(ti * tm + min(5, M - ti * tm - 1), tj * tn + min(6, N - tj * tn - 1), K // 2, 0, oracle.INJ_ADD, 0, 5000.0)
           for ti, tj in tiles[:3]]
    inj = list(dict.fromkeys(inj))
    g = F.FTGemm(dtype, M, N, K)
    g.encode(A, B)
    g.run(A, B, C, injections=inj)
    counts, events = g.report()
    assert counts["corrected"] == len(inj) and counts["tiles_detected"] == len(inj), counts
    assert counts["tiles_checked"] == plan.tiles_m * plan.tiles_n
    for (ti, tj) in tiles:
        r0, c0 = ti * tm, tj * tn
        r1, c1 = min(M, r0 + tm), min(N, c0 + tn)
        Ab = oracle_operand(synth.matrix(seedA, M, K, dtype=odt(dtype), r0=r0, r1=r1), dtype)
        Bb = oracle_operand(synth.matrix(seedB, K, N, dtype=odt(dtype), c0=c0, c1=c1), dtype)
        loc = [(r - r0, c - c0, k, b, m, tg, ad) for (r, c, k, b, m, tg, ad) in inj if r0 <= r < r1 and c0 <= c < c1]
        ref = oracle.ftgemm(Ab, Bb, out=odt(dtype), tile_m=tm, tile_n=tn, bk=plan.bk, u_acc=plan.u_acc,
                            lambda1=plan.lambda1, lambda2=plan.lambda2, injections=loc)
        assert ref.counts["corrected"] == len(loc)
        blk = C[r0:r1, c0:c1].float().cpu().numpy().astype(np.float64)
        assert np.linalg.norm(blk - ref.C) / np.linalg.norm(ref.C) < TOL[dtype], (ti, tj)
        assert elementwise_ratio(blk, ref, Ab, Bb, plan=plan, out=odt(dtype)) <= 1.0, (ti, tj)
        mine = sorted((e["row"] - r0, e["col"] - c0) for e in events if e["tile_m"] == ti and e["tile_n"] == tj)
        assert mine == sorted((e["row"], e["col"]) for e in ref.events)
    del A, B, C


@pytest.mark.parametrize("dtype", ["f32_simt", "tf32"])
def test_cfg2_full_size_sampled(dtype):
    """cfg2 at its largest size (8192^3, FP32 operands) in the plan's launch
    configuration, faults in 3 tiles; sampled whole tiles against the tile-local
    oracle -- for the SIMT kernel in FP32SEQ mode, so every clean element must
    be bit-identical (the paper's SGEMM numerics at full K)."""
    import torch
    F = ftmod()
    M = N = K = 8192
    plan = F.plan(dtype, M, N, K)
    tm, tn = plan.check_tile_m, plan.check_tile_n
    seedA, seedB = synth.BASE_SEED + 31, synth.BASE_SEED + 32
    A = synth.to_torch(synth.matrix(seedA, M, K, dtype="f32"), "f32").cuda()
    B = synth.to_torch(synth.matrix(seedB, K, N, dtype="f32"), "f32").cuda()
    C = torch.empty(M, N, dtype=torch.float32, device="cuda")
    tiles = [(0, 0), (plan.tiles_m // 3, plan.tiles_n // 2), (plan.tiles_m - 1, plan.tiles_n - 1), (5, plan.tiles_n - 1)]
    inj = [(ti * tm + min(9, M - ti * tm - 1), tj * tn + min(4, N - tj * tn - 1), 5000, 0, oracle.INJ_ADD, 0, 700.0)
           for ti, tj in tiles[:3]]
    g = F.FTGemm(dtype, M, N, K)
    g.encode(A, B)
    g.run(A, B, C, injections=inj)
    counts, events = g.report()
    assert counts["corrected"] == 3 and counts["tiles_detected"] == 3, counts
    acc = "fp32seq" if dtype == "f32_simt" else "fp64"
    for (ti, tj) in tiles:
        r0, c0 = ti * tm, tj * tn
        r1, c1 = min(M, r0 + tm), min(N, c0 + tn)
        Ab = oracle_operand(synth.matrix(seedA, M, K, dtype="f32", r0=r0, r1=r1), dtype)
        Bb = oracle_operand(synth.matrix(seedB, K, N, dtype="f32", c0=c0, c1=c1), dtype)
        loc = [(r - r0, c - c0, k, b, m, tg, ad) for (r, c, k, b, m, tg, ad) in inj if r0 <= r < r1 and c0 <= c < c1]
        ref = oracle.ftgemm(Ab, Bb, out="f32", acc=acc, tile_m=tm, tile_n=tn, bk=plan.bk, u_acc=plan.u_acc,
                            lambda1=plan.lambda1, lambda2=plan.lambda2, injections=loc)
        assert ref.counts["corrected"] == len(loc)
        blk = C[r0:r1, c0:c1].cpu().numpy()
        if dtype == "f32_simt":
            clean = np.ones(blk.shape, dtype=bool)
            for (r, c, *_) in loc:
                clean[r, c] = False                       # the corrected element: row-sum rounding
            assert np.array_equal(blk[clean], ref.C[clean].astype(np.float32)), (ti, tj)
        rel = np.linalg.norm(blk.astype(np.float64) - ref.C) / np.linalg.norm(ref.C)
        assert rel < (2 * 2 ** -24 * math.sqrt(K) if dtype == "f32_simt" else TOL[dtype]), (ti, tj, rel)
        if dtype != "f32_simt":       # (SIMT: every clean element is bit-exact above; the FP32SEQ
            # reference has no FP64 accumulator to bound against)
            assert elementwise_ratio(blk, ref, Ab, Bb, plan=plan, out="f32") <= 1.0, (ti, tj)
        mine = sorted((e["row"] - r0, e["col"] - c0) for e in events if e["tile_m"] == ti and e["tile_n"] == tj)
        assert mine == sorted((e["row"], e["col"]) for e in ref.events)
    del A, B, C


def test_large_indexing_sampled():
    """C with more than 2^31 elements (65539 x 32768 BF16, 4.3 GB; ragged last
    check-tile row): 64-bit offsets in the encode, fused kernel and epilogue
    stores.  Faults in the first, an interior and the very last tile; whole
    tiles checked against the tile-local oracle."""
    import torch
    F = ftmod()
    M, N, K = 65539, 32768, 256
    plan = F.plan("bf16", M, N, K)
    tm, tn = plan.check_tile_m, plan.check_tile_n
    assert M * N > 2 ** 31
    seedA, seedB = synth.BASE_SEED + 7, synth.BASE_SEED + 8
    A = synth.to_torch(synth.matrix(seedA, M, K, dtype="bf16"), "bf16").cuda()
    B = synth.to_torch(synth.matrix(seedB, K, N, dtype="bf16"), "bf16").cuda()
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    last = (plan.tiles_m - 1, plan.tiles_n - 1)
    tiles = [(0, 0), (300, 70), last, (plan.tiles_m - 1, 0)]
    inj = [(ti * tm + (ti * 7) % min(tm, M - ti * tm), tj * tn + 5, 200, 0, oracle.INJ_ADD, 0, 3000.0)
           for ti, tj in tiles[:3]]
    g = F.FTGemm("bf16", M, N, K)
    g.encode(A, B)
    g.run(A, B, C, injections=inj)
    counts, events = g.report()
    assert counts["corrected"] == 3 and counts["tiles_detected"] == 3
    assert counts["tiles_checked"] == plan.tiles_m * plan.tiles_n
    for (ti, tj) in tiles:
        r0, c0 = ti * tm, tj * tn
        r1, c1 = min(M, r0 + tm), min(N, c0 + tn)
        Ab = synth.matrix(seedA, M, K, dtype="bf16", r0=r0, r1=r1)
        Bb = synth.matrix(seedB, K, N, dtype="bf16", c0=c0, c1=c1)
        loc = [(r - r0, c - c0, k, b, m, tg, ad) for (r, c, k, b, m, tg, ad) in inj if r0 <= r < r1 and c0 <= c < c1]
        ref = oracle.ftgemm(Ab, Bb, out="bf16", tile_m=tm, tile_n=tn, bk=plan.bk, u_acc=plan.u_acc,
                            lambda1=plan.lambda1, lambda2=plan.lambda2, injections=loc)
        blk = C[r0:r1, c0:c1].float().cpu().numpy().astype(np.float64)
        assert np.linalg.norm(blk - ref.C) / np.linalg.norm(ref.C) < TOL["bf16"], (ti, tj)
        assert elementwise_ratio(blk, ref, Ab, Bb, plan=plan, out="bf16") <= 1.0, (ti, tj)
        mine = sorted((e["row"] - r0, e["col"] - c0) for e in events if e["tile_m"] == ti and e["tile_n"] == tj)
        assert mine == sorted((e["row"], e["col"]) for e in ref.events)
    del C


# --------------------------------------------------------------- API errors --

def test_device_argument_errors():
    import torch
    F = ftmod()
    A = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    C = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(F.FtgemmError) as e:
        F.run("bf16", A[:, 1:], A[1:, 1:], C[:, 1:], ft_level=F.FT_OFF)    # misaligned base
    assert e.value.code == 2
    g = F.FTGemm("bf16", 64, 64, 64)
    with pytest.raises(F.FtgemmError) as e:
        F.run("bf16", A, A, C, ft_level=F.FT_OFF, injections=[(0, 0, 0, 3, 0, 0, 0.0)], enc_ws=g.enc_ws,
              report_ws=g.report_ws)
    assert e.value.code == 1


@pytest.mark.parametrize("dtype", ["bf16", "tf32", "f32_simt"])
def test_back_to_back_steps_no_stale_encode(dtype):
    """Steps issued back to back on one stream with alternating inputs: the
    fused GEMM starts under programmatic dependent launch while the encode of
    the same step drains, and must still read only that encode's results.  Every
    C equals (bit for bit) the C of an isolated, synchronised step on the same
    inputs, and no tile is flagged."""
    import torch
    from paper_2305_01024_b200 import ftgemm as F
    M = N = K = 2048
    sets = []
    for s in range(2):
        A, B, _ = synth.problem(M, N, K, dtype=odt(dtype), seed=230501024 + 17 * s)
        sets.append((synth.to_torch(A, odt(dtype)).cuda(), synth.to_torch(B, odt(dtype)).cuda()))
    g = F.FTGemm(dtype, M, N, K)
    ref = []
    for A, B in sets:
        C = torch.empty(M, N, dtype=A.dtype, device="cuda")
        g.encode(A, B)
        g.run(A, B, C)
        torch.cuda.synchronize()
        ref.append(C)
    g.reset()
    outs = []
    for i in range(8):
        A, B = sets[i % 2]
        C = torch.empty(M, N, dtype=A.dtype, device="cuda")
        g.encode(A, B)
        g.run(A, B, C)
        outs.append(C)
    counts, _ = g.report()
    assert counts["tiles_detected"] == 0, counts
    for i, C in enumerate(outs):
        assert torch.equal(C, ref[i % 2]), i


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("beta", [0.0, 0.5])
def test_host_pipeline_matches_isolated_steps(dtype, beta):
    """paper_2305_01024_b200.pipeline.HostPipeline (H2D of step s+1, kernels of
    step s, D2H of step s-1 on three streams, two device slots) returns, for
    every step, the same bits as an isolated synchronised step on the same host
    inputs -- with alternating inputs, so a slot reused too early would show."""
    import torch
    from paper_2305_01024_b200 import ftgemm as F
    from paper_2305_01024_b200.pipeline import HostPipeline
    M, N, K = 1000, 2016, 1024
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    sets = []
    for s in range(3):
        A, B, Cin = synth.problem(M, N, K, dtype=odt(dtype), seed=230501024 + 31 * s)
        sets.append(tuple(synth.to_torch(x, odt(dtype)).pin_memory() for x in (A, B, Cin)))
    g = F.FTGemm(dtype, M, N, K)
    ref = []
    for A, B, Cin in sets:
        C = Cin.cuda()
        g.encode(A.cuda(), B.cuda())
        g.run(A.cuda(), B.cuda(), C, beta=beta)
        torch.cuda.synchronize()
        ref.append(C.cpu())
    g.reset()
    pipe = HostPipeline(g)
    outs = []
    for i in range(7):
        A, B, Cin = sets[i % 3]
        Ch = Cin.clone().pin_memory()          # beta != 0: C_in travels in, C out
        pipe.submit(A, B, Ch, beta=beta)
        outs.append(Ch)
    pipe.synchronize()
    counts, _ = g.report()
    assert counts["tiles_detected"] == 0, counts
    for i, Ch in enumerate(outs):
        assert torch.equal(Ch, ref[i % 3]), i


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("cls", [(256, 2), (256, 1), (128, 1), (128, 2)], ids=lambda c: f"bn{c[0]}cg{c[1]}")
def test_forced_tile_classes_parity(dtype, cls):
    """Every tensor-core tile class the plan's cost model can choose (and
    an explicit FTGEMM_TILE class in the dtype code can force) gives the oracle's C, events and counts,
    with detectable flips in several tiles, including the ragged last ones."""
    F = ftmod()
    M, N, K = 1000, 2016, 1024
    plan = F.plan(dtype, M, N, K, tile=cls)
    assert (plan.bn, plan.cta_group) == cls
    A, B, _ = synth.problem(M, N, K, dtype=odt(dtype))
    inj = detectable_sites(dtype, 8, M, N, K, plan, A, B, seed=71)
    assert len(inj) >= 5
    c = Case(dtype, M, N, K, injections=inj, alpha=1.0, beta=0.25, tile=cls)
    assert c.counts["corrected"] == len(inj), (c.counts, c.ref.counts)
    assert c.events_match() and c.counts_match()
    assert c.fro() < TOL[dtype]
    assert c.elementwise() <= 1.0
