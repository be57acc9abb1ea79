"""Batched launches (ftgemm_run_batched; cfg4 "tall-skinny batches", PAPER.md:450,
:501): `batch` independent problems in ONE persistent launch give, problem by
problem, the bits, events and counts of the single-problem call with the same
tile class, and match the oracle."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import TOL, elementwise_ratio, odt, oracle_operand

pytestmark = pytest.mark.gpu


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


def _stack(dtype, batch, rows, cols, seed, dist="signed"):
    import torch
    xs = [synth.matrix(seed + 97 * b, rows, cols, dist=dist, dtype=odt(dtype)) for b in range(batch)]
    return xs, torch.stack([synth.to_torch(x, odt(dtype)) for x in xs]).cuda()


@pytest.mark.parametrize("tile", [(256, 2), (256, 1), (128, 1), (128, 2)], ids=lambda t: f"bn{t[0]}cg{t[1]}")
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_batched_equals_single_problem_runs(dtype, tile):
    import torch
    F = _F()
    batch, M, N, K = 5, 600, 504, 640
    As, A = _stack(dtype, batch, M, K, 1000)
    Bs, B = _stack(dtype, batch, K, N, 2000)
    Cs, Cin = _stack(dtype, batch, M, N, 3000)
    gb = F.FTGemmBatched(dtype, batch, M, N, K, tile=tile)
    p = gb.plan
    tm, tn = p.check_tile_m, p.check_tile_n
    # faults in problems 0, 2 and 4 (stacked rows), incl. an SEU violation and a checksum fault
    inj = [(0 * M + 3, 7, 100, 30, F.INJ_FLIP, 0, 0.0), (2 * M + tm + 1, tn + 2, 500, 0, F.INJ_ADD, 0, 400.0),
           (4 * M + M - 1, N - 1, K - 1, 0, F.INJ_ADD, 0, -300.0),
           (4 * M + 2, 2, 10, 0, F.INJ_ADD, 0, 77.0), (4 * M + 5, 9, 20, 0, F.INJ_ADD, 0, 55.0),
           (2 * M + 4, 3, 30, 0, F.INJ_ADD, F.TGT_ROW_REF, 300.0)]
    C = Cin.clone()
    gb.encode(A, B)
    gb.run(A, B, C, alpha=1.5, beta=-0.5, injections=inj)
    counts, events = gb.report()
    assert counts["tiles_checked"] == batch * p.tiles_m * p.tiles_n
    key = lambda e: (e["tile_m"], e["tile_n"], e["kind"], e["row"], e["col"], e["n_rows"], e["n_cols"])
    ev_single = []
    for b in range(batch):
        g = F.FTGemm(p.dtype, M, N, K)
        assert (g.plan.bn, g.plan.cta_group) == (p.bn, p.cta_group)
        Cb = Cin[b].clone()
        mine = [(r - b * M, c, k, bt, m, t, a) for (r, c, k, bt, m, t, a) in inj if b * M <= r < (b + 1) * M]
        g.encode(A[b], B[b])
        g.run(A[b], B[b], Cb, alpha=1.5, beta=-0.5, injections=mine)
        _, e = g.report()
        for x in e:
            x = dict(x)
            x["row"] += b * M if x["row"] >= 0 else 0
            x["tile_m"] += b * p.tiles_m
            ev_single.append(x)
        torch.cuda.synchronize()
        assert torch.equal(C[b], Cb), b
    assert sorted(map(key, events)) == sorted(map(key, ev_single))
    assert counts["corrected"] == 3 and counts["uncorrectable"] == 1 and counts["checksum_only"] == 1
    # problem 2 against the oracle, element by element
    loc = [(r - 2 * M, c, k, bt, m, t, a) for (r, c, k, bt, m, t, a) in inj if 2 * M <= r < 3 * M]
    Ao, Bo = oracle_operand(As[2], dtype), oracle_operand(Bs[2], dtype)
    ref = oracle.ftgemm(Ao, Bo, Cs[2], alpha=1.5, beta=-0.5, out=odt(dtype), tile_m=tm, tile_n=tn, bk=p.bk,
                        u_acc=p.u_acc, lambda1=p.lambda1, lambda2=p.lambda2, injections=loc)
    Cg = C[2].float().cpu().numpy()
    assert elementwise_ratio(Cg, ref, Ao, Bo, Cs[2], alpha=1.5, beta=-0.5, plan=p, out=odt(dtype)) <= 1.0


def test_batched_integer_bit_exact_shared_b():
    """Integer inputs, one B shared by every problem (stride_b = 0), integer
    faults: C bit-identical to the oracle in every problem."""
    F = _F()
    batch, M, N, K = 4, 333, 264, 512
    As, A = _stack("bf16", batch, M, K, 4000, dist="int")
    Bs, B1 = _stack("bf16", 1, K, N, 5000, dist="int")
    B = B1.expand(batch, K, N)
    gb = F.FTGemmBatched("bf16", batch, M, N, K)
    p = gb.plan
    inj = [(b * M + 7 * b + 1, 11 * b + 3, 64 * b + 5, 0, F.INJ_ADD, 0, float(13 + b)) for b in range(batch)]
    import torch
    C = torch.empty(batch, M, N, dtype=torch.bfloat16, device="cuda")
    gb.encode(A, B)
    gb.run(A, B, C, injections=inj)
    counts, _ = gb.report()
    assert counts["corrected"] == batch
    for b in range(batch):
        loc = [(r - b * M, c, k, bt, m, t, a) for (r, c, k, bt, m, t, a) in inj if b * M <= r < (b + 1) * M]
        ref = oracle.ftgemm(As[b], Bs[0], out="bf16", tile_m=p.check_tile_m, tile_n=p.check_tile_n, bk=p.bk,
                            u_acc=p.u_acc, lambda1=p.lambda1, lambda2=p.lambda2, injections=loc)
        assert np.array_equal(C[b].float().cpu().numpy(), ref.C), b


def test_cfg4_tall_skinny_batch32_sampled():
    """cfg4 tall-skinny batch: 32 x (4096, 128, 4096) BF16 in one launch, faults
    in problems 0, 17 and 31; sampled whole check tiles against the tile-local
    oracle; every tile checked, every fault corrected."""
    import torch
    F = _F()
    batch, M, N, K = 32, 4096, 128, 4096
    A = torch.stack([synth.matrix_torch(synth.BASE_SEED + 41 + b, M, K, dtype="bf16") for b in range(batch)])
    B = torch.stack([synth.matrix_torch(synth.BASE_SEED + 141 + b, K, N, dtype="bf16") for b in range(batch)])
    C = torch.empty(batch, M, N, dtype=torch.bfloat16, device="cuda")
    gb = F.FTGemmBatched("bf16", batch, M, N, K)
    p = gb.plan
    tm, tn = p.check_tile_m, p.check_tile_n
    inj = [(0 * M + 5, 6, 2000, 30, F.INJ_FLIP, 0, 0.0), (17 * M + 2000, 100, 4095, 0, F.INJ_ADD, 0, 900.0),
           (31 * M + M - 1, N - 1, 17, 30, F.INJ_FLIP, 0, 0.0)]
    gb.encode(A, B)
    gb.run(A, B, C, injections=inj)
    counts, events = gb.report()
    assert counts["corrected"] == 3 and counts["tiles_detected"] == 3
    assert counts["tiles_checked"] == batch * p.tiles_m * p.tiles_n
    for b, ti in ((0, 0), (17, 2000 // tm), (31, p.tiles_m - 1), (9, 5)):
        r0, r1 = ti * tm, min(M, ti * tm + tm)
        Ab = synth.matrix(synth.BASE_SEED + 41 + b, M, K, dtype="bf16", r0=r0, r1=r1)
        Bb = synth.matrix(synth.BASE_SEED + 141 + b, K, N, dtype="bf16")
        loc = [(r - b * M - r0, c, k, bt, m, t, a) for (r, c, k, bt, m, t, a) in inj if b * M + r0 <= r < b * M + r1]
        ref = oracle.ftgemm(Ab, Bb, out="bf16", tile_m=tm, tile_n=tn, bk=p.bk, u_acc=p.u_acc, lambda1=p.lambda1,
                            lambda2=p.lambda2, injections=loc)
        assert ref.counts["corrected"] == len(loc)
        blk = C[b, r0:r1].float().cpu().numpy()
        assert np.linalg.norm(blk - ref.C) / np.linalg.norm(ref.C) < TOL["bf16"]
        assert elementwise_ratio(blk, ref, Ab, Bb, plan=p, out="bf16") <= 1.0, (b, ti)
        mine = sorted((e["row"] - b * M - r0, e["col"]) for e in events if e["tile_m"] == b * p.tiles_m + ti)
        assert mine == sorted((e["row"], e["col"]) for e in ref.events)
