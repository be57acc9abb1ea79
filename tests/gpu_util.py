"""Shared helpers for the GPU parity tests: run one problem through the C ABI
(paper_2305_01024_b200.ftgemm) and through the CPU oracle on the same seeded
inputs, and compare."""
from __future__ import annotations

import numpy as np

import oracle
import synth

TOL = {"f32_simt": 1e-6, "tf32": 5e-3, "bf16": 2e-2}   # north_star relative Frobenius bounds


def odt(dtype: str) -> str:
    return "bf16" if dtype == "bf16" else "f32"


def padded(x: np.ndarray, dtype: str, ld: int | None):
    """Device tensor holding x with leading dimension ld (a strided view)."""
    import torch
    t = synth.to_torch(x, odt(dtype))
    if ld is None or ld == x.shape[1]:
        return t.cuda()
    big = torch.zeros(x.shape[0], ld, dtype=t.dtype)
    big[:, :x.shape[1]] = t
    return big.cuda()[:, :x.shape[1]]


def frob(gpu: np.ndarray, ref: np.ndarray, mask: np.ndarray | None = None) -> float:
    g = gpu.astype(np.float64)
    r = ref.astype(np.float64)
    if mask is not None:
        g, r = g[mask], r[mask]
    return float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300))


class Case:
    """One problem: inputs, the GPU result through the C ABI, the oracle result."""

    def __init__(self, dtype, M, N, K, *, dist="signed", alpha=1.0, beta=0.0, ft=2, injections=(),
                 seed=synth.BASE_SEED, lda=None, ldb=None, ldc=None, acc="fp64", run_oracle=True):
        import torch
        from paper_2305_01024_b200 import ftgemm as F
        self.dtype, self.M, self.N, self.K = dtype, M, N, K
        self.A, self.B, self.Cin = synth.problem(M, N, K, dist=dist, dtype=odt(dtype), seed=seed)
        self.g = F.FTGemm(dtype, M, N, K)
        self.plan = p = self.g.plan
        Ad, Bd = padded(self.A, dtype, lda), padded(self.B, dtype, ldb)
        Cd = padded(self.Cin, dtype, ldc)
        self.injections = list(injections)
        if ft != F.FT_OFF:
            self.g.encode(Ad, Bd)
        self.g.run(Ad, Bd, Cd, alpha=alpha, beta=beta, ft_level=ft, injections=self.injections)
        torch.cuda.synchronize()
        self.counts, self.events = self.g.report() if ft != F.FT_OFF else ({}, [])
        self.C = Cd.float().cpu().numpy()
        self.C_raw = Cd.cpu()
        self.ref = None
        if run_oracle:
            tm, tn = (p.check_tile_m, p.check_tile_n) if ft != F.FT_OFF else (p.off_tile_m, p.off_tile_n)
            self.ref = oracle.ftgemm(self.A, self.B, self.Cin, alpha=alpha, beta=beta, out=odt(dtype), acc=acc,
                                     tile_m=tm, tile_n=tn, bk=p.bk, u_acc=p.u_acc, lambda1=p.lambda1,
                                     lambda2=p.lambda2, ft_level=ft, injections=self.injections)

    def fro(self, mask=None) -> float:
        return frob(self.C, self.ref.C, mask)

    def event_keys(self, evs):
        return sorted((e["tile_m"], e["tile_n"], e["kind"], e["row"], e["col"], e["n_rows"], e["n_cols"]) for e in evs)

    def events_match(self) -> bool:
        return self.event_keys(self.events) == self.event_keys(self.ref.events)

    def counts_match(self) -> bool:
        keys = ("tiles_checked", "tiles_detected", "corrected", "checksum_only", "uncorrectable", "located", "events")
        return all(int(self.counts.get(k, 0)) == int(self.ref.counts.get(k, 0)) for k in keys)


def detectable_sites(dtype, n, M, N, K, plan, A, B, seed, *, benign=False):
    """Seeded fault sites with a bit whose flip is >= 4 tau (or benign, <= tau/4)
    according to the oracle (oracle/sites.py)."""
    from oracle.sites import classify_bits
    sites = synth.injection_sites(n, M, N, K, plan.check_tile_m, plan.check_tile_n, plan.bk, seed=seed)
    out = []
    for i, (r, c, k) in enumerate(sites):
        det, ben, _, _ = classify_bits(A, B, r, c, k, tile_m=plan.check_tile_m, tile_n=plan.check_tile_n,
                                       bk=plan.bk, u_acc=plan.u_acc, lambda1=plan.lambda1, lambda2=plan.lambda2)
        pool = ben if benign else det
        if not pool:
            continue
        out.append((r, c, k, pool[(i * 7 + seed) % len(pool)], oracle.INJ_FLIP, oracle.TGT_ACC, 0.0))
    return out
