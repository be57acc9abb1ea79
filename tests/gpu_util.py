"""Shared helpers for the GPU parity tests: run one problem through the C ABI
(paper_2305_01024_b200.ftgemm) and through the CPU oracle on the same seeded
inputs, and compare."""
from __future__ import annotations

import math

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


def tf32(x: np.ndarray) -> np.ndarray:
    """The operand values a kind::tf32 MMA multiplies: FP32 with the low 13
    mantissa bits dropped (truncation, pinned on the device by
    test_tf32_operand_semantics; R8).  The oracle is given these, so
    it computes the product of the values the tensor core actually sees."""
    return (np.ascontiguousarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def oracle_operand(x: np.ndarray, dtype: str) -> np.ndarray:
    return tf32(x) if dtype == "tf32" else x


def elementwise_ratio(Cg, ref, A, B, Cin=None, *, alpha=1.0, beta=0.0, plan, out, skip=None) -> float:
    """max over elements of |C_gpu - C_oracle| / bound (<= 1 passes), R18.

    Clean element (p,q), from the accumulation-error model the threshold uses
    (R1; products exact in every variant, FP32 accumulation):
        |alpha| u (l1 sqrt(K) |P_pq| + l2 ||A_p|| ||B_q||)
      + 2^-23 (|alpha P_pq| + |beta Cin_pq|)          (FP32 alpha/beta epilogue)
      + ulp_out |C_pq|                                  (both sides round once: 2^-7 BF16, 2^-23 FP32)
    Corrected element (row reconstruction R_row[p] - sum_{q' != q} acc, R2):
        |alpha| (tau_row(p) + u bn sum_q' |P_pq'|) + the same epilogue / rounding terms,
    tau_row from the oracle.  skip: boolean mask of elements compared elsewhere
    (uncorrectable / DETECT tiles: by position and kind only, R13)."""
    K = A.shape[1]
    u, l1, l2 = float(plan.u_acc), float(plan.lambda1), float(plan.lambda2)
    P = ref.P
    na = np.linalg.norm(A.astype(np.float64), axis=1)[:, None]
    nb = np.linalg.norm(B.astype(np.float64), axis=0)[None, :]
    uo = 2.0 ** -7 if out == "bf16" else 2.0 ** -23
    cin = np.abs(Cin.astype(np.float64)) if (Cin is not None and beta != 0.0) else 0.0
    ep = 2.0 ** -23 * (abs(alpha) * np.abs(P) + abs(beta) * cin) + uo * np.abs(ref.C.astype(np.float64)) + 1e-30
    bound = abs(alpha) * u * (l1 * math.sqrt(K) * np.abs(P) + l2 * na * nb) + ep
    tn = plan.check_tile_n
    for e in ref.events:
        if e["kind"] == oracle.EV_CORRECTED:
            p, q = e["row"], e["col"]
            tj = q // tn
            rowabs = np.abs(P[p, tj * tn:(tj + 1) * tn]).sum()
            epq = ep if np.isscalar(ep) else ep[p, q]
            bound[p, q] = abs(alpha) * (ref.tau_row[p, tj] + u * tn * rowabs) + epq
    diff = np.abs(Cg.astype(np.float64) - ref.C.astype(np.float64))
    ratio = diff / bound
    ratio[~np.isfinite(diff)] = np.inf
    if skip is not None:
        ratio[skip] = 0.0
    return float(ratio.max()) if ratio.size else 0.0


def uncorrectable_mask(ref, M, N, tm, tn):
    bad = np.zeros((M, N), bool)
    for e in ref.events:
        if e["kind"] == oracle.EV_UNCORRECTABLE:
            bad[e["tile_m"] * tm:(e["tile_m"] + 1) * tm, e["tile_n"] * tn:(e["tile_n"] + 1) * tn] = True
    return bad


def frob(gpu: np.ndarray, ref: np.ndarray, mask: np.ndarray | None = None) -> float:
    g = gpu.astype(np.float64)
    r = ref.astype(np.float64)
    if mask is not None:
        g, r = g[mask], r[mask]
    return float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300))


class Case:
    """One problem: inputs, the GPU result through the C ABI, the oracle result."""

    def __init__(self, dtype, M, N, K, *, dist="signed", alpha=1.0, beta=0.0, ft=2, injections=(),
                 seed=synth.BASE_SEED, lda=None, ldb=None, ldc=None, acc="fp64", run_oracle=True, tile=None):
        import torch
        from paper_2305_01024_b200 import ftgemm as F
        self.dtype, self.M, self.N, self.K = dtype, M, N, K
        self.A, self.B, self.Cin = synth.problem(M, N, K, dist=dist, dtype=odt(dtype), seed=seed)
        self.g = F.FTGemm(dtype, M, N, K, tile=tile)
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
        self.alpha, self.beta = alpha, beta
        if run_oracle:
            tm, tn = (p.check_tile_m, p.check_tile_n) if ft != F.FT_OFF else (p.off_tile_m, p.off_tile_n)
            self.Ao, self.Bo = oracle_operand(self.A, dtype), oracle_operand(self.B, dtype)
            self.ref = oracle.ftgemm(self.Ao, self.Bo, self.Cin, alpha=alpha, beta=beta, out=odt(dtype), acc=acc,
                                     tile_m=tm, tile_n=tn, bk=p.bk, u_acc=p.u_acc, lambda1=p.lambda1,
                                     lambda2=p.lambda2, ft_level=ft, injections=self.injections)

    def fro(self, mask=None) -> float:
        return frob(self.C, self.ref.C, mask)

    def elementwise(self, skip=None) -> float:
        """max |C_gpu - C_oracle| / per-element bound (elementwise_ratio)."""
        return elementwise_ratio(self.C, self.ref, self.Ao, self.Bo, self.Cin, alpha=self.alpha, beta=self.beta,
                                 plan=self.plan, out=odt(self.dtype), skip=skip)

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
