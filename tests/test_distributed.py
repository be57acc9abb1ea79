"""Host logic of the M-block partition (paper_2305_01024_b200/distributed.py)
with world_size 2 over gloo on CPU: row partition, the one-time broadcast of B
and its encode, the counter all-reduce and the event gather.  The per-rank GEMM
is replaced by the oracle (tests may use it) so that the concatenated result
and the global event list can be compared with a single-process run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2305_01024_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_partition():
    for M, world, tm in [(8192, 2, 125), (8192, 8, 125), (1000, 3, 128), (10, 4, 125), (32768, 8, 125)]:
        parts = D.row_partition(M, world, tm)
        assert len(parts) == world
        assert sum(r for _, r in parts) == M
        assert parts[0][0] == 0
        for (r0, n), (r1, _) in zip(parts, parts[1:]):
            assert r0 + n == r1
        for r0, n in parts:
            assert n == 0 or r0 % tm == 0            # check tiles coincide with the 1-GPU tiles
        sizes = [n for _, n in parts if n]
        assert max(sizes) - min(sizes) <= 2 * tm     # whole tiles; the last one may be partial


class _StubG:
    """Stands in for FTGemm on CPU: enc_b holds the FP64 B-encode bytes."""

    def __init__(self, K, N, tile_n):
        self.K, self.N, self.tile_n = K, N, tile_n
        nbytes = 8 * K * (-(-N // tile_n))
        self.enc_ws = torch.zeros(nbytes + 64, dtype=torch.uint8)
        self.enc_b = self.enc_ws[64:]

    def encode_b(self, B):
        Br = oracle.encode_row(B.numpy(), self.tile_n)
        self.enc_b.copy_(torch.from_numpy(Br.reshape(-1).view(np.uint8).copy()))


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M, N, K, tm, tn = 300, 200, 96, 64, 64
        A_full, B_np, _ = synth.problem(M, N, K, with_c=False)
        g = _StubG(K, N, tn)
        B = torch.from_numpy(B_np.copy()) if rank == 0 else torch.zeros(K, N)
        D.broadcast_b(g, B, src=0, encode_fn=lambda: g.encode_b(B))
        assert torch.equal(B, torch.from_numpy(B_np))
        ref_enc = oracle.encode_row(B_np, tn).reshape(-1).view(np.uint8)
        assert np.array_equal(g.enc_b.numpy(), ref_enc)
        # the local share, computed by the oracle as the stand-in GEMM
        row0, rows = D.row_partition(M, world, tm)[rank]
        inj_global = [(70, 10, 50, 0, oracle.INJ_ADD, 0, 99.0), (250, 150, 20, 0, oracle.INJ_ADD, 0, -42.0)]
        inj = [(r - row0, c, k, b, m, t, a) for (r, c, k, b, m, t, a) in inj_global if row0 <= r < row0 + rows]
        res = oracle.ftgemm(A_full[row0:row0 + rows], B_np, tile_m=tm, tile_n=tn, bk=8, injections=inj)
        total = D.allreduce_counts(res.counts, torch.device("cpu"))
        evs = D.gather_events(res.events, row0, row0 // tm)
        parts = [None] * world
        dist.all_gather_object(parts, (row0, res.C))
        if rank == 0:
            import pickle
            with open(out_path, "wb") as f:
                pickle.dump((total, evs, parts), f)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partition_matches_single_process(tmp_path):
    import pickle
    world = 2
    out = str(tmp_path / "res.pkl")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    with open(out, "rb") as f:
        total, evs, parts = pickle.load(f)
    M, N, K, tm, tn = 300, 200, 96, 64, 64
    A, B, _ = synth.problem(M, N, K, with_c=False)
    inj = [(70, 10, 50, 0, oracle.INJ_ADD, 0, 99.0), (250, 150, 20, 0, oracle.INJ_ADD, 0, -42.0)]
    ref = oracle.ftgemm(A, B, tile_m=tm, tile_n=tn, bk=8, injections=inj)
    C = np.concatenate([c for _, c in sorted(parts, key=lambda x: x[0])], axis=0)
    assert np.array_equal(C, ref.C)
    for k in ("tiles_checked", "corrected", "tiles_detected"):
        assert total[k] == ref.counts[k]
    key = lambda e: (e["tile_m"], e["tile_n"], e["row"], e["col"], e["kind"])
    assert sorted(map(key, evs)) == sorted(map(key, ref.events))


class _HostFTGemm:
    """Host stand-in for ftgemm.FTGemm with the real plan (the C ABI's pure-host
    ftgemm_plan) and workspace layout sizes; encode writes the oracle's FP64
    B-encode into the B part of enc_ws, run is the oracle on the plan's check
    tiles.  Lets the real PartitionedFTGemm logic run over gloo on CPU."""

    def __init__(self, code, M, N, K, device=None):
        from paper_2305_01024_b200 import ftgemm as F
        self.M, self.N, self.K = M, N, K
        self.plan = F.plan(code, M, N, K)
        self.dtype = self.plan.dtype
        self.enc_ws = torch.zeros(self.plan.enc_bytes, dtype=torch.uint8)
        self.counts, self.events, self.encoded_a = None, [], False

    @property
    def enc_b(self):
        p = self.plan
        return self.enc_ws[p.enc_b_offset:p.enc_b_offset + p.enc_b_bytes]

    def encode(self, A=None, B=None, which=3, stream=None):
        if which & 2:
            Br = oracle.encode_row(B.numpy(), self.plan.check_tile_n).reshape(-1).view(np.uint8)
            self.enc_b[:Br.size].copy_(torch.from_numpy(Br.copy()))
        if which & 1:
            self.encoded_a = True

    def run(self, A, B, C, ft_level=2, injections=(), **kw):
        p = self.plan
        Br = oracle.encode_row(B.numpy(), p.check_tile_n).reshape(-1).view(np.uint8)
        assert self.encoded_a and np.array_equal(self.enc_b[:Br.size].numpy(), Br), "B part of enc_ws not shared"
        res = oracle.ftgemm(A.numpy(), B.numpy(), out="f32", tile_m=p.check_tile_m, tile_n=p.check_tile_n, bk=p.bk,
                            u_acc=p.u_acc, lambda1=p.lambda1, lambda2=p.lambda2, injections=injections)
        C.copy_(torch.from_numpy(res.C))
        self.counts, self.events = res.counts, res.events

    def report(self):
        return dict(self.counts), list(self.events)


def _worker_partitioned(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M, N, K = 700, 520, 128
        A_full, B_np, _ = synth.problem(M, N, K, with_c=False, dtype="bf16")
        P = D.PartitionedFTGemm("bf16", M, N, K, device=torch.device("cpu"), gemm_factory=_HostFTGemm)
        assert P.share_b
        B = torch.from_numpy(B_np.copy()) if rank == 0 else torch.zeros(K, N)
        P.set_b(B)                                    # B and its encode from rank 0, once
        assert torch.equal(B, torch.from_numpy(B_np))
        tm = P.g.plan.check_tile_m
        inj_global = [(3, 10, 50, 0, oracle.INJ_ADD, 0, 99.0), (2 * tm + 4, 300, 20, 0, oracle.INJ_ADD, 0, -42.0),
                      (M - 1, N - 1, 100, 0, oracle.INJ_ADD, 0, 7.0)]
        inj = [(r - P.row0, c, k, b, m, t, a) for (r, c, k, b, m, t, a) in inj_global
               if P.row0 <= r < P.row0 + P.rows]
        A = torch.from_numpy(A_full[P.row0:P.row0 + P.rows].copy())
        C = torch.zeros(P.rows, N)
        P.run(A, B, C, injections=inj)
        total, evs = P.report()
        parts = [None] * world
        dist.all_gather_object(parts, (P.row0, C.numpy()))
        if rank == 0:
            import pickle
            with open(out_path, "wb") as f:
                pickle.dump((total, evs, parts, (P.g.plan.check_tile_m, P.g.plan.check_tile_n, P.g.plan.bk,
                                                 P.g.plan.u_acc, P.g.plan.lambda1, P.g.plan.lambda2)), f)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partitioned_ftgemm(tmp_path):
    """The real PartitionedFTGemm (set_b, run, report) over gloo, world 2, with
    a host stand-in GEMM: every rank uses the full problem's tile class, B and
    its encode arrive from rank 0, counters are all-reduced and events gathered
    in global coordinates; the concatenated C and the events equal the
    single-process oracle on the full problem."""
    import pickle
    world = 2
    out = str(tmp_path / "res.pkl")
    mp.spawn(_worker_partitioned, args=(world, _free_port(), out), nprocs=world, join=True)
    with open(out, "rb") as f:
        total, evs, parts, (tm, tn, bk, u, l1, l2) = pickle.load(f)
    M, N, K = 700, 520, 128
    A, B, _ = synth.problem(M, N, K, with_c=False, dtype="bf16")
    inj = [(3, 10, 50, 0, oracle.INJ_ADD, 0, 99.0), (2 * tm + 4, 300, 20, 0, oracle.INJ_ADD, 0, -42.0),
           (M - 1, N - 1, 100, 0, oracle.INJ_ADD, 0, 7.0)]
    ref = oracle.ftgemm(A, B, out="f32", tile_m=tm, tile_n=tn, bk=bk, u_acc=u, lambda1=l1, lambda2=l2, injections=inj)
    C = np.concatenate([c for _, c in sorted(parts, key=lambda x: x[0])], axis=0)
    assert np.array_equal(C, ref.C)
    for k in ("tiles_checked", "corrected", "tiles_detected", "uncorrectable"):
        assert total[k] == ref.counts[k], k
    assert total["corrected"] == 3
    key = lambda e: (e["tile_m"], e["tile_n"], e["row"], e["col"], e["kind"])
    assert sorted(map(key, evs)) == sorted(map(key, ref.events))
