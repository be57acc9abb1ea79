"""M-block partition of the FT GEMM over the GPUs of one node (north_star item 6).

C = A B is split by rows of A / C: rank r owns the check-tile-aligned row block
``row_partition(M, world, tile_m)[r]``; B (and its encoded row checksums, the B
part of the encode workspace) are broadcast ONCE from the source rank with NCCL
(torch.distributed) -- over NVLink 5 / NVSwitch on a B200 box -- and every rank
then runs its fused FT GEMM independently.  The only other collectives are the
all-reduce of the report counters and the gather of fault events.  There is no
collective on the data path of a step: the partition is embarrassingly parallel
(DESIGN.md §Multi-GPU).

One process per GPU; the process group is created by the caller (bench.py /
tests) with backend "nccl" on GPUs or "gloo" for the host-logic tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

COUNT_KEYS = ("tiles_checked", "tiles_detected", "corrected", "checksum_only", "uncorrectable", "located",
              "events", "dropped")


def row_partition(M: int, world: int, tile_m: int):
    """[(row0, rows)] per rank: whole check tiles, as even as possible, so that
    every rank's check tiles coincide with the 1-GPU check tiles."""
    tiles = -(-M // tile_m)
    base, extra = divmod(tiles, world)
    out, t = [], 0
    for r in range(world):
        nt = base + (1 if r < extra else 0)
        row0 = min(M, t * tile_m)
        row1 = min(M, (t + nt) * tile_m)
        out.append((row0, row1 - row0))
        t += nt
    return out


def broadcast_b(g, B: torch.Tensor, src: int = 0, group=None, encode_fn=None) -> float:
    """Encode B on ``src`` and broadcast B and the B part of the encode workspace.

    ``g`` is an FTGemm (or any object with ``enc_b`` and ``encode``);
    returns the elapsed milliseconds of encode + broadcast (host wall clock on
    CPU backends, CUDA events on GPUs)."""
    rank = dist.get_rank(group)
    on_gpu = B.is_cuda
    if on_gpu:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    else:
        import time
        t0 = time.perf_counter()
    if rank == src:
        (encode_fn or (lambda: g.encode(None, B, which=2)))()
    dist.broadcast(B, src, group=group)
    dist.broadcast(g.enc_b, src, group=group)
    if on_gpu:
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1)
    return (time.perf_counter() - t0) * 1e3


def allreduce_counts(counts: dict, device, group=None) -> dict:
    v = torch.tensor([int(counts.get(k, 0)) for k in COUNT_KEYS], dtype=torch.int64, device=device)
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    return {k: int(x) for k, x in zip(COUNT_KEYS, v.tolist())}


def gather_events(events: list, row0: int, tile_row0: int, group=None) -> list:
    """All ranks' events in global coordinates (rows and tile_m shifted by the
    rank's block offset), sorted like the single-GPU report."""
    mine = []
    for e in events:
        e = dict(e)
        if e["row"] >= 0:
            e["row"] += row0
        e["tile_m"] += tile_row0
        mine.append(e)
    world = dist.get_world_size(group)
    allv = [None] * world
    dist.all_gather_object(allv, mine, group=group)
    out = [e for part in allv for e in part]
    out.sort(key=lambda e: (e["tile_m"], e["tile_n"], e["kind"], e["row"], e["col"]))
    return out


class PartitionedFTGemm:
    """The local share of an M-block-partitioned FT GEMM on this rank."""

    def __init__(self, dtype, M: int, N: int, K: int, device=None, group=None, gemm_factory=None):
        """gemm_factory(code, rows, N, K, device=...) builds the per-rank GEMM
        object (default: ftgemm.FTGemm; tests substitute a host stand-in to
        drive this logic over gloo on CPU)."""
        from . import ftgemm as F
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        full = F.plan(dtype, M, N, K)
        self.parts = row_partition(M, self.world, full.check_tile_m)
        self.row0, self.rows = self.parts[self.rank]
        self.tile_row0 = self.row0 // full.check_tile_m
        self.M, self.N, self.K = M, N, K
        # every rank runs the full problem's tile class (its own, smaller M could
        # make the plan's wave model pick another check-tile width): full.dtype is
        # the full plan's explicit dtype code (dtype | FTGEMM_TILE(bn, cta_group))
        self.g = (gemm_factory or F.FTGemm)(full.dtype, max(self.rows, 1), N, K,
                                            device=device or torch.device("cuda", torch.cuda.current_device()))
        # the B part of the workspace is only shareable when every rank has the same geometry
        sig = torch.tensor([self.g.plan.bn, self.g.plan.tiles_n, self.g.plan.enc_b_bytes], dtype=torch.int64,
                           device=self.g.enc_ws.device)
        ref = sig.clone()
        dist.broadcast(ref, 0, group=group)
        self.same_geometry = bool(torch.equal(sig, ref))
        agree = torch.tensor([1 if self.same_geometry else 0], dtype=torch.int64, device=sig.device)
        dist.all_reduce(agree, op=dist.ReduceOp.MIN, group=group)
        self.share_b = bool(agree.item())

    def set_b(self, B: torch.Tensor, src: int = 0) -> float:
        """Broadcast B once (and its encode when all ranks share the geometry)."""
        if self.share_b:
            return broadcast_b(self.g, B, src, self.group)
        dist.broadcast(B, src, group=self.group)
        self.g.encode(None, B, which=2)
        return 0.0

    def run(self, A_local, B, C_local, **kw):
        """kw as FTGemm.run; fuse_a=True encodes the rank's A block inside the
        GEMM kernel (ftgemm_run_fused) instead of a separate pass."""
        if self.rows == 0:
            return
        if kw.get("ft_level", 2) != 0 and not kw.get("fuse_a", False):
            self.g.encode(A_local, None, which=1)
        self.g.run(A_local, B, C_local, **kw)

    def report(self):
        counts, events = self.g.report()
        total = allreduce_counts(counts, self.g.enc_ws.device, self.group)
        return total, gather_events(events, self.row0, self.tile_row0, self.group)
