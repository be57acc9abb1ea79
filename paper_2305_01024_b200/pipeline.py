"""Host <-> device pipeline of FT GEMM steps (stream orchestration only).

A step takes host operands A, B and returns the host result C = alpha*A*B +
beta*C with the fused online ABFT of the C ABI (ftgemm_encode + ftgemm_run).
Run one step at a time, the H2D copies, the kernels and the D2H copy serialise
(B200 BF16 8192^3: ~4.7 ms + 0.9 ms + 2.3 ms over PCIe).  HostPipeline overlaps
them across steps on three CUDA streams with double-buffered device operands:

    copy-in stream   H2D A_s, B_s into slot s % 2          (waits: compute of s-2 done)
    compute stream   ftgemm_encode + ftgemm_run on slot s  (waits: H2D of s, D2H of s-2)
    copy-out stream  D2H C_s from slot s % 2               (waits: compute of s)

so a step costs max(H2D, compute, D2H) instead of their sum (with a resident,
pre-encoded B -- weights, or the broadcast B of an M-block partition -- only A
travels and only A is encoded per step): H2D and D2H use
separate copy engines (opposite PCIe directions) and the kernels run beside
them.  Every slot's reuse is ordered by CUDA events, so the results are the
same bits as isolated steps (tests/test_gpu_parity.py).  The workspaces of the
FT GEMM are shared by all steps: the compute stream serialises encode and run.
No arithmetic happens here; every step's work runs in libftgemm's kernels.
"""
from __future__ import annotations

import torch

from . import ftgemm as F


class HostPipeline:
    """Pipelined FT GEMM steps over pinned host buffers for one (dtype, M, N, K)."""

    def __init__(self, g: "F.FTGemm", *, depth: int = 2, device="cuda", b_resident: torch.Tensor | None = None):
        """b_resident: a device B already encoded into g (ftgemm_encode which=2);
        steps then upload and encode only A (submit(A_host, None, C_host))."""
        if depth < 2:
            raise ValueError("depth must be >= 2 (double buffering)")
        self.g = g
        self.depth = depth
        dt = {F.BF16: torch.bfloat16}.get(g.dtype & F.DTYPE_MASK, torch.float32)
        M, N, K = g.M, g.N, g.K
        self.A = [torch.empty(M, K, dtype=dt, device=device) for _ in range(depth)]
        self.b_resident = b_resident
        self.B = [b_resident] * depth if b_resident is not None else \
            [torch.empty(K, N, dtype=dt, device=device) for _ in range(depth)]
        self.C = [torch.empty(M, N, dtype=dt, device=device) for _ in range(depth)]
        self.s_in = torch.cuda.Stream(device=device)
        self.s_cmp = torch.cuda.Stream(device=device)
        self.s_out = torch.cuda.Stream(device=device)
        ev = lambda: [torch.cuda.Event() for _ in range(depth)]  # noqa: E731
        self.in_done, self.cmp_done, self.out_done = ev(), ev(), ev()
        self.n = 0                                   # steps submitted

    def begin(self, stream=None):
        """Order the pipeline's streams after the work queued so far on `stream`
        (default: the current stream), e.g. after a timing event."""
        st = stream or torch.cuda.current_stream()
        e = torch.cuda.Event()
        e.record(st)
        for s in (self.s_in, self.s_cmp, self.s_out):
            s.wait_event(e)

    def submit(self, A_host: torch.Tensor, B_host: torch.Tensor, C_host: torch.Tensor, *, alpha=1.0, beta=0.0,
               ft_level=F.FT_CORRECT, injections=()):
        """Queue one step: H2D of A_host / B_host (and C_host when beta != 0),
        encode + fused FT GEMM, D2H of the result into C_host (pinned host
        tensors; C_host must stay alive until synchronize())."""
        s, k = self.n % self.depth, self.n
        if k >= self.depth:                      # slot s was last used by step k - depth
            self.s_in.wait_event(self.cmp_done[s])
        with torch.cuda.stream(self.s_in):
            self.A[s].copy_(A_host, non_blocking=True)
            if self.b_resident is None:
                self.B[s].copy_(B_host, non_blocking=True)
            if beta != 0.0:
                if k >= self.depth:
                    self.s_in.wait_event(self.out_done[s])
                self.C[s].copy_(C_host, non_blocking=True)
            self.in_done[s].record(self.s_in)
        self.s_cmp.wait_event(self.in_done[s])
        if k >= self.depth:
            self.s_cmp.wait_event(self.out_done[s])  # C slot read back before it is overwritten
        g, st = self.g, self.s_cmp
        if ft_level != F.FT_OFF:
            if self.b_resident is None:
                g.encode(self.A[s], self.B[s], stream=st)
            else:
                g.encode(self.A[s], None, which=1, stream=st)
        g.run(self.A[s], self.B[s], self.C[s], alpha=alpha, beta=beta, ft_level=ft_level, injections=injections,
              stream=st)
        self.cmp_done[s].record(st)
        self.s_out.wait_event(self.cmp_done[s])
        with torch.cuda.stream(self.s_out):
            C_host.copy_(self.C[s], non_blocking=True)
            self.out_done[s].record(self.s_out)
        self.n += 1

    def join(self, stream=None):
        """Make `stream` (default: the current stream) wait for every queued step."""
        st = stream or torch.cuda.current_stream()
        for s in range(min(self.n, self.depth)):
            st.wait_event(self.out_done[s])
            st.wait_event(self.cmp_done[s])

    def synchronize(self):
        for s in (self.s_in, self.s_cmp, self.s_out):
            s.synchronize()
