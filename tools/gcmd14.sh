#!/bin/bash
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q -k "fused_encode" 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python - <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2305_01024_b200 import ftgemm as F
for dt, (M, N, K) in [("bf16", (8192, 8192, 8192)), ("tf32", (8192, 8192, 8192)), ("bf16", (16384, 16384, 128)), ("bf16", (8192, 8192, 1024))]:
    odt = "bf16" if dt == "bf16" else "f32"
    A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
    B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
    C = torch.empty(M, N, dtype=A.dtype, device="cuda")
    g = F.FTGemm(dt, M, N, K)
    g.encode(A, B)
    def t(fn, n=20):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(n): fn()
        e1.record(); e1.synchronize()
        return e0.elapsed_time(e1) / n
    names = {"run": lambda: g.run(A, B, C), "run_fused": lambda: g.run(A, B, C, fuse_a=True),
             "step": lambda: (g.encode(A, B), g.run(A, B, C)),
             "step_fused": lambda: (g.encode(None, B, which=2), g.run(A, B, C, fuse_a=True)),
             "off": lambda: g.run(A, B, C, ft_level=F.FT_OFF)}
    res = {k: [] for k in names}
    for _ in range(3):
        for k, fn in names.items(): res[k].append(t(fn))
    print(dt, M, N, K, {k: round(sorted(v)[1], 4) for k, v in res.items()})
PY
