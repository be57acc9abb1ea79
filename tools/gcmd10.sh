#!/bin/bash
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python - <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2305_01024_b200 import ftgemm as F
for dt in ("bf16", "tf32", "f32_simt"):
    odt = "bf16" if dt == "bf16" else "f32"
    M = N = K = 8192
    A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
    B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
    g = F.FTGemm(dt, M, N, K)
    def t(fn, n=20):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(n): fn()
        e1.record(); e1.synchronize()
        return e0.elapsed_time(e1) / n * 1e3
    both = t(lambda: g.encode(A, B)); a = t(lambda: g.encode(A, None, which=1)); b = t(lambda: g.encode(None, B, which=2))
    print(dt, f"encode both {both:.1f} us  A {a:.1f} us  B {b:.1f} us")
PY
