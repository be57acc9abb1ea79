"""Tile-class variants (explicit FTGEMM_TILE(bn, cta_group) codes) of the FT run at one shape,
interleaved call by call (development timing; never a bench number):
python tools/bn_sweep.py dtype M N K  "BN:CG" ["BN:CG" ...]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_01024_b200 import ftgemm as F  # noqa: E402

dt, M, N, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
variants = sys.argv[5:]
odt = "bf16" if dt == "bf16" else "f32"
A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
gs = {}
for v in variants:
    bn, cg = v.split(":")
    g = F.FTGemm(dt, M, N, K, tile=(int(bn), int(cg)))
    g.encode(A, B)
    gs[v] = g
n = int(os.environ.get("NREP", "30"))
s = torch.cuda.current_stream()
ev = {v: [] for v in variants}
for j in range(n + 2):
    for v, g in gs.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.run(A, B, C, ft_level=F.FT_CORRECT)
        e1.record(s)
        if j >= 2:
            ev[v].append((e0, e1))
torch.cuda.synchronize()
for v, g in gs.items():
    med = statistics.median(a.elapsed_time(b) for a, b in ev[v])
    p = g.plan
    print(json.dumps({"dt": dt, "M": M, "N": N, "K": K, "bn:cg": v, "plan_bn": p.bn, "plan_cg": p.cta_group,
                      "ms": round(med, 4), "tflops": round(2 * M * N * K / med / 1e9, 1),
                      "detected": g.report()[0]["tiles_detected"]}), flush=True)
