"""Schedule-group / TMA L2-hint variants of the fused kernel, interleaved call by
call (development timing; never a bench number):
python tools/l2_sweep.py dtype M N K ft "G:HINT" ["G:HINT" ...]
G = FTGEMM_GROUP (0 = default), HINT = FTGEMM_L2HINT bits (A | B<<2 | C<<4).
The FTGEMM_L2HINT knob was removed from the kernel after this experiment
(profiles/r1b_l2_schedule.md); with the current library HINT has no effect."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_01024_b200 import ftgemm as F  # noqa: E402

dt, M, N, K, ft = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
variants = sys.argv[6:]
odt = "bf16" if dt == "bf16" else "f32"
A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
g = F.FTGemm(dt, M, N, K)
g.encode(A, B)


def setv(v):
    gs, h = v.split(":")
    if int(gs) > 0:
        os.environ["FTGEMM_GROUP"] = gs
    else:
        os.environ.pop("FTGEMM_GROUP", None)
    os.environ["FTGEMM_L2HINT"] = h


n = int(os.environ.get("NREP", "30"))
ev = {v: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
      for v in variants}
s = torch.cuda.current_stream()
for v in variants:
    setv(v)
    g.run(A, B, C, ft_level=ft)
torch.cuda.synchronize()
for j in range(n):
    for v in variants:
        setv(v)
        ev[v][j][0].record(s)
        g.run(A, B, C, ft_level=ft)
        ev[v][j][1].record(s)
torch.cuda.synchronize()
for v in variants:
    med = statistics.median(a.elapsed_time(b) for a, b in ev[v])
    print(json.dumps({"dt": dt, "M": M, "N": N, "K": K, "ft": ft, "variant": v, "ms": round(med, 4),
                      "tflops": round(2 * M * N * K / med / 1e9, 1)}), flush=True)
if os.environ.get("NCU_ONE"):
    pass
