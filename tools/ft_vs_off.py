"""FT run vs FT off (same kernel family) and cuBLAS, interleaved call by call,
median of N calls each (development timing; never a bench number):
python tools/ft_vs_off.py dtype M N K [dtype M N K ...]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_01024_b200 import ftgemm as F  # noqa: E402

args = sys.argv[1:]
for i in range(0, len(args), 4):
    dt, M, N, K = args[i], int(args[i + 1]), int(args[i + 2]), int(args[i + 3])
    odt = "bf16" if dt == "bf16" else "f32"
    A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
    B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
    C = torch.empty(M, N, dtype=A.dtype, device="cuda")
    g = F.FTGemm(dt, M, N, K)
    g.encode(A, B)
    fns = {"ft": lambda: g.run(A, B, C, ft_level=F.FT_CORRECT), "off": lambda: g.run(A, B, C, ft_level=F.FT_OFF),
           "cublas": lambda: torch.matmul(A, B, out=C), "encode": lambda: g.encode(A, B)}
    n = 30
    ev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
          for k in fns}
    for f in fns.values():
        f()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    for j in range(n):
        for k, f in fns.items():
            ev[k][j][0].record(s)
            f()
            ev[k][j][1].record(s)
    torch.cuda.synchronize()
    med = {k: statistics.median(a.elapsed_time(b) for a, b in v) for k, v in ev.items()}
    cnt, _ = g.report()
    print(json.dumps({"dt": dt, "M": M, "N": N, "K": K, **{k + "_ms": round(v, 4) for k, v in med.items()},
                      "ft/off": round(med["ft"] / med["off"], 3), "tflops_ft": round(2 * M * N * K / med["ft"] / 1e9, 1),
                      "detected": cnt["tiles_detected"]}), flush=True)
