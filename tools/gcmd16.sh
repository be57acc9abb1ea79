#!/bin/bash
export PYTHONUNBUFFERED=1
timeout 300 python - <<'PY'
import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import torch, synth, importlib
def bench(lib, dt, M, N, K, ft):
    os.environ["FTGEMM_LIB"] = lib
    from paper_2305_01024_b200 import ftgemm as F
    importlib.reload(F)
    odt = "bf16" if dt == "bf16" else "f32"
    A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
    B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
    C = torch.empty(M, N, dtype=A.dtype, device="cuda")
    g = F.FTGemm(dt, M, N, K); g.encode(A, B)
    return g, (lambda: g.run(A, B, C, ft_level=ft))
cases = {"ft8192": ("paper_2305_01024_b200/libftgemm.so", "bf16", 8192, 8192, 8192, 2),
         "nover8192": ("paper_2305_01024_b200/libftgemm_no_verify.so", "bf16", 8192, 8192, 8192, 2),
         "off8192": ("paper_2305_01024_b200/libftgemm.so", "bf16", 8192, 8192, 8192, 0),
         "off8448": ("paper_2305_01024_b200/libftgemm.so", "bf16", 8448, 8448, 8192, 0)}
fns = {}
for k, v in cases.items():
    g, fn = bench(*v); fns[k] = (g, fn)
# interleave per call
ev = {k: [] for k in fns}
for k, (g, fn) in fns.items():
    for _ in range(3): fn()
torch.cuda.synchronize()
for i in range(40):
    for k, (g, fn) in fns.items():
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); ev[k].append((e0, e1))
torch.cuda.synchronize()
import statistics
for k in fns:
    print(k, round(statistics.median(a.elapsed_time(b) for a, b in ev[k]), 4))
PY
