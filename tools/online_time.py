"""Online (per-K_s) verification against the end-of-K run, interleaved call by
call for one or more builds (development timing; never a bench number):
    LIBS=a.so,b.so python tools/online_time.py dtype M N K"""
import importlib.util
import json
import os
import random
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def load_binding(lib, i):
    os.environ["FTGEMM_LIB"] = lib
    spec = importlib.util.spec_from_file_location(f"ftgemm_o{i}", os.path.join(ROOT, "paper_2305_01024_b200", "ftgemm.py"))
    m = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = m
    spec.loader.exec_module(m)
    return m


LIBS = [x for x in os.environ.get("LIBS", os.path.join(ROOT, "paper_2305_01024_b200", "libftgemm.so")).split(",") if x]
dt, M, N, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
odt = "bf16" if dt == "bf16" else "f32"
A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
fns, gs = {}, {}
for i, lib in enumerate(LIBS):
    Fv = load_binding(lib, i)
    g = Fv.FTGemm(dt, M, N, K)
    g.encode(A, B)
    nm = os.path.basename(lib)
    gs[nm] = g
    fns[nm + ":run"] = (lambda g=g: g.run(A, B, C))
    fns[nm + ":ks256"] = (lambda g=g: g.run_online(A, B, C, ks=256))
    fns[nm + ":ks2048"] = (lambda g=g: g.run_online(A, B, C, ks=2048))
n = int(os.environ.get("NREP", "20"))
for f in fns.values():
    f()
torch.cuda.synchronize()
s = torch.cuda.current_stream()
ev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)] for k in fns}
rng = random.Random(5)
for j in range(n):
    order = list(fns)
    rng.shuffle(order)
    for k in order:
        ev[k][j][0].record(s)
        fns[k]()
        ev[k][j][1].record(s)
torch.cuda.synchronize()
res = {k: round(statistics.median(a.elapsed_time(b) for a, b in ev[k]), 4) for k in fns}
print(json.dumps({"dt": dt, "M": M, "N": N, "K": K, "ms": res,
                  "detected": {nm: int(g.report()[0]["tiles_detected"]) for nm, g in gs.items()}}))
