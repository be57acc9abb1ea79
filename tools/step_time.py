"""Per-call step timing (encode + fused run), run only and encode only, for one
or more library builds, interleaved call by call (development timing; never a
bench number): python tools/step_time.py dtype M N K lib1.so [lib2.so ...]"""
import ctypes
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

dt, M, N, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
libs = sys.argv[5:]
odt = "bf16" if dt == "bf16" else "f32"
A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
import importlib.util  # noqa: E402
gs = []
for i, lib in enumerate(libs):
    # one private copy of the binding module per library (its own ctypes handle)
    os.environ["FTGEMM_LIB"] = lib
    spec = importlib.util.spec_from_file_location(f"ftgemm_v{i}", os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2305_01024_b200", "ftgemm.py"))
    F = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = F
    spec.loader.exec_module(F)
    g = F.FTGemm(dt, M, N, K)
    gs.append((lib, F, g))
n = int(os.environ.get("NREP", "40"))
s = torch.cuda.current_stream()
fns = {}
for lib, F, g in gs:
    name = os.path.basename(lib)
    fns[name + ":step"] = (lambda g=g, F=F: (g.encode(A, B), g.run(A, B, C, ft_level=F.FT_CORRECT)))
    fns[name + ":run"] = (lambda g=g, F=F: g.run(A, B, C, ft_level=F.FT_CORRECT))
    fns[name + ":encode"] = (lambda g=g: g.encode(A, B))
    fns[name + ":off"] = (lambda g=g, F=F: g.run(A, B, C, ft_level=F.FT_OFF))
ev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)] for k in fns}
for f in fns.values():
    f()
torch.cuda.synchronize()
for j in range(n):
    for k, f in fns.items():
        ev[k][j][0].record(s)
        f()
        ev[k][j][1].record(s)
torch.cuda.synchronize()
for k in fns:
    med = statistics.median(a.elapsed_time(b) for a, b in ev[k])
    print(json.dumps({"dt": dt, "M": M, "N": N, "K": K, "what": k, "ms": round(med, 4)}), flush=True)
for lib, F, g in gs:
    print(os.path.basename(lib), g.report()[0])
