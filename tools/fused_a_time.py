"""In-kernel A encode (ftgemm_run_fused) against the separate encode, interleaved
call by call (development timing; never a bench number):
    python tools/fused_a_time.py dtype M N K [M N K ...]
step    = encode A + B (one launch) + ftgemm_run
step_fa = encode B + ftgemm_run_fused
run / run_fa = the GEMM alone with B (and A) pre-encoded; off = FT off.
Also checks run_fused's C against run's C bitwise and the fault-free counts."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import importlib.util  # noqa: E402


def load_binding(lib, i):
    """one private copy of the binding module per library (its own ctypes handle)"""
    os.environ["FTGEMM_LIB"] = lib
    spec = importlib.util.spec_from_file_location(f"ftgemm_v{i}", os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2305_01024_b200", "ftgemm.py"))
    m = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = m
    spec.loader.exec_module(m)
    return m


LIBS = [x for x in os.environ.get("LIBS", "").split(",") if x]
if LIBS:
    VARIANTS = [(os.path.basename(x), load_binding(x, i)) for i, x in enumerate(LIBS)]
else:
    from paper_2305_01024_b200 import ftgemm as F0  # noqa: E402
    VARIANTS = [("", F0)]
F = VARIANTS[0][1]

dt = sys.argv[1]
shapes = [tuple(int(x) for x in sys.argv[i:i + 3]) for i in range(2, len(sys.argv), 3)]
odt = "bf16" if dt == "bf16" else "f32"
n = int(os.environ.get("NREP", "30"))
for M, N, K in shapes:
    A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
    B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
    C = torch.empty(M, N, dtype=A.dtype, device="cuda")
    C2 = torch.empty(M, N, dtype=A.dtype, device="cuda")
    g = F.FTGemm(dt, M, N, K)
    g2 = F.FTGemm(dt, M, N, K)
    g.encode(A, B)
    g2.encode(None, B, which=2)
    g.run(A, B, C)
    g2.run(A, B, C2, fuse_a=True)
    torch.cuda.synchronize()
    same = bool((C == C2).all())
    c1, _ = g.report()
    c2, _ = g2.report()
    fns = {
        "step": lambda: (g.encode(A, B), g.run(A, B, C)),
        "step_fa": lambda: (g2.encode(None, B, which=2), g2.run(A, B, C2, fuse_a=True)),
        "run": lambda: g.run(A, B, C),
        "run_fa": lambda: g2.run(A, B, C2, fuse_a=True),
        "off": lambda: g.run(A, B, C, ft_level=F.FT_OFF),
        "encode_b": lambda: g2.encode(None, B, which=2),
    }
    for name, Fv in VARIANTS[1:]:
        gv = Fv.FTGemm(dt, M, N, K)
        gv.encode(None, B, which=2)
        fns["run_fa:" + name] = (lambda gv=gv: gv.run(A, B, C2, fuse_a=True))
        if os.environ.get("VSTEP"):
            gw = Fv.FTGemm(dt, M, N, K)
            fns["step:" + name] = (lambda gw=gw: (gw.encode(A, B), gw.run(A, B, C)))
            fns["encode:" + name] = (lambda gw=gw: gw.encode(A, B))
    s = torch.cuda.current_stream()
    ev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
          for k in fns}
    for f in fns.values():
        f()
    torch.cuda.synchronize()
    import random
    rng = random.Random(7)
    for j in range(n):
        order = list(fns)
        rng.shuffle(order)
        for k in order:
            ev[k][j][0].record(s)
            fns[k]()
            ev[k][j][1].record(s)
    torch.cuda.synchronize()
    res = {k: round(statistics.median(a.elapsed_time(b) for a, b in ev[k]), 4) for k in fns}
    c2b, _ = g2.report()
    print(json.dumps({"dt": dt, "M": M, "N": N, "K": K, "ms": res, "C_fused_eq_run": same,
                      "det_run": int(c1["tiles_detected"]), "det_fused": int(c2["tiles_detected"]),
                      "det_fused_timed": int(c2b["tiles_detected"]), "checked_fused": int(c2["tiles_checked"]),
                      "max_ratio_fused": float(c2b["max_resid_ratio"]) if "max_resid_ratio" in c2b.keys() else None}),
          flush=True)
