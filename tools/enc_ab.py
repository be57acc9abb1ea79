"""Encode A / B / both for several library builds, interleaved call by call
(development timing; never a bench number):
    LIBS=a.so,b.so python tools/enc_ab.py dtype M N K [M N K ...]
Per call: the encode launch (+ its ticket memsets) between two CUDA events.
Also the B^r operand and the split rows of the builds compared bytewise."""
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
    spec = importlib.util.spec_from_file_location(f"ftgemm_e{i}", os.path.join(ROOT, "paper_2305_01024_b200", "ftgemm.py"))
    m = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = m
    spec.loader.exec_module(m)
    return m


LIBS = [x for x in os.environ.get("LIBS", os.path.join(ROOT, "paper_2305_01024_b200", "libftgemm.so")).split(",") if x]
VS = [(os.path.basename(x), load_binding(x, i)) for i, x in enumerate(LIBS)]
dt = sys.argv[1]
shapes = [tuple(int(x) for x in sys.argv[i:i + 3]) for i in range(2, len(sys.argv), 3)]
odt = "bf16" if dt == "bf16" else "f32"
n = int(os.environ.get("NREP", "30"))
for M, N, K in shapes:
    A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
    B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
    gs = {name: Fv.FTGemm(dt, M, N, K) for name, Fv in VS}
    fns = {}
    for name, g in gs.items():
        fns[name + ":a"] = (lambda g=g: g.encode(A, None, which=1))
        fns[name + ":b"] = (lambda g=g: g.encode(None, B, which=2))
        fns[name + ":ab"] = (lambda g=g: g.encode(A, B))
    for f in fns.values():
        f()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    ev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)] for k in fns}
    rng = random.Random(3)
    for j in range(n):
        order = list(fns)
        rng.shuffle(order)
        for k in order:
            ev[k][j][0].record(s)
            fns[k]()
            ev[k][j][1].record(s)
    torch.cuda.synchronize()
    res = {k: round(statistics.median(a.elapsed_time(b) for a, b in ev[k]) * 1e3, 1) for k in fns}
    first = next(iter(gs.values()))
    pl = first.plan
    elt = A.element_size()
    bytes_ab = M * K * elt + K * N * elt + (K * pl.tiles_n * pl.bn * elt if dt != "f32_simt" else 0)
    same = {}
    fnames = list(gs)
    for name, Fv in VS[1:]:
        g = gs[name]
        L0, L1 = VS[0][1].encode_layout(dt, M, N, K), Fv.encode_layout(dt, M, N, K)
        nbt = L0["kp"] * L0["bt_ld"] * elt
        ny = pl.tiles_m * ((K + pl.bk - 1) // pl.bk) * 384
        bt0 = first.enc_ws[L0["bt"]:L0["bt"] + nbt]
        bt1 = g.enc_ws[L1["bt"]:L1["bt"] + nbt]
        y0 = first.enc_ws[L0["y"]:L0["y"] + ny]
        y1 = g.enc_ws[L1["y"]:L1["y"] + ny]
        same[name] = {"bt_equal": bool(torch.equal(bt0, bt1)), "y_equal": bool(torch.equal(y0, y1))}
    print(json.dumps({"dt": dt, "M": M, "N": N, "K": K, "us": res,
                      "ab_TBps": {nm: round(bytes_ab / res[nm + ":ab"] / 1e6, 2) for nm in gs}, "cmp": same}), flush=True)
