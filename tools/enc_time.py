"""Time the encode kernels (A, B, both) at one shape, GPU-side (20 back-to-back
calls between two events, so host launch overhead is hidden), for each encode
variant: python tools/enc_time.py dtype M N K  (variants: builds with -DFTGEMM_*
selected through FTGEMM_LIB; the rows-per-block knob is compile-time since round 2)"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_01024_b200 import ftgemm as F  # noqa: E402

dt, M, N, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
tdt = torch.bfloat16 if dt == "bf16" else torch.float32
A = (torch.rand(M, K, device="cuda") * 2 - 1).to(tdt)
B = (torch.rand(K, N, device="cuda") * 2 - 1).to(tdt)
s = torch.cuda.current_stream()
elt = A.element_size()
VARIANTS = {"default": {}}
for vname, env in VARIANTS.items():
    for k in ("FTGEMM_ENC_B_ROWS",):
        os.environ.pop(k, None)
    os.environ.update(env)
    g = F.FTGemm(dt, M, N, K)   # the workspace size depends on the rows-per-block choice
    pl = g.plan
    out = {}
    for name, which in (("a", 1), ("b", 2), ("ab", 3)):
        fn = lambda: g.encode(A if which & 1 else None, B if which & 2 else None, which=which)  # noqa: E731
        for _ in range(3):
            fn()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20):
                fn()
            e1.record(s)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / 20)
        out[name] = best
    out["a_gbs"] = M * K * elt / out["a"] / 1e3
    out["b_gbs"] = (K * N * elt + K * pl.tiles_n * pl.bn * elt * (dt != "f32_simt")) / out["b"] / 1e3
    out["ab_gbs"] = (M * K * elt + K * N * elt + K * pl.tiles_n * pl.bn * elt * (dt != "f32_simt")) / out["ab"] / 1e3
    print(json.dumps({"variant": vname, "dtype": dt, "M": M, "N": N, "K": K,
                      **{k: round(v, 1) for k, v in out.items()}}), flush=True)

# reference points: torch's own streaming kernels on the same bytes
def _best(fn):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            fn()
        e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / 20)
    return best


Bc = torch.empty_like(B)
t_sum = _best(lambda: A.sum(dim=0))
t_cp = _best(lambda: Bc.copy_(B))
print(json.dumps({"ref": "torch", "dtype": dt, "colsum_A_us": round(t_sum, 1),
                  "colsum_A_gbs": round(M * K * elt / t_sum / 1e3, 1), "copy_B_us": round(t_cp, 1),
                  "copy_B_gbs": round(2 * K * N * elt / t_cp / 1e3, 1)}), flush=True)
