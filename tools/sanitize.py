"""Run every kernel class once on a small problem (<= 512^3) with faults, for
compute-sanitizer (memcheck / racecheck / synccheck): tools/g_sanitize.sh."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2305_01024_b200 import ftgemm as F  # noqa: E402

cases = [("f32_simt", None), ("bf16", (256, 2)), ("bf16", (256, 1)), ("bf16", (128, 1)), ("bf16", (128, 2)),
         ("tf32", (256, 2)), ("tf32", (256, 1)), ("tf32", (128, 1)), ("tf32", (128, 2))]
M, N, K = 500, 504, 320
for dt, tile in cases:
    odt = "bf16" if dt == "bf16" else "f32"
    A, B, Cin = (synth.to_torch(x, odt).cuda() for x in synth.problem(M, N, K, dtype=odt))
    g = F.FTGemm(dt, M, N, K, tile=tile)
    p = g.plan
    inj = [(3, 5, 100, 30, F.INJ_FLIP, 0, 0.0), (p.check_tile_m + 1, p.check_tile_n + 2, 7, 0, F.INJ_ADD, 0, 50.0)]
    C = Cin.clone()
    g.encode(A, B)
    g.run(A, B, C, alpha=1.5, beta=0.5, injections=inj)
    g.run(A, B, C, ft_level=F.FT_OFF)
    if dt != "f32_simt":
        g.run_online(A, B, C, ks=p.bk * 2, injections=inj)
        g.run(A, B, C, fuse_a=True)
    g.run(A, B, C, ft_level=F.FT_DETECT_ROWS)
    cnt, _ = g.report()
    torch.cuda.synchronize()
    print(dt, tile, "corrected", cnt["corrected"], flush=True)
nf = F.FTGemm("bf16", M, N, K)
A, B, _ = (synth.to_torch(x, "bf16").cuda() for x in synth.problem(M, N, K, dtype="bf16"))
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
nf.encode(A, B, which=3 | 4)
nf.run_nonfused(A, B, C, injections=[(3, 5, 0, 30, F.INJ_FLIP, 0, 0.0)])
torch.cuda.synchronize()
print("nonfused ok", nf.report()[0]["corrected"])
