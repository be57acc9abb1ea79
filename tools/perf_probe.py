"""Time ftgemm_run variants (development; never a bench number)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01024_b200 import ftgemm as F
dt = sys.argv[1]; M, N, K = map(int, sys.argv[2:5]); ft = int(sys.argv[5])
odt = "bf16" if dt == "bf16" else "f32"
A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
g = F.FTGemm(dt, M, N, K)
g.encode(A, B)
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / n
ms = t(lambda: g.run(A, B, C, ft_level=ft))
out = {"dt": dt, "M": M, "N": N, "K": K, "ft": ft, "ms": ms, "tflops": 2 * M * N * K / ms / 1e9}
if ft:
    ea = t(lambda: g.encode(A, None, which=1)); eb = t(lambda: g.encode(None, B, which=2))
    el = A.element_size()
    out.update(enc_a_ms=ea, enc_a_gbs=M * K * el / ea / 1e6, enc_b_ms=eb,
               enc_b_gbs=(K * N * el + g.plan.tiles_n * g.plan.bn * K * el) / eb / 1e6)
print(json.dumps(out))
