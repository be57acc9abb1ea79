import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_01024_b200 import ftgemm as F
M = N = K = 8192
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / n
Ab = torch.randn(M, K + 64, device="cuda").to(torch.bfloat16)
Bb = torch.randn(K, N + 64, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for name, A, B in [("aligned", Ab[:, :K], Bb[:, :N]), ("B+8", Ab[:, :K], Bb[:, 8:8 + N]), ("A+8", Ab[:, 8:8 + K], Bb[:, :N]),
                   ("B+32", Ab[:, :K], Bb[:, 32:32 + N])]:
    ms = t(lambda: F.run("bf16", A, B, C, ft_level=0))
    print(json.dumps({"case": name, "ms": ms, "tflops": 2 * M * N * K / ms / 1e9}))
