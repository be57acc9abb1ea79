"""Drive the hot path a few times for ncu (never used for timing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01024_b200 import ftgemm as F
dt = sys.argv[1] if len(sys.argv) > 1 else "bf16"
M = N = K = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
ft = int(sys.argv[3]) if len(sys.argv) > 3 else 2
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
odt = "bf16" if dt == "bf16" else "f32"
A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
g = F.FTGemm(dt, M, N, K)
for _ in range(reps):
    if ft:
        g.encode(A, B)
    g.run(A, B, C, ft_level=ft)
torch.cuda.synchronize()
print("ok", g.report()[0] if ft else "")
