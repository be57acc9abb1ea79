import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01024_b200 import ftgemm as F
dt = sys.argv[1]; M, N, K = map(int, sys.argv[2:5]); ft = int(sys.argv[5])
odt = "bf16" if dt == "bf16" else "f32"
A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
g = F.FTGemm(dt, M, N, K)
for _ in range(3):
    if ft: g.encode(A, B)
    g.run(A, B, C, ft_level=ft)
torch.cuda.synchronize(); print("ok")
