"""Drive one tile class of the fused kernel for ncu: prof_cls.py dtype M N K ft bn cg"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01024_b200 import ftgemm as F
dt = sys.argv[1]; M, N, K, ft, bn, cg = map(int, sys.argv[2:8])
odt = "bf16" if dt == "bf16" else "f32"
A = synth.matrix_torch(1, M, K, dtype=odt); B = synth.matrix_torch(2, K, N, dtype=odt)
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
g = F.FTGemm(dt, M, N, K, tile=(bn, cg))
for _ in range(3):
    if ft: g.encode(A, B)
    g.run(A, B, C, ft_level=ft)
torch.cuda.synchronize(); print("ok")
