import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01024_b200 import ftgemm as F
M = N = K = 4096
A = synth.to_torch(synth.matrix(1, M, K, dtype="bf16"), "bf16").cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype="bf16"), "bf16").cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
g = F.FTGemm("bf16", M, N, K)
g.encode(None, B, which=2)
for _ in range(3):
    g.run(A, B, C, fuse_a=True)
torch.cuda.synchronize(); print("ok")
