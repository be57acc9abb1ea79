"""Drive the in-kernel A encode (ftgemm_run_fused) under ncu: python tools/prof_fused.py [M N K]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
from paper_2305_01024_b200 import ftgemm as F  # noqa: E402
M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (8192, 8192, 8192)
A = synth.to_torch(synth.matrix(1, M, K, dtype="bf16"), "bf16").cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype="bf16"), "bf16").cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
g = F.FTGemm("bf16", M, N, K)
g.encode(None, B, which=2)
for _ in range(3):
    g.run(A, B, C, fuse_a=True)
torch.cuda.synchronize()
print("ok", g.report()[0]["tiles_detected"])
