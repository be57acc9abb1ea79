"""One configuration, median of per-call CUDA-event times (development)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2305_01024_b200 import ftgemm as F
dt = sys.argv[1]; M, N, K = map(int, sys.argv[2:5]); ft = int(sys.argv[5]); tag = sys.argv[6] if len(sys.argv) > 6 else ""
odt = "bf16" if dt == "bf16" else "f32"
A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
g = F.FTGemm(dt, M, N, K); g.encode(A, B)
fn = lambda: g.run(A, B, C, ft_level=ft)
for _ in range(5): fn()
torch.cuda.synchronize()
ev = []
for _ in range(40):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); ev.append((e0, e1))
torch.cuda.synchronize()
print(tag, dt, M, N, K, ft, round(statistics.median(a.elapsed_time(b) for a, b in ev), 4))
