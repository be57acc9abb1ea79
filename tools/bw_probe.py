"""Read-bandwidth calibration for the encode kernels (development)."""
import torch, time
A = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
A32 = torch.randn(8192, 8192, device="cuda")
out = torch.empty(8192, device="cuda")
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / n
for name, fn, by in [("bf16 sum", lambda: A.sum(), A.numel() * 2), ("bf16 colsum", lambda: A.sum(dim=0), A.numel() * 2),
                     ("bf16 rowsum", lambda: A.float().sum(dim=1) if False else A.sum(dim=1), A.numel() * 2),
                     ("f32 sum", lambda: A32.sum(), A32.numel() * 4), ("bf16 copy", lambda: A.clone(), A.numel() * 4),
                     ("f32 copy", lambda: A32.clone(), A32.numel() * 8)]:
    ms = t(fn)
    print(f"{name:12s} {ms*1e3:8.1f} us  {by / ms / 1e6:8.0f} GB/s")
