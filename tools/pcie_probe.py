"""PCIe copy-rate probe (development): pinned H2D / D2H of the cfg3 step's bytes
on one or two streams, alone and concurrently."""
import json
import torch

A = torch.empty(8192, 8192, dtype=torch.bfloat16).pin_memory()
B = torch.empty(8192, 8192, dtype=torch.bfloat16).pin_memory()
C = torch.empty(8192, 8192, dtype=torch.bfloat16).pin_memory()
Ad, Bd, Cd = (torch.empty(8192, 8192, dtype=torch.bfloat16, device="cuda") for _ in range(3))
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m = torch.cuda.current_stream()
    e0.record(m)
    for _ in range(n):
        ev = torch.cuda.Event(); ev.record(m)
        for s in (s1, s2, s3):
            s.wait_event(ev)
        fn()
        for s in (s1, s2, s3):
            e = torch.cuda.Event(); e.record(s); m.wait_event(e)
    e1.record(m); e1.synchronize()
    return e0.elapsed_time(e1) / n


def h2d_one():
    with torch.cuda.stream(s1):
        Ad.copy_(A, non_blocking=True); Bd.copy_(B, non_blocking=True)


def h2d_two():
    with torch.cuda.stream(s1):
        Ad.copy_(A, non_blocking=True)
    with torch.cuda.stream(s2):
        Bd.copy_(B, non_blocking=True)


def d2h():
    with torch.cuda.stream(s3):
        C.copy_(Cd, non_blocking=True)


def both_one():
    h2d_one(); d2h()


def both_two():
    h2d_two(); d2h()


res = {k: round(t(f), 3) for k, f in [("h2d_256MB_1stream", h2d_one), ("h2d_256MB_2streams", h2d_two),
                                      ("d2h_128MB", d2h), ("h2d1+d2h", both_one), ("h2d2+d2h", both_two)]}
res["h2d_GBs_1stream"] = round(2 * 2 ** 27 / res["h2d_256MB_1stream"] / 1e6, 1)
res["d2h_GBs"] = round(2 ** 27 / res["d2h_128MB"] / 1e6, 1)
print(json.dumps(res))
