"""Sustained back-to-back runs of FT and FT-off (and cuBLAS) with nvidia-smi
sampling of SM clock and board power during each block (development; never a
bench number): python tools/power_probe.py [dtype] [n]"""
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_01024_b200 import ftgemm as F  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "bf16"
M = N = K = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
odt = "bf16" if dt == "bf16" else "f32"
A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
g = F.FTGemm(dt, M, N, K)
g.encode(A, B)


def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True).stdout.strip()
        try:
            c, p, t, th = [x.strip() for x in r.split(",")]
            out.append((float(c), float(p), float(t), th))
        except ValueError:
            pass
        time.sleep(0.05)


fns = {"ft": lambda: g.run(A, B, C, ft_level=F.FT_CORRECT), "off": lambda: g.run(A, B, C, ft_level=F.FT_OFF),
       "cublas": lambda: torch.matmul(A, B, out=C)}
s = torch.cuda.current_stream()
for rnd in range(2):
    for name, f in fns.items():
        for _ in range(50):
            f()
        torch.cuda.synchronize()
        stop, smp = threading.Event(), []
        th = threading.Thread(target=sample, args=(stop, smp))
        th.start()
        times = []
        t_end = time.time() + 3.0
        while time.time() < t_end:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20):
                f()
            e1.record(s)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 20)
        stop.set()
        th.join()
        clk = statistics.median(x[0] for x in smp) if smp else None
        pw = statistics.median(x[1] for x in smp) if smp else None
        print(json.dumps({"round": rnd, "what": name, "ms_median": round(statistics.median(times), 4),
                          "ms_first": round(times[0], 4), "ms_last": round(times[-1], 4), "n": len(times),
                          "sm_mhz_median": clk, "power_w_median": pw,
                          "temp_max": max((x[2] for x in smp), default=None),
                          "throttle": sorted(set(x[3] for x in smp))}), flush=True)
