"""Shape sweep for BASELINE configs 2 and 4 (measurement rows of SURVEY §8(d)).

    python tools/sweep.py [--out profiles/sweep_r1.json] [--quick]

For each (dtype, M, N, K): FT-on step (encode + run, CORRECT level, no faults),
FT-on run alone, FT-off run, cuBLAS (torch.matmul; FP32 with TF32 disabled for
the SIMT rows, TF32 enabled for the TF32 rows, BF16), encode alone; TFLOPS
(2MNK / t) and the fraction of the relevant measured peak (MEASURED_PEAKS.json:
BF16 burst; TF32 = BF16 / 2 (nominal ratio); FP32 SIMT = 148 SM x 128 FMA x 2 x
1.965 GHz = 74.4 TFLOP/s).  Inputs U[-1,1); times are medians of 3 interleaved
rounds of CUDA-event-timed loops.  HBM-bound shapes also report GB/s.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2305_01024_b200 import ftgemm as F  # noqa: E402


_FLUSH = None
FLUSH_BELOW = 256 << 20          # operand sets below 2x the 126 MB L2: flush L2 between calls


def timeit(fn, reps, flush=False):
    """ms per call.  flush: an L2-sized buffer is rewritten before every call and
    only the call itself is timed (per-call events), so small operand sets are
    read from HBM as in a cold-cache call (SURVEY 8(d) timing rule)."""
    global _FLUSH
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    if flush:
        if _FLUSH is None:
            _FLUSH = torch.empty(FLUSH_BELOW, dtype=torch.uint8, device="cuda")
        evs = []
        for _ in range(reps):
            _FLUSH.fill_(1)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in evs)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def measure_batched(dt, M, N, K, batch):
    """One persistent launch over the batch (ftgemm_run_batched) vs torch.bmm."""
    odt = "bf16" if dt == "bf16" else "f32"
    A = torch.stack([synth.matrix_torch(synth.BASE_SEED + b, M, K, dtype=odt) for b in range(batch)])
    B = torch.stack([synth.matrix_torch(synth.BASE_SEED + 100 + b, K, N, dtype=odt) for b in range(batch)])
    C = torch.empty(batch, M, N, dtype=A.dtype, device="cuda")
    g = F.FTGemmBatched(dt, batch, M, N, K)
    flops = 2.0 * M * N * K * batch
    reps = max(3, min(200, int(2e10 / flops) + 1))
    torch.backends.cuda.matmul.allow_tf32 = dt == "tf32"
    cfg = {"ft_step": lambda: (g.encode(A, B), g.run(A, B, C)), "ft_run": lambda: g.run(A, B, C),
           "ft_off": lambda: g.run(A, B, C, ft_level=F.FT_OFF), "encode": lambda: g.encode(A, B),
           "cublas": lambda: torch.bmm(A, B, out=C),
           "detect_rows_run": lambda: g.run(A, B, C, ft_level=F.FT_DETECT_ROWS)}
    g.encode(A, B)
    samp = {k: [] for k in cfg}
    fl = batch * (M * K + K * N + M * N) * A.element_size() < FLUSH_BELOW
    for _ in range(3):
        for k, fn in cfg.items():
            samp[k].append(timeit(fn, reps, fl))
    med = {k: statistics.median(v) for k, v in samp.items()}
    counts, _ = g.report(0)
    assert counts["tiles_detected"] == 0, counts
    peak = {"bf16": PEAK_BF16, "tf32": PEAK_BF16 / 2, "f32_simt": 74.4}[dt]
    out = {"dtype": dt, "M": M, "N": N, "K": K, "batch": batch, "reps": reps, "launch": "one batched launch",
           "check_tile": [g.plan.check_tile_m, g.plan.check_tile_n], "mma_tile": [g.plan.bm, g.plan.bn, g.plan.bk]}
    for k, v in med.items():
        out[f"{k}_ms"] = v
        if k != "encode":
            out[f"{k}_tflops"] = flops / (v * 1e-3) / 1e12
    out["ft_step_frac_of_peak"] = out["ft_step_tflops"] / peak
    out["ft_run_frac_of_peak"] = out["ft_run_tflops"] / peak
    out["ft_off_frac_of_peak"] = out["ft_off_tflops"] / peak
    out["overhead_step_vs_ft_off_pct"] = 100 * (med["ft_step"] - med["ft_off"]) / med["ft_off"]
    out["overhead_run_vs_ft_off_pct"] = 100 * (med["ft_run"] - med["ft_off"]) / med["ft_off"]
    out["overhead_step_vs_cublas_pct"] = 100 * (med["ft_step"] - med["cublas"]) / med["cublas"]
    out["ft_run_io_gbs"] = batch * (M * K + K * N + M * N) * A.element_size() / (med["ft_run"] * 1e-3) / 1e9
    out["peak_tflops"] = peak
    return out


def measure(dt, M, N, K, batch=1):
    if batch > 1 and dt != "f32_simt":
        return measure_batched(dt, M, N, K, batch)
    odt = "bf16" if dt == "bf16" else "f32"
    A = synth.to_torch(synth.matrix(synth.BASE_SEED, M, K, dtype=odt), odt).cuda()
    B = synth.to_torch(synth.matrix(synth.BASE_SEED + 1, K, N, dtype=odt), odt).cuda()
    C = torch.empty(M, N, dtype=A.dtype, device="cuda")
    g = F.FTGemm(dt, M, N, K)
    flops = 2.0 * M * N * K
    reps = max(3, min(200, int(2e10 / flops) + 1))
    torch.backends.cuda.matmul.allow_tf32 = dt == "tf32"

    def step():
        g.encode(A, B)
        g.run(A, B, C)
    cfg = {"ft_step": step, "ft_run": lambda: g.run(A, B, C), "ft_off": lambda: g.run(A, B, C, ft_level=F.FT_OFF),
           "encode": lambda: g.encode(A, B), "cublas": lambda: torch.matmul(A, B, out=C),
           "detect_rows_run": lambda: g.run(A, B, C, ft_level=F.FT_DETECT_ROWS)}
    if dt != "tf32":                     # the non-fused baseline (paper's comparison scheme)
        def nf_step():
            g.encode(A, B, which=3 | 4)
            g.run_nonfused(A, B, C)
        cfg["nonfused_step"] = nf_step
    g.encode(A, B)
    samp = {k: [] for k in cfg}
    if "nonfused_step" in cfg:
        nf_step()
        g.encode(A, B)
    fl = (M * K + K * N + M * N) * A.element_size() < FLUSH_BELOW
    for _ in range(3):
        for k, fn in cfg.items():
            samp[k].append(timeit(fn, reps, fl))
    med = {k: statistics.median(v) * batch for k, v in samp.items()}
    counts, _ = g.report(0)
    assert counts["tiles_detected"] == 0, counts
    el = A.element_size()
    peak = {"bf16": PEAK_BF16, "tf32": PEAK_BF16 / 2, "f32_simt": 74.4}[dt]
    io_bytes = (M * K + K * N + M * N) * el
    out = {"dtype": dt, "M": M, "N": N, "K": K, "batch": batch, "reps": reps, "l2_flushed": bool(fl),
           "check_tile": [g.plan.check_tile_m, g.plan.check_tile_n], "mma_tile": [g.plan.bm, g.plan.bn, g.plan.bk]}
    for k, v in med.items():
        out[f"{k}_ms"] = v
        if k != "encode":
            out[f"{k}_tflops"] = batch * flops / (v * 1e-3) / 1e12
    out["ft_step_frac_of_peak"] = out["ft_step_tflops"] / peak
    out["ft_run_frac_of_peak"] = out["ft_run_tflops"] / peak
    out["ft_off_frac_of_peak"] = out["ft_off_tflops"] / peak
    out["overhead_step_vs_ft_off_pct"] = 100 * (med["ft_step"] - med["ft_off"]) / med["ft_off"]
    out["overhead_run_vs_ft_off_pct"] = 100 * (med["ft_run"] - med["ft_off"]) / med["ft_off"]
    out["overhead_step_vs_cublas_pct"] = 100 * (med["ft_step"] - med["cublas"]) / med["cublas"]
    if "nonfused_step" in med:
        out["fused_speedup_vs_nonfused_pct"] = 100 * (med["nonfused_step"] - med["ft_step"]) / med["ft_step"]
    out["ft_run_io_gbs"] = batch * io_bytes / (med["ft_run"] * 1e-3) / 1e9
    out["peak_tflops"] = peak
    return out


PEAK_BF16 = 1712.3


def main():
    global PEAK_BF16
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweep_r1.json"))
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        PEAK_BF16 = json.load(open(pk))["bf16_tflops"]
    rows = []
    cfg2 = [1024, 2048, 4096, 8192] if args.quick else [1024, 2048, 3072, 4096, 6144, 8192]
    for dt in ("f32_simt", "tf32"):
        for s in cfg2:
            rows.append(("cfg2", dt, s, s, s, 1))
        for s in (2048, 4096, 8192):
            rows.append(("cfg2-K1024", dt, s, s, 1024, 1))
    for s in cfg2:
        rows.append(("square-bf16", "bf16", s, s, s, 1))
    for dt in ("bf16", "tf32"):
        for (M, N, K) in [(16384, 16384, 128), (128, 16384, 16384), (16384, 128, 16384)]:
            rows.append(("cfg4", dt, M, N, K, 1))
        rows.append(("cfg4-batch32", dt, 4096, 128, 4096, 32))
    for s in (64, 160, 256, 480):
        rows.append(("paper-K256", "bf16", s, s, 256, 1))
    out = []
    for tag, dt, M, N, K, batch in rows:
        try:
            r = measure(dt, M, N, K, batch)
            r["config"] = tag
            out.append(r)
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
        except Exception as e:  # keep sweeping, record the failure
            out.append({"config": tag, "dtype": dt, "M": M, "N": N, "K": K, "error": str(e)})
            print("ERROR", tag, dt, M, N, K, e, flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"gpu": torch.cuda.get_device_name(0), "peak_bf16_tflops": PEAK_BF16, "rows": out},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
