"""Render a tools/sweep.py JSON into a markdown table (profiles/<tag>_sweep.md)."""
import json, sys
src, dst = sys.argv[1], sys.argv[2]
d = json.load(open(src))
peak = d.get("peak_bf16_tflops")
L = [f"# Shape sweep ({d.get('gpu')}) — medians of 3 interleaved rounds, CUDA events", "",
     "step = encode + FT run; run = FT run alone (CORRECT, no faults); off = same kernel family FT compiled out;",
     "rows = offline detect-only (row checks); nf = non-fused baseline step (encode + cuBLAS GEMMs + verify kernel).",
     f"TFLOPS = 2MNK / t.  Peaks: BF16 {peak} (measured burst), TF32 = BF16/2, FP32 SIMT 74.4.",
     "Rows whose operands total < 256 MB (2x L2) are timed call by call with an L2 flush before every call;",
     "larger ones back to back (their operands exceed L2).", "",
     "| cfg | dtype | M | N | K | step ms | run ms | off ms | cuBLAS ms | rows ms | nf step ms | run TFLOPS | run / off | step vs nf |",
     "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for r in d["rows"]:
    if "error" in r:
        L.append(f"| {r['config']} | {r['dtype']} | {r['M']} | {r['N']} | {r['K']} | error: {r['error'][:60]} |"); continue
    nf = r.get("nonfused_step_ms")
    L.append(f"| {r['config']} | {r['dtype']} | {r['M']} | {r['N']} | {r['K']} | {r['ft_step_ms']:.4f} | {r['ft_run_ms']:.4f} | "
             f"{r['ft_off_ms']:.4f} | {r['cublas_ms']:.4f} | {r.get('detect_rows_run_ms', float('nan')):.4f} | "
             f"{nf:.4f} | " if nf else f"| {r['config']} | {r['dtype']} | {r['M']} | {r['N']} | {r['K']} | {r['ft_step_ms']:.4f} | {r['ft_run_ms']:.4f} | "
             f"{r['ft_off_ms']:.4f} | {r['cublas_ms']:.4f} | {r.get('detect_rows_run_ms', float('nan')):.4f} | — | ")
    L[-1] += (f"{r['ft_run_tflops']:.1f} | {r['ft_run_ms'] / r['ft_off_ms']:.3f} | "
              + (f"{r['fused_speedup_vs_nonfused_pct']:+.1f}% |" if nf else "— |"))
open(dst, "w").write("\n".join(L) + "\n")
print("wrote", dst)
