"""Per-source-line warp-stall breakdown from an ncu report (source page).
    python tools/stall_reasons.py <rep.ncu-rep> [n]"""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; agg = []
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr) or not r[0]: continue
    d = dict(zip(hdr, r))
    try: s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    except ValueError: continue
    st = {k[6:]: int(v or 0) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k}
    agg.append((s, cur, r[0], r[1][:70], int(d["Instructions Executed"] or 0), st))
tot = sum(a[0] for a in agg)
print("total", tot)
for s, f, l, src, ie, st in sorted(agg, key=lambda a: -a[0])[:n]:
    top = ", ".join(f"{k}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:4] if v)
    print(f"{s:6d} {100*s/tot:5.1f}% {f}:{l} inst={ie} [{top}] {src}")
