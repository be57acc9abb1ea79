import csv, subprocess, sys, collections
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = None; agg = collections.Counter(); text = {}
hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; i_s = r.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) < len(hdr): continue
    try:
        line = int(r[0]); s = int(r[i_s] or 0)
    except ValueError:
        continue
    agg[(cur_file, line)] += s
    text[(cur_file, line)] = r[1][:90]
tot = sum(agg.values()); print("total", tot)
for (f, l), s in agg.most_common(n): print(f"{s:6d} {100*s/tot:5.1f}% {f}:{l} {text[(f,l)]}")
