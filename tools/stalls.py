import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
i_src = hdr.index("Source"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for k, r in enumerate(rows[2:]):
    try: data.append((int(r[i_s] or 0), k, r[i_src]))
    except Exception: pass
tot = sum(d[0] for d in data)
print("total samples", tot)
for d in sorted(data, reverse=True)[:n]: print(d[0], d[1], d[2][:110])
