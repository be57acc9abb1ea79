"""Per-source-line instructions executed and stall samples from an ncu report:
python tools/src_lines.py report.ncu-rep [n]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
inst, stall, text = collections.Counter(), collections.Counter(), {}
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "Line No":
        hdr = r
        i_inst = r.index("Instructions Executed")
        i_st = r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    try:
        inst[line] += int(float(r[i_inst] or 0))
        stall[line] += int(float(r[i_st] or 0))
    except ValueError:
        pass
    text[line] = r[1][:100]
ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
for line, v in inst.most_common(n):
    print(f"{v:10d} {100 * v / ti:5.1f}%  stall {100 * stall[line] / ts:5.1f}%  L{line}: {text[line]}")
