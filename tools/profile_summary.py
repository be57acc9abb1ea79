"""Summarise ncu outputs into profiles/ (committed evidence).

    python tools/profile_summary.py <round-tag> <launches.csv> <full.ncu-rep> [<full2.ncu-rep> ...]

Writes profiles/<tag>_launches.md (per-launch device time of every kernel in the
command, shares per kernel name), profiles/<tag>_ncu_<name>.md (key metrics of
each --set full capture) and profiles/ncu_traffic.json (DRAM bytes per launch of
the fused kernel, read by bench.py's roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    idx = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        k = (int(r[idx["ID"]]), r[idx["Kernel Name"]])
        per.setdefault(k, {})[r[idx["Metric Name"]]] = (float(r[idx["Metric Value"]].replace(",", "")),
                                                       r[idx["Metric Unit"]])
    return per


def to_ns(v, unit):
    return v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second"]


def main():
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    os.makedirs(PROF, exist_ok=True)
    per = launches(lcsv)
    lines = [f"# ncu launch list ({tag})", "",
             "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none`",
             "(cold-cache, serialised launches: compare SHARES, not absolutes)", "",
             "| id | kernel | time (us) | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|---|"]
    tot = defaultdict(float)
    for (i, name), m in sorted(per.items()):
        t = to_ns(*m["gpu__time_duration.sum"]) / 1e3 if "gpu__time_duration.sum" in m else 0.0
        rd = m.get("dram__bytes_read.sum", (0, ""))[0]
        wr = m.get("dram__bytes_write.sum", (0, ""))[0]
        short = name.split("(")[0][:70]
        tot[short] += t
        lines.append(f"| {i} | `{short}` | {t:.1f} | {rd / 1e6 if m.get('dram__bytes_read.sum', (0, 'byte'))[1] == 'byte' else rd:.1f} | "
                     f"{wr / 1e6 if m.get('dram__bytes_write.sum', (0, 'byte'))[1] == 'byte' else wr:.1f} |")
    s = sum(tot.values()) or 1.0
    lines += ["", "All launches of the command (incl. the harness's device-side input generation):", "",
              "| kernel | total (us) | share |", "|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {v:.1f} | {100 * v / s:.1f}% |")
    # the step's kernels: libftgemm's own (namespace ftg)
    mine = {k: v for k, v in tot.items() if "ftg::" in k}
    sm = sum(mine.values()) or 1.0
    lines += ["", "Shares of the step (libftgemm kernels only):", "", "| kernel | total (us) | share of step |",
              "|---|---|---|"]
    for k, v in sorted(mine.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {v:.1f} | {100 * v / sm:.1f}% |")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    traffic = {}
    for rep in reps:
        m = raw_metrics(rep)
        name = os.path.splitext(os.path.basename(rep))[0]
        out = [f"# ncu --set full: {name} ({tag})", "", "| metric | value | unit |", "|---|---|---|"]
        for k in KEYS:
            if k in m:
                out.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
        open(os.path.join(PROF, f"{tag}_ncu_{name}.md"), "w").write("\n".join(out) + "\n")
        try:
            rd = float(m["dram__bytes_read.sum"][0].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m["dram__bytes_read.sum"][1]]
            wr = float(m["dram__bytes_write.sum"][0].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m["dram__bytes_write.sum"][1]]
            traffic[name] = rd + wr
        except Exception:
            pass
    tj = os.path.join(PROF, "ncu_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    d.update({f"{tag}:{k}": v for k, v in traffic.items()})
    if f"{tag}:fused_ft" in d:
        d["fused_gemm_bf16_8192_bytes_per_launch"] = d[f"{tag}:fused_ft"]
    json.dump(d, open(tj, "w"), indent=1)
    print("wrote", PROF)


if __name__ == "__main__":
    main()
