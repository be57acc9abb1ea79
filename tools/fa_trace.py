"""Timeline of the in-kernel A encode (build with -DFTGEMM_EXP_FA_TRACE):
per unit the MMA's first-k-block and accumulator-complete stamps, per item the
publish stamp; prints when each schedule group's items were done against when
its first unit started (development timing; never a bench number)."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_01024_b200 import ftgemm as F  # noqa: E402

dt, M, N, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
odt = "bf16" if dt == "bf16" else "f32"
A = synth.to_torch(synth.matrix(1, M, K, dtype=odt), odt).cuda()
B = synth.to_torch(synth.matrix(2, K, N, dtype=odt), odt).cuda()
Cm = torch.empty(M, N, dtype=A.dtype, device="cuda")
g = F.FTGemm(dt, M, N, K)
FUSE = os.environ.get("FUSE", "1") == "1"
g.encode(A if not FUSE else None, B, which=2 if FUSE else 3)
for _ in range(3):
    g.run(A, B, Cm, fuse_a=FUSE)
torch.cuda.synchronize()
buf = (C.c_uint64 * (1 << 17))()
F.lib().ftgemm_debug_trace.argtypes = [C.c_void_p, C.c_size_t]
assert F.lib().ftgemm_debug_trace(C.cast(buf, C.c_void_p), C.sizeof(buf)) == 0
tr = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
p = g.plan
cg, tiles_m, tiles_n = p.cta_group, p.tiles_m, p.tiles_n
nkb = (K + p.bk - 1) // p.bk
units_m = (tiles_m + cg - 1) // cg
units = units_m * tiles_n
g0 = max(1, 16 // cg)
ng = (units_m + g0 // 2) // g0 if units_m // g0 > 0 else 1
group = (units_m + ng - 1) // ng
us = tr[0:2 * units:2]
ue = tr[1:2 * units:2]
items = tr[4096:4096 + tiles_m * nkb].reshape(tiles_m, nkb)
starts = tr[20480:20480 + tiles_m * nkb].reshape(tiles_m, nkb)
t0 = us.min()
cs = tr[40000:40000 + 148]
ce = tr[41000:41000 + 148]
cs, ce = cs[cs > 0], ce[ce > 0]
print(json.dumps({"fuse": FUSE, "cta_start_us": [round((cs.min() - t0) / 1e3, 1), round((cs.max() - t0) / 1e3, 1)],
                  "cta_end_us": [round((ce.min() - t0) / 1e3, 1), round((ce.max() - t0) / 1e3, 1)]}))
print(json.dumps({"units": units, "group": group, "kernel_span_us": (ue.max() - t0) / 1e3,
                  "items_done_us": (items.max() - t0) / 1e3}))
tpg = group * cg
for grp in range((tiles_m + tpg - 1) // tpg):
    first_unit = grp * group * tiles_n
    tis = list(range(grp * tpg, min(tiles_m, (grp + 1) * tpg)))
    it = items[tis]
    gus = us[first_unit:min(units, first_unit + group * tiles_n)]
    print(json.dumps({"group": grp, "first_unit_start_us": round((gus.min() - t0) / 1e3, 1),
                      "items_first_done_us": round((it.min() - t0) / 1e3, 1),
                      "items_kb0_done_us": round((it[:, 0].max() - t0) / 1e3, 1),
                      "items_all_done_us": round((it.max() - t0) / 1e3, 1),
                      "kb_done_us_at": {k: round((it[:, k].max() - t0) / 1e3, 1) for k in range(0, nkb, max(1, nkb // 8))}}))
tl = tr[60000:60000 + tiles_m * nkb].reshape(tiles_m, nkb)
tc = tr[80000:80000 + tiles_m * nkb].reshape(tiles_m, nkb)
tf = tr[100000:100000 + tiles_m * nkb].reshape(tiles_m, nkb)
for nm, x0, x1 in (("load", starts, tl), ("compute", tl, tc), ("proxy_fence", tc, tf), ("release", tf, items)):
    dd = (x1 - x0) / 1e3
    print(json.dumps({"phase": nm, "median_us": float(np.median(dd)), "p90_us": float(np.percentile(dd, 90)),
                      "kb0_us": [round(v, 2) for v in dd[:6, 0]]}))
d = (items - starts) / 1e3
print(json.dumps({"item_us_median": float(np.median(d)), "item_us_p90": float(np.percentile(d, 90)),
                  "kb0_items_start_us": [round((x - t0) / 1e3, 1) for x in starts[:8, 0]],
                  "kb0_items_dur_us": [round(x, 1) for x in d[:8, 0]],
                  "g0_item_us_median": float(np.median(d[:group * cg])),
                  "later_item_us_median": float(np.median(d[group * cg:]))}))
# unit durations of the first wave vs later
dur = (ue - us) / 1e3
nclu = 148 // cg
print(json.dumps({"wave1_unit_dur_us_median": float(np.median(dur[:nclu])),
                  "later_unit_dur_us_median": float(np.median(dur[nclu:])),
                  "wave_ends_us": [round((ue[w * nclu:(w + 1) * nclu].max() - t0) / 1e3, 1)
                                   for w in range((units + nclu - 1) // nclu)]}))
