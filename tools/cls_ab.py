"""Tile classes of two library builds, interleaved call by call (dev timing):
python tools/cls_ab.py dtype M N K lib1 lib2 "bn:cg" ["bn:cg" ...]"""
import importlib.util, json, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
dt, M, N, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
libs, classes = sys.argv[5:7], sys.argv[7:]
odt = "bf16" if dt == "bf16" else "f32"
A = synth.matrix_torch(1, M, K, dtype=odt); B = synth.matrix_torch(2, K, N, dtype=odt)
C = torch.empty(M, N, dtype=A.dtype, device="cuda")
fns, gs = {}, []
for i, lib in enumerate(libs):
    os.environ["FTGEMM_LIB"] = lib
    spec = importlib.util.spec_from_file_location(f"ftg{i}", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2305_01024_b200", "ftgemm.py"))
    F = importlib.util.module_from_spec(spec); sys.modules[spec.name] = F; spec.loader.exec_module(F)
    for c in classes:
        bn, cg = map(int, c.split(":"))
        g = F.FTGemm(dt, M, N, K, tile=(bn, cg)); g.encode(A, B); gs.append(g)
        fns[f"{os.path.basename(lib)}:{c}:run"] = (lambda g=g: g.run(A, B, C))
        fns[f"{os.path.basename(lib)}:{c}:off"] = (lambda g=g, F=F: g.run(A, B, C, ft_level=F.FT_OFF))
ev = {k: [] for k in fns}
for f in fns.values(): f()
torch.cuda.synchronize()
for j in range(int(os.environ.get("NREP", "40"))):
    for k, f in fns.items():
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record(); f(); e1.record(); ev[k].append((e0, e1))
torch.cuda.synchronize()
for k, v in ev.items():
    print(json.dumps({"shape": f"{dt} {M}x{N}x{K}", "what": k, "ms": round(statistics.median(a.elapsed_time(b) for a, b in v), 4)}), flush=True)
print("detected", [g.report()[0]["tiles_detected"] for g in gs])
