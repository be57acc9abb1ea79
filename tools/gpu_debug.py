"""Development probe: run the CUDA path on small problems and print diagnostics."""
import sys, os, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
from paper_2305_01024_b200 import ftgemm as F

torch.cuda.init()
print("device", torch.cuda.get_device_name(0), torch.cuda.get_device_capability(0), flush=True)

def dev(x, dt):
    return synth.to_torch(x, "bf16" if dt == "bf16" else "f32").cuda()

def host(t):
    return t.float().cpu().numpy()

def check(dt, M, N, K, ft=F.FT_CORRECT, inj=(), dist="signed", alpha=1.0, beta=0.0):
    t0 = time.time()
    odt = "bf16" if dt == "bf16" else "f32"
    A, B, Cin = synth.problem(M, N, K, dist=dist, dtype=odt)
    g = F.FTGemm(dt, M, N, K)
    pl = g.plan
    Ad, Bd, Cd = dev(A, dt), dev(B, dt), dev(Cin, dt)
    if ft != F.FT_OFF:
        g.encode(Ad, Bd)
    g.run(Ad, Bd, Cd, alpha=alpha, beta=beta, ft_level=ft, injections=inj)
    torch.cuda.synchronize()
    cnt, evs = g.report() if ft != F.FT_OFF else ({}, [])
    Cg = host(Cd)
    tm, tn = (pl.check_tile_m, pl.check_tile_n) if ft != F.FT_OFF else (pl.off_tile_m, pl.off_tile_n)
    r = oracle.ftgemm(A, B, Cin, alpha=alpha, beta=beta, out=odt, tile_m=tm, tile_n=tn, bk=pl.bk,
                      u_acc=pl.u_acc, lambda1=pl.lambda1, lambda2=pl.lambda2,
                      ft_level=ft if ft != F.FT_OFF else oracle.FT_OFF, injections=inj)
    ref = r.C.astype(np.float64)
    fro = np.linalg.norm(Cg - ref) / max(np.linalg.norm(ref), 1e-300)
    mx = np.nanmax(np.abs(Cg - ref))
    print(f"[{dt} {M}x{N}x{K} ft={ft} inj={len(inj)}] fro={fro:.3e} maxabs={mx:.3e} plan=({pl.bm},{pl.bn},{pl.bk},{tm}x{tn}) "
          f"gpu={ {k:v for k,v in cnt.items() if v} } oracle={ {k:v for k,v in r.counts.items() if v} } ({time.time()-t0:.1f}s)", flush=True)
    if evs or r.events:
        print("   gpu ev:", [(e['row'], e['col'], e['kind'], round(e['resid_row'],4), round(e['tau_row'],5)) for e in evs[:6]])
        print("   orc ev:", [(e['row'], e['col'], e['kind'], round(e['resid_row'],4), round(e['tau_row'],5)) for e in r.events[:6]])
    return fro, cnt, evs, r

def guarded(f, *a, **k):
    try:
        return f(*a, **k)
    except Exception:
        traceback.print_exc()
        sys.stdout.flush()

# TF32 operand semantics probe: x = 1 + 2^-11 + 2^-12 ; trunc -> 1.0 ; RN -> 1 + 2^-10
def tf32_probe():
    M = N = 128; K = 32
    A = np.zeros((M, K), np.float32); B = np.zeros((K, N), np.float32)
    x = np.float32(1 + 2**-11 + 2**-12)
    A[0, 0] = x; B[0, 0] = 1.0
    A[1, 0] = 1.0; B[0, 1] = 1.0
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    Cd = torch.zeros(M, N, device="cuda")
    F.run("tf32", Ad, Bd, Cd, ft_level=F.FT_OFF)
    torch.cuda.synchronize()
    v = Cd[0, 0].item()
    print(f"TF32 probe: C[0,0]={v!r}  trunc->1.0  rn->{1+2**-10!r}  C[1,1]={Cd[1,1].item()}", flush=True)

CASES = {
    "off": lambda: [guarded(check, dt, 256, 256, 256, ft=F.FT_OFF) for dt in ["bf16", "tf32", "f32_simt"]],
    "probe": lambda: guarded(tf32_probe),
    "bf16": lambda: guarded(check, "bf16", 256, 256, 256),
    "tf32": lambda: guarded(check, "tf32", 256, 256, 256),
    "simt": lambda: guarded(check, "f32_simt", 256, 256, 256),
}
def full(dt):
    guarded(check, dt, 256, 256, 256)
    guarded(check, dt, 300, 520, 200, dist="int")
    guarded(check, dt, 257, 300, 333, alpha=1.5, beta=-0.5)
    guarded(check, dt, 256, 256, 256, inj=[(130, 5, 100, 30, 0, 0, 0.0)])
    guarded(check, dt, 256, 256, 256, inj=[(3, 200, 10, 0, 1, 0, 1000.0), (200, 7, 250, 29, 0, 0, 0.0)])
for dt in ["bf16", "tf32", "f32_simt"]:
    CASES["full_" + dt] = (lambda d: (lambda: full(d)))(dt)
CASES["rag_off"] = lambda: [guarded(check, dt, M, N, K, ft=F.FT_OFF) for dt in ["bf16", "tf32"] for (M, N, K) in [(130, 130, 130), (300, 520, 200), (256, 256, 256)]]
CASES["big"] = lambda: [guarded(check, "bf16", 2048, 2048, 2048), guarded(check, "tf32", 2048, 2048, 2048),
                        guarded(check, "f32_simt", 1024, 1024, 1024)]
for name in (sys.argv[1:] or ["off", "probe", "full_bf16", "full_tf32", "full_f32_simt", "big"]):
    print("== case", name, flush=True)
    CASES[name]()
print("done", flush=True)
