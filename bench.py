#!/usr/bin/env python
"""bench.py -- FT-GEMM TFLOPS and % overhead vs non-FT / cuBLAS at 0..N errors/min.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], "cfg3"): BF16 tcgen05 ABFT GEMM 8192^3,
C = A B (alpha 1, beta 0), inputs U[-1,1) rounded to BF16 (synthetic, seeded).
One STEP = the whole hot path of SURVEY.md §8(a): encode A (a1), encode B (a2),
the fused FT GEMM with verify / locate / correct (a3-a7) at ft_level CORRECT,
with faults injected by a seeded schedule at ERRORS_PER_MIN (a4); the report
counters (a8) accumulate on the device and are read and checked after the timed
region.  N > 1 (torchrun): M-block partition (weak scaling): every rank owns an
8192 x 8192 block of A and C, B (8192 x 8192) is generated on rank 0 and
broadcast ONCE over NCCL before timing; each rank's step is the same as the
1-GPU step.  Timing: W warm-up steps, then K steps bracketed by a barrier +
cuda.synchronize on both sides, CUDA events on the launch stream, max over
ranks.  Inputs (A + B = 256 MiB per rank) are larger than the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FT-GEMM TFLOPS & % overhead vs non-FT/cuBLAS at 0..N errors/min, 1-8 B200"
M_PER_RANK, N_DIM, K_DIM = 8192, 8192, 8192
ERRORS_PER_MIN = 500.0           # "hundreds of errors per minute" (north_star)
SWEEP_RATES = (0.0, 1.0, 10.0, 100.0, 500.0)
OFFLINE_GAMMA0 = (1e-5, 1e-4, 2e-4)   # per-tile error probability per execution (online vs offline)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)   # ~0.35 s timed: several clock samples, ~3 faults at 500/min
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-sweep", action="store_true", help="skip the injection-rate sweep and comparators")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU-oracle sample budget")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------- CPU oracle leg ---
def cpu_oracle_sample(budget_s: float):
    """Time the oracle (as it stands) on a bounded tile sample of the workload:
    whole check tiles (125 x 252 x 8192) of the 8192^3 problem, FP64, all host
    cores.  Returns (TFLOPS, cores, description)."""
    import oracle
    import synth
    oracle.build()
    tm, tn, K = 125, 252, K_DIM                # the plan's BF16 check tile
    done_tiles, flops, t_spent = 0, 0.0, 0.0
    ti = tj = 0
    t0 = time.time()
    while True:
        A = synth.matrix(synth.BASE_SEED + synth.SEED_A, M_PER_RANK, K, dtype="bf16", r0=ti * tm, r1=ti * tm + tm)
        B = synth.matrix(synth.BASE_SEED + synth.SEED_B, K, N_DIM, dtype="bf16", c0=tj * tn, c1=tj * tn + tn)
        t1 = time.time()
        oracle.ftgemm(A, B, out="bf16", tile_m=tm, tile_n=tn, bk=64, u_acc=2.0 ** -23, lambda1=8.0, lambda2=16.0)
        t_spent += time.time() - t1
        flops += 2.0 * tm * tn * K
        done_tiles += 1
        ti, tj = (ti + 7) % 65, (tj + 5) % 32
        if time.time() - t0 > budget_s or done_tiles >= 4096:
            break
    tflops = flops / t_spent / 1e12
    return tflops, oracle.num_threads(), (f"{done_tiles} check tiles of 125x252x8192 (BF16 values, FP64 oracle incl. "
                                           f"encode/verify), {flops / 1e9:.1f} GFLOP in {t_spent:.1f}s")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    tflops, cores, desc = cpu_oracle_sample(min(args.cpu_seconds, 60.0))
    steps = args.steps
    ms = 2.0 * M_PER_RANK * N_DIM * K_DIM / (tflops * 1e12) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": tflops, "unit": "TFLOPS", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg3: BF16 ABFT GEMM 8192^3 (tile-sampled CPU oracle)", "M": M_PER_RANK,
                       "N": N_DIM, "K": K_DIM},
            "cpu_baseline": {"value": tflops, "unit": "TFLOPS", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": tflops, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "the reference arm is the paper-derived CPU oracle (no reference implementation exists)"}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- clocks ---
class ClockSampler:
    def __init__(self, index: int):
        self.proc = None
        self.path = f"/tmp/ftgemm_clocks_{os.getpid()}.csv"
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for ln in open(self.path):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[4:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        smax = max(r[1] for r in rows)
        loaded = [r for r in rows if r[2] > 300.0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in loaded:
            for n, v in zip(names, r[3][1:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": smax,
                "samples": len(loaded), "power_w_max": max(r[2] for r in rows), "reasons": sorted(reasons)}


# ------------------------------------------------------------------ ours ---
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2305_01024_b200 import ftgemm as F
    from paper_2305_01024_b200 import distributed as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    Mr, N, K = M_PER_RANK, N_DIM, K_DIM
    flops_rank = 2.0 * Mr * N * K

    # ---- inputs: A block by global row index, B on rank 0 + one broadcast ----
    A_h = synth.matrix(synth.BASE_SEED + synth.SEED_A, Mr * world, K, dtype="bf16", r0=rank * Mr, r1=(rank + 1) * Mr)
    A = synth.to_torch(A_h, "bf16").to(dev)
    del A_h
    g = F.FTGemm("bf16", Mr, N, K, device=dev)
    pl = g.plan
    bcast_ms = 0.0
    if rank == 0:
        B = synth.to_torch(synth.matrix(synth.BASE_SEED + synth.SEED_B, K, N, dtype="bf16"), "bf16").to(dev)
    else:
        B = torch.empty(K, N, dtype=torch.bfloat16, device=dev)
    if world > 1:
        bcast_ms = D.broadcast_b(g, B, src=0)
    C = torch.empty(Mr, N, dtype=torch.bfloat16, device=dev)

    # ---- seeded fault schedule at a rate (errors / minute) ----
    rng = np.random.default_rng(synth.BASE_SEED + synth.SEED_PLAN + rank)
    tiles_total = pl.tiles_m * pl.tiles_n

    def site():
        t = int(rng.integers(tiles_total))
        ti, tj = divmod(t, pl.tiles_n)
        bm = min(pl.check_tile_m, Mr - ti * pl.check_tile_m)
        bn = min(pl.check_tile_n, N - tj * pl.check_tile_n)
        return (ti * pl.check_tile_m + int(rng.integers(bm)), tj * pl.check_tile_n + int(rng.integers(bn)),
                int(rng.integers(K)), 30, F.INJ_FLIP, F.TGT_ACC, 0.0)

    def schedule(rate, nsteps, step_ms):
        """rate errors/min over nsteps steps of step_ms: round(rate x time)
        faults at evenly spaced steps, seeded sites"""
        n = int(round(rate * nsteps * step_ms / 60000.0))
        out = [[] for _ in range(nsteps)]
        for i in range(n):
            out[int((i + 0.5) * nsteps / n)].append(site())
        return out

    def step(inj=()):
        g.encode(A, B)
        g.run(A, B, C, ft_level=F.FT_CORRECT, injections=inj)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn_list, warm: int):
        """fn_list: per-step callables; returns ms/step (max over ranks)."""
        for i in range(warm):
            fn_list[i % len(fn_list)]()
        barrier(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for fn in fn_list:
            fn()
        e1.record(stream)
        e1.synchronize()
        barrier(); torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / len(fn_list))

    # ---- warm-up + rough step time for the schedule ----
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    g.reset()
    est = timed([step] * 5, 0)

    # ---- main timed region: K steps at ERRORS_PER_MIN, kernel events per step ----
    sched = schedule(ERRORS_PER_MIN, args.steps, est)
    n_injected = sum(len(s) for s in sched)
    g.reset()
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    g.reset()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    barrier(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        g.encode(A, B)
        kev[i][0].record(stream)
        g.run(A, B, C, ft_level=F.FT_CORRECT, injections=sched[i])
        kev[i][1].record(stream)
    e1.record(stream)
    e1.synchronize()
    barrier(); torch.cuda.synchronize()
    clk = clocks.stop()
    ms_step = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    ms_kernel = max_over_ranks(sum(a.elapsed_time(b) for a, b in kev) / args.steps)
    counts, events = g.report()
    ok_faults = counts["corrected"] == n_injected and counts["uncorrectable"] == 0 and counts["checksum_only"] == 0
    value = flops_rank * world / (ms_step * 1e-3) / 1e12
    launches_per_step = 2   # encode_ab (both operands, one launch), fused GEMM (tickets reset by cudaMemsetAsync, not kernels)

    extra = {}
    if not args.no_sweep:
        reps, rounds = max(20, args.steps), 3
        stress = []
        for ti in range(pl.tiles_m):
            for tj in range(pl.tiles_n):
                r = ti * pl.check_tile_m + (ti * 7 + tj) % min(pl.check_tile_m, Mr - ti * pl.check_tile_m)
                c = tj * pl.check_tile_n + (tj * 5 + ti) % min(pl.check_tile_n, N - tj * pl.check_tile_n)
                stress.append((r, c, (ti * 131 + tj * 17) % K, 30, F.INJ_FLIP, F.TGT_ACC, 0.0))
        one = [site()]
        n_calls = reps * rounds
        # the injection-rate sweep: one seeded schedule per rate, call i of that
        # rate's configuration uses step i of its schedule
        rate_sched = {str(int(r)): schedule(r, n_calls, est) for r in SWEEP_RATES}
        configs = {
            "ft_off": lambda i: g.run(A, B, C, ft_level=F.FT_OFF),
            "cublas": lambda i: torch.matmul(A, B, out=C),
            "ft_run": lambda i: g.run(A, B, C, ft_level=F.FT_CORRECT),
            "ft_step": lambda i: step(),
            "encode": lambda i: g.encode(A, B),
            "encode_a": lambda i: g.encode(A, None, which=1),
            "one_fault_run": lambda i: g.run(A, B, C, ft_level=F.FT_CORRECT, injections=one),
            # the paper's comparison scheme (Ding 2011): cuBLAS GEMMs + separate verification
            "nonfused_step": lambda i: (g.encode(A, B, which=3 | 4), g.run_nonfused(A, B, C, ft_level=F.FT_CORRECT)),
            "nonfused_run": lambda i: g.run_nonfused(A, B, C, ft_level=F.FT_CORRECT),
            # online verification after every K_s = 256 step: 32 checks per tile
            "online_ks256_run": lambda i: g.run_online(A, B, C, ks=256),
            "online_ks2048_run": lambda i: g.run_online(A, B, C, ks=2048),
        }
        for key, sc in rate_sched.items():
            configs["rate_" + key] = (lambda sc_: (lambda i: step(sc_[i])))(sc)
        # every configuration timed CALL BY CALL in one interleaved loop (one event
        # pair per call on the launch stream, median per configuration), so all
        # of them -- the rate sweep included -- see the same clock / power state:
        # under the B200's power cap, back-to-back blocks of one configuration
        # drift apart by tens of percent
        names = list(configs)
        evs = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(n_calls)] for k in names}
        for k in names:
            if not k.startswith("rate_"):
                configs[k](0)
        barrier(); torch.cuda.synchronize()
        g.reset()
        for i in range(n_calls):
            for k in names:
                evs[k][i][0].record(stream)
                configs[k](i)
                evs[k][i][1].record(stream)
        torch.cuda.synchronize()
        samples = {k: [a.elapsed_time(b) for a, b in evs[k]] for k in names}
        cs_sweep, _ = g.report(0)
        rate_inj = {k: sum(len(x) for x in sc) for k, sc in rate_sched.items()}
        med = {k: max_over_ranks(statistics.median(v)) for k, v in samples.items()}
        g.reset()
        t_stress = timed([lambda: g.run(A, B, C, ft_level=F.FT_CORRECT, injections=stress)] * 3, 1)
        cs, _ = g.report(0)
        stress_ok = cs["corrected"] == 4 * len(stress) and cs["uncorrectable"] == 0
        t_off, t_cub = med["ft_off"], med["cublas"]
        sweep = {}
        for rate in SWEEP_RATES:
            key = str(int(rate))
            t = med["rate_" + key]
            sweep[key] = {"ms_per_step": t, "tflops": flops_rank * world / (t * 1e-3) / 1e12,
                          "steps": n_calls, "injected": rate_inj[key],
                          "overhead_vs_ft_off_pct": 100.0 * (t - t_off) / t_off,
                          "overhead_vs_cublas_pct": 100.0 * (t - t_cub) / t_cub,
                          "run_only_overhead_vs_ft_off_pct": 100.0 * (t - med["encode"] - t_off) / t_off}
        # every injected fault of the sweep (and of the one-fault comparator) corrected
        n_sweep_inj = sum(rate_inj.values()) + n_calls
        sweep_ok = (cs_sweep["corrected"] == n_sweep_inj and cs_sweep["uncorrectable"] == 0
                    and cs_sweep["checksum_only"] == 0)
        # ---- online vs offline ABFT: per-tile error rate gamma0 ----
        offline = {}
        t_rows = timed([lambda: g.run(A, B, C, ft_level=F.FT_DETECT_ROWS)] * reps, 2)

        def draw(g0):
            hit = np.nonzero(rng.random(tiles_total) < g0)[0]
            out = []
            for t in hit:
                ti, tj = divmod(int(t), pl.tiles_n)
                out.append((ti * pl.check_tile_m + int(rng.integers(min(pl.check_tile_m, Mr - ti * pl.check_tile_m))),
                            tj * pl.check_tile_n + int(rng.integers(min(pl.check_tile_n, N - tj * pl.check_tile_n))),
                            int(rng.integers(K)), 30, F.INJ_FLIP, F.TGT_ACC, 0.0))
            return out
        calls, max_runs = 20, 8
        for g0 in OFFLINE_GAMMA0:
            cm = F.cost_model(g0, tiles_total)
            on_inj = [draw(g0) for _ in range(calls)]
            t_on = timed([(lambda inj: (lambda: step(inj)))(x) for x in on_inj], 2)
            execs = []
            e0o, e1o = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0o.record(stream)
            for _ in range(calls):
                inj, run_of = [], []
                for r in range(max_runs):
                    d = draw(g0)
                    inj += d
                    run_of += [r] * len(d)
                g.encode(A, B)
                n_exec, clean = g.run_offline(A, B, C, injections=inj, inj_run=run_of, max_runs=max_runs)
                execs.append(n_exec)
            e1o.record(stream)
            e1o.synchronize()
            t_off_call = e0o.elapsed_time(e1o) / calls
            offline[f"{g0:g}"] = {
                "gamma": cm["gamma"], "tiles": tiles_total, "calls": calls,
                "online_ms_per_call": t_on, "online_faults": sum(len(x) for x in on_inj),
                "offline_ms_per_call": t_off_call, "offline_mean_executions": float(np.mean(execs)),
                "offline_restart_model_executions": 1.0 / (1.0 - cm["gamma"]),
                "paper_model_offline_expected_runs": cm["offline_expected_runs"],
                "paper_model_offline_ms": med["encode"] + cm["offline_expected_runs"] * t_rows,
                "offline_vs_online_pct": 100.0 * (t_off_call - t_on) / t_on}
        g.reset()
        g.encode(A, B)                               # restore the fused path's encoded operand
        extra = {
            "nonfused_step_ms": med["nonfused_step"], "nonfused_run_ms": med["nonfused_run"],
            "online_ks256_run_ms": med["online_ks256_run"], "online_ks2048_run_ms": med["online_ks2048_run"],
            "fused_speedup_vs_nonfused_pct": 100.0 * (med["nonfused_step"] - med["ft_step"]) / med["ft_step"],
            "detect_rows_run_ms": t_rows,
            "detect_rows_overhead_vs_ft_off_pct": 100.0 * (t_rows - med["ft_off"]) / med["ft_off"],
            "online_vs_offline": offline,
            "ft_off_ms": t_off, "ft_off_tflops": flops_rank * world / (t_off * 1e-3) / 1e12,
            "cublas_ms": t_cub, "cublas_tflops": flops_rank * world / (t_cub * 1e-3) / 1e12,
            "ft_step_ms": med["ft_step"], "ft_run_only_ms": med["ft_run"],
            "encode_ms": med["encode"], "encode_a_ms": med["encode_a"],
            "encode_gbs": (2 * Mr * K + 2 * K * N + 2 * K * pl.tiles_n * pl.bn) / (med["encode"] * 1e-3) / 1e9,
            "encode_hbm_frac": (2 * Mr * K + 2 * K * N + 2 * K * pl.tiles_n * pl.bn) / (med["encode"] * 1e-3) / 1e9
            / load_peaks()[0]["hbm_gbs"],
            "overhead_vs_ft_off_pct": 100.0 * (med["ft_step"] - t_off) / t_off,
            "overhead_vs_cublas_pct": 100.0 * (med["ft_step"] - t_cub) / t_cub,
            "overhead_run_only_vs_ft_off_pct": 100.0 * (med["ft_run"] - t_off) / t_off,
            "overhead_pre_encoded_B_vs_ft_off_pct": 100.0 * (med["ft_run"] + med["encode_a"] - t_off) / t_off,
            "one_fault_call_ms": med["one_fault_run"], "stress_one_fault_per_tile_ms": t_stress,
            "stress_faults": len(stress), "stress_all_corrected": bool(stress_ok),
            "rate_sweep_errors_per_min": sweep, "rate_sweep_all_corrected": bool(sweep_ok),
            "comparator_rounds": rounds, "comparator_reps": reps,
        }

    # ---- e2e: public API with host buffers, H2D inputs + D2H result per step ----
    A_pin = A.cpu().pin_memory(); B_pin = B.cpu().pin_memory()
    C_pin = torch.empty(Mr, N, dtype=torch.bfloat16).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))

    def e2e_step():
        A.copy_(A_pin, non_blocking=True)
        B.copy_(B_pin, non_blocking=True)
        g.encode(A, B)
        g.run(A, B, C, ft_level=F.FT_CORRECT)
        C_pin.copy_(C, non_blocking=True)
    t_e2e_serial = timed([e2e_step] * e2e_steps, 2)
    # the same steps through paper_2305_01024_b200.pipeline.HostPipeline: H2D of
    # step s+1, kernels of step s and D2H of step s-1 overlap on three streams
    from paper_2305_01024_b200.pipeline import HostPipeline
    pipe = HostPipeline(g)
    C_pins = [torch.empty(Mr, N, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    for i in range(2):                                    # warm-up
        pipe.submit(A_pin, B_pin, C_pins[i % 2])
    pipe.synchronize()
    barrier(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    pipe.begin(stream)
    for i in range(e2e_steps):
        pipe.submit(A_pin, B_pin, C_pins[i % 2])
    pipe.join(stream)
    e1.record(stream)
    e1.synchronize()
    barrier(); torch.cuda.synchronize()
    t_e2e = max_over_ranks(e0.elapsed_time(e1) / e2e_steps)
    pipe_ok = bool(torch.equal(C_pins[(e2e_steps - 1) % 2], C_pin))      # same bits as the serial step
    e2e = {"value": flops_rank * world / (t_e2e * 1e-3) / 1e12, "unit": "TFLOPS",
           "h2d_bytes_per_step": A.numel() * 2 + B.numel() * 2, "d2h_bytes_per_step": C.numel() * 2,
           "ms_per_step": t_e2e, "api": "paper_2305_01024_b200.pipeline.HostPipeline (3 streams, 2 slots)",
           "serial_ms_per_step": t_e2e_serial, "pipelined_equals_serial": pipe_ok}

    peaks, kind = load_peaks()
    # the kernel is timed inside ~0.4 s of back-to-back steps (power-capped,
    # sustained regime): the sustained cuBLAS figure is its peak; the burst
    # figure is reported beside it
    sustained = peaks.get("bf16_tflops_sustained")
    peak = sustained or peaks["bf16_tflops"]
    achieved = flops_rank / (ms_kernel * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("fused_gemm_bf16_8192_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "tc_ftgemm_kernel<bf16,256,FT>",
                "peak_kind": f"{kind} bf16 {'sustained (cuBLAS back to back, power-capped)' if sustained else 'burst'}",
                "algorithmic_flops_per_launch": flops_rank,
                "peak_burst": peaks["bf16_tflops"], "frac_burst": achieved / peaks["bf16_tflops"]}

    if rank == 0:
        cpu = None
        if world == 1:
            tfl, cores, desc = cpu_oracle_sample(args.cpu_seconds)
            cpu = {"value": tfl, "unit": "TFLOPS", "cores": cores, "kind": "oracle", "sample": desc}
        line = {"metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": "cfg3: BF16 tcgen05 ABFT GEMM 8192^3 per GPU (M-block partition for N>1)",
                           "M": Mr * world, "N": N, "K": K, "alpha": 1.0, "beta": 0.0, "ft_level": "CORRECT",
                           "errors_per_min": ERRORS_PER_MIN, "check_tile": [pl.check_tile_m, pl.check_tile_n],
                           "mma_tile": [pl.bm, pl.bn, pl.bk], "l2": "inputs larger than L2 (A+B 256 MiB/rank)",
                           "parallelism": f"mblock{world}" if world > 1 else "single"},
                "faults": {"injected": n_injected, **{k: v for k, v in counts.items() if v}, "all_corrected": ok_faults},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
                "clocks": clk, "kernel_ms": ms_kernel, "b_broadcast_ms": bcast_ms, **extra}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
