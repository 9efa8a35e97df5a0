#!/usr/bin/env python3
"""bench.py -- time-to-solution of the B200 mixed-precision IR Lyapunov solver.

Contract:
  python bench.py --gpus N --steps K --warmup W [--impl reference] [--config cfg1]

A "step" is one complete IR solve (Algorithm 2 with the LDL^T
sign-function Newton solver, Algorithm 4) of BASELINE.json configs[1]:
n = 1024, m = 4, W = L S L^T, bf16 solver, fp64 refinement, tol 1e-14 -- with
the inputs resident in HBM.  L2 is flushed (256 MB write) before every timed
step; step times are CUDA-event device times on the solver's stream.  With N
ranks every rank solves its own equation (seed 1 + rank; "weak" scaling, no
data-path collective; the final residual norms are all-gathered over NCCL
after the timed region).  `value` = solves/s of the whole job.

The metric's second half, sign-Newton TFLOP/s as a fraction of the fp16 peak, is
measured on rank 0 after the timed region as the fp16 A-sequence (the u_s
inversions, 2 n^3 flops each) at configs[3]'s n = 16384 (`sign_newton_at_scale`)
and configs[2]'s n = 4096 (`sign_newton_at_scale_cfg2`); `--scale` selects them.

--impl reference times the CPU oracle (oracle/, plain C) as it stands on the
host cores: each step is one emulated-bf16 inversion of A_0 (a bounded sample
of the workload), scaled to solves/s by the number of inversions the method
needs for this equation.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Lyapunov IR time-to-solution; sign-Newton TFLOP/s as fraction of B200 fp16 peak"
UNIT = "solves/s"

WORKLOADS = {
    "cfg0": dict(gen="cfg0", us="fp16", tol=1e-14, maxit=10, max_cols=128,
                 desc="configs[0]: n=64 m=2 Cholesky W=LL^T, A=Q diag(-lambda) Q^T, fp16 solver, tol 1e-14"),
    "cfg1": dict(gen="cfg1", us="bf16", tol=1e-14, maxit=50, max_cols=640,
                 desc="configs[1]: n=1024 m=4 LDL^T W=LSL^T, A=-(Q diag(lambda) Q^T)+K, bf16 solver, "
                      "fp64 refinement, tol 1e-14"),
    "cfg2": dict(gen="cfg2", us="fp16", tol=1e-14, maxit=50, max_cols=512,
                 desc="configs[2]: n=4096 m=8 convection-diffusion 64x64, fp16 solver"),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------ reference arm (oracle)
REF_N = {"cfg0": 64, "cfg1": 192, "cfg2": 100, "cfg4": 192}


def _oracle_solve(p, us, imax):
    import oracle
    with oracle.model("tc"):
        if p.S is not None:
            return oracle.ir_ldlt(p.A, p.L, p.S, us=us, tol=1e-14, imax=imax)
        return oracle.ir_chol(p.A, p.L, us=us, tol=1e-14, imax=imax)


def _reduced_problem(config, n):
    import problems as P
    if config == "cfg2":
        return P.cfg2(g=int(round(n ** 0.5)))
    if config == "cfg4":
        return P.cfg4_member(0, n=n)
    return getattr(P, config)(n=n)


def run_reference(args):
    """Reference arm = the CPU oracle (oracle/, plain C, tc precision model) as it stands,
    one host core.  Each step is one COMPLETE IR solve (A-sequence, Z-sides, residual
    factorizations, solution updates) of the same recipe at a reduced order n (the
    oracle needs ~20 min for n = 1024); value = solves/s of exactly that timed work."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    cfgname = args.config if args.config in REF_N else "cfg1"
    n = REF_N[cfgname]
    p = _reduced_problem(cfgname, n)
    us = {"cfg0": "fp16", "cfg1": "bf16", "cfg2": "fp16", "cfg4": "fp16"}[cfgname]
    oracle.lib()
    for _ in range(max(0, args.warmup)):
        _oracle_solve(p, us, 30)
        break                                   # one warm-up solve (page-in); the rest are identical
    times, r = [], None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = _oracle_solve(p, us, 30)
        times.append(time.perf_counter() - t0)
    t_solve = sum(times) / len(times)
    value = 1.0 / t_solve
    desc = WORKLOADS[cfgname]["desc"] if cfgname in WORKLOADS else "configs[4] member"
    sample = (f"one complete oracle IR solve per step (tc model, {us} solver, fp64 refinement) of the "
              f"{cfgname} recipe at n={n} (status {r.status}, {r.steps} IR steps, {r.newton_total} Newton "
              f"steps); 1 core; not extrapolated")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_solve,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": us,
            "data": "synthetic", "config": {"workload": f"{desc} -- recipe at reduced n={n}", "n": n, "m": p.m},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_sample(config, budget_s=30.0):
    """The oracle as it stands (tc model, one core) on a bounded sample: one complete IR
    solve of the benched recipe at n = 256 (~20 s); value scaled to the benched n by the
    method's n^3 cost (every phase is O(n^3) or O(n p^2) at ranks p ~ n / 10)."""
    import problems as P
    n_s = 256
    p = P.cfg1(n=n_s) if config == "cfg1" else _reduced_problem(config, n_s)
    us = WORKLOADS[config]["us"]
    t0 = time.perf_counter()
    r = _oracle_solve(p, us, 30)
    t = time.perf_counter() - t0
    n_full = {"cfg0": 64, "cfg1": 1024, "cfg2": 4096}.get(config, 1024)
    scale = (n_full / n_s) ** 3
    return {"value": 1.0 / (t * scale), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"one complete oracle IR solve (tc model, {us}) of the {config} recipe at n={n_s}: "
                      f"{t:.1f} s on 1 core ({r.status}, {r.steps} IR steps); value = 1 / (that time x "
                      f"(n/{n_s})^3 = {scale:.0f})",
            "measured_s_at_sample": t}


# ------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    importlib_build()
    import paper_2510_02126_b200 as G
    import problems as P
    wl = WORKLOADS[args.config]
    p = getattr(P, wl["gen"])(seed={"cfg0": 0, "cfg1": 1, "cfg2": 2}[args.config] + rank)
    n, m = p.n, p.m
    ldlt = p.S is not None
    A = torch.tensor(p.A, dtype=torch.float64, device=dev)
    Lt = torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device=dev)
    S = torch.tensor(p.S, dtype=torch.float64, device=dev) if ldlt else None
    solver = G.Solver(n, us=wl["us"], max_cols=wl["max_cols"])
    cm = wl["max_cols"]
    Zt = torch.empty((cm, n), dtype=torch.float64, device=dev)
    Yb = torch.zeros((cm, cm), dtype=torch.float64, device=dev) if ldlt else None
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)    # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream()

    def solve():
        return solver.solve(A, Lt, S, tol=wl["tol"], maxit=wl["maxit"], out=(Zt, Yb))

    for _ in range(args.warmup):
        res = solve()
    # pick the dominant kernel class by device time over one (untimed) solve
    # device time per kernel class over one (untimed) solve; the dominant single kernel is
    # chosen among the single-kernel classes
    shares = {}
    for name in ["dgemm", "tc_gemm", "qr_panel", "tridiag", "gje_panel", "eig", "qr", "zside_gemm",
                 "gje_update", "resid_gemm", "newton_update"]:
        G.kernel_timing(name)
        solve()
        shares[name] = G.kernel_stats()
    G.kernel_timing(None)
    single = ["dgemm", "tc_gemm", "qr_panel", "tridiag", "gje_panel"]
    dom = max(single, key=lambda k: shares[k][0])
    # ---- timed region (device time per solve, L2 flushed before each); kernel-class
    # event timing is OFF here (per-launch events would perturb a launch-bound step)
    launches0 = G.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    reports = []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            res = solve()
            ev[i][1].record(stream)
            reports.append(res.report)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = G.launch_count() - launches0
    # ---- roofline pass: the same K solves again with CUDA events around every launch of
    # the dominant kernel (on its launch stream)
    G.kernel_timing(dom)
    for i in range(args.steps):
        flush.fill_(float(i))
        solve()
    torch.cuda.synchronize()
    dom_ms, dom_cnt, dom_flops, dom_bytes = G.kernel_stats()
    G.kernel_timing("tc_gemm")
    for i in range(args.steps):
        solve()
    torch.cuda.synchronize()
    tcs = G.kernel_stats()
    G.kernel_timing(None)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_max = t.item()
    value = world * args.steps / (total_max / 1e3)
    rep = reports[-1]
    # ---- end-to-end through the host-buffer API (H2D of inputs, D2H of the factors)
    A_h = torch.tensor(p.A).pin_memory().numpy()
    L_h = torch.tensor(np.ascontiguousarray(p.L.T)).pin_memory().numpy()
    S_h = torch.tensor(p.S).pin_memory().numpy() if ldlt else None
    solver.solve_host(A_h, L_h, S_h, tol=wl["tol"], maxit=wl["maxit"])
    torch.cuda.synchronize()
    e2e_t = []
    rank_h = 0
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Zh, Yh, rh = solver.solve_host(A_h, L_h, S_h, tol=wl["tol"], maxit=wl["maxit"])
        e2e_t.append(time.perf_counter() - t0)
        rank_h = rh["rank"]
    te = torch.tensor([sum(e2e_t)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * args.steps / te.item()
    h2d = 8 * (n * n + n * m + (m * m if ldlt else 0))
    d2h = 8 * (n * rank_h + (cm * rank_h if ldlt else 0))
    # ---- NCCL gather of the final residual norms (not in the timed data path)
    resid = torch.tensor([rep["final_res"]], dtype=torch.float64, device=dev)
    all_res = [resid.clone() for _ in range(world)]
    if world > 1:
        dist.all_gather(all_res, resid)
    if rank != 0:
        dist.destroy_process_group()
        return 0
    pk = load_peaks()
    # roofline of the dominant single kernel (algorithmic work accumulated per launch by
    # the library, device time from CUDA events around each launch on its stream)
    traffic_all = {}
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        traffic_all = json.load(open(tf))

    def roof(name, ms, cnt, flops, nbytes):
        per_launch_s = ms / max(cnt, 1) / 1e3
        if name == "dgemm":        # fp64 DMMA: measured bf16 peak x nominal fp64:bf16 ratio (40 : 2250)
            peak, unit, bound = pk["bf16_sus"] * 40.0 / 2250.0, "TFLOP/s", "tensor"
            ach = flops / max(cnt, 1) / per_launch_s / 1e12
            src = pk["src"] + " bf16 sustained x 40/2250 (nominal fp64:bf16 dense tensor ratio)"
        elif name == "tc_gemm":
            peak, unit, bound = pk["bf16_sus"], "TFLOP/s", "tensor"
            ach = flops / max(cnt, 1) / per_launch_s / 1e12
            src = pk["src"] + " bf16 sustained"
        else:                      # sequential (reflector / pivot chain) kernels: FMA work vs the ALU peak
            # fp64 FMA peak = 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz = 37.2 TFLOP/s;
            # the Gauss-Jordan panel runs in fp32 (128 FMA/clk/SM): 74.4 TFLOP/s
            fma_per_clk = 128 if name == "gje_panel" else 64
            peak, unit, bound = 148 * fma_per_clk * 2 * 1.965e9 / 1e12, "TFLOP/s", "alu"
            ach = flops / max(cnt, 1) / per_launch_s / 1e12
            src = (f"derived: 148 SMs x {fma_per_clk} FMA/clk x 2 x 1.965 GHz (DESIGN.md); the kernel is "
                   "latency bound by its sequential reflector / pivot chain")
        return {"kernel": name, "bound": bound, "achieved": ach, "peak": peak, "unit": unit,
                "frac": ach / peak if peak else None, "traffic": traffic_all.get(name),
                "algorithmic_per_launch": (flops if unit == "TFLOP/s" else nbytes) / max(cnt, 1),
                "launches_timed": cnt, "avg_launch_us": per_launch_s * 1e6, "peak_source": src}

    roofline = roof(dom, dom_ms, dom_cnt, dom_flops, dom_bytes)
    roofline["measured_over"] = f"a second timed pass of the same {args.steps} solves (events per launch)"
    roofline_sign_newton = roof("tc_gemm", *tcs) if tcs[1] > 0 else None
    # the residual factor's A Z (fp64, Fragments 1/3): its fp64 tensor rate and the HBM rate of
    # its algorithmic bytes (A once, Z in, A Z out); at the ranks configs[1] reaches
    # (c ~ 420) it is a contraction with ~50 flop/byte, i.e. tensor-, not HBM-bound
    rg_ms, rg_cnt, rg_fl, rg_by = shares["resid_gemm"]
    roofline_residual = None
    if rg_cnt > 0 and rg_ms > 0:
        roofline_residual = roof("dgemm", rg_ms, rg_cnt, rg_fl, rg_by)
        roofline_residual["kernel"] = "resid_gemm (A Z, fp64 DMMA)"
        roofline_residual["traffic"] = traffic_all.get("resid_gemm")
        roofline_residual["hbm_gbs_algorithmic"] = rg_by / (rg_ms / 1e3) / 1e9
        roofline_residual["hbm_frac"] = roofline_residual["hbm_gbs_algorithmic"] / pk["hbm"]
        roofline_residual["measured_over"] = "one untimed solve (events per launch)"
    nu_ms, nu_cnt, _, nu_by = shares["newton_update"]
    roofline_newton_update = None
    if nu_cnt > 0 and nu_ms > 0:
        g = nu_by / (nu_ms / 1e3) / 1e9
        roofline_newton_update = {"kernel": "newton_update", "bound": "hbm", "achieved": g, "peak": pk["hbm"],
                                  "unit": "GB/s", "frac": g / pk["hbm"], "launches_timed": nu_cnt,
                                  "algorithmic_per_launch": nu_by / nu_cnt,
                                  "avg_launch_us": nu_ms / nu_cnt * 1e3, "traffic": None,
                                  "measured_over": "one untimed solve (events per launch)"}
    newton_tflops = rep["newton_flops"] / (rep["newton_ms"] / 1e3) / 1e12 if rep["newton_ms"] > 0 else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": wl["us"], "data": "synthetic",
        "config": {"workload": wl["desc"], "n": n, "m": m, "solver_precision": wl["us"],
                   "refinement_precision": "fp64", "tol": wl["tol"], "equations_per_gpu": 1,
                   "l2": "flushed (256 MB write) before every timed step", "parallelism": f"dp{world}"},
        "time_to_solution_ms": total_max / args.steps,
        "ir_steps": rep["steps"], "newton_steps_per_call": rep["newton_steps"],
        "inversions": rep["inversions"], "final_rel_residual": rep["final_res"], "rank": rep["rank"],
        "status": rep["status"],
        "phase_ms": {"newton": rep["newton_ms"], "residual": rep["residual_ms"], "update": rep["update_ms"]},
        "sign_newton_tflops": newton_tflops,
        "sign_newton_frac_of_fp16_peak": (newton_tflops / pk["bf16"]) if newton_tflops else None,
        "roofline_residual": roofline_residual, "roofline_newton_update": roofline_newton_update,
        "kernel_class_ms_one_solve": {k: round(v[0], 4) for k, v in shares.items()},
        "roofline": roofline,
        "roofline_sign_newton_tc_gemm": roofline_sign_newton,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "residuals_all_ranks": [r.item() for r in all_res],
    }
    # the largest configuration's A-sequence is the headline sign-Newton rate
    # (sign_newton_at_scale); configs[2]'s n = 4096 is reported beside it
    if args.scale in ("cfg3", "both"):
        line["sign_newton_at_scale"] = sign_newton_scale(G, P, dev, pk, "cfg3")
    if args.scale in ("cfg2", "both"):
        line["sign_newton_at_scale" if args.scale == "cfg2" else "sign_newton_at_scale_cfg2"] = \
            sign_newton_scale(G, P, dev, pk, "cfg2")
    if args.cfg3 != "none" and world == 1:
        line["time_to_solution_cfg3"] = cfg3_solves(G, P, dev, args.cfg3)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(args.config)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


CFG3_SOLVERS = {
    "fp16": dict(max_cols=4096, newton_cols=8192, work_cols=10240),
    "fp32": dict(max_cols=6144, newton_cols=14336, work_cols=16384),
}


def cfg3_solves(G, P, dev, which):
    """configs[3] (n = 16384, m = 16, convection-diffusion 128 x 128, conv. 50) end to end
    with the fp16 and the fp32 solver: one warm-up solve (workspace, inverse cache), then one
    solve timed with CUDA events on the solver's stream; status, IR steps, residuals, ranks
    and the phase split are the library's report."""
    import numpy as np
    import torch
    p = P.cfg3()
    A = torch.tensor(p.A, dtype=torch.float64, device=dev)
    Lt = torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device=dev)
    out = {"workload": "configs[3]: n=16384 m=16 Cholesky, convection-diffusion 128x128 (conv 50), "
                       "L ~ N(0,1), tol 1e-14, maxit 10"}
    for us in (["fp16", "fp32"] if which == "both" else [which]):
        s = G.Solver(p.n, us=us, **CFG3_SOLVERS[us])
        s.solve(A, Lt, None, tol=1e-14, maxit=10)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = s.solve(A, Lt, None, tol=1e-14, maxit=10)
        e1.record()
        torch.cuda.synchronize()
        rep = r.report
        ms = e0.elapsed_time(e1)
        out[us] = {"ms": ms, "status": rep["status"], "ir_steps": rep["steps"], "inversions": rep["inversions"],
                   "newton_steps_per_call": rep["newton_steps"], "res": rep["res"], "ranks": rep["ranks"],
                   "final_rel_residual": rep["final_res"], "rank": rep["rank"],
                   "phase_ms": {"newton": rep["newton_ms"], "residual": rep["residual_ms"],
                                "update": rep["update_ms"]},
                   "sign_newton_tflops": rep["newton_flops"] / (rep["newton_ms"] / 1e3) / 1e12}
        del s, r
        torch.cuda.empty_cache()
    del A, Lt
    torch.cuda.empty_cache()
    return out


def sign_newton_scale(G, P, dev, pk, which):
    """The sign-Newton A-sequence (the u_s inversions, Eq. newton-lyapu1) at a larger
    configuration's size: TFLOP/s of the whole sequence and of its tensor-core GEMM."""
    import torch
    p = getattr(P, which)()
    n = p.n
    A = torch.tensor(p.A, dtype=torch.float64, device=dev)
    del p
    s = G.Solver(n, us="fp16", max_cols=64)
    out = s.newton_aseq(A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 2
    e0.record()
    for _ in range(reps):
        out = s.newton_aseq(A)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    k = out["steps"]
    flops = k * 2.0 * n ** 3                      # Gauss-Jordan inversion: 2 n^3 per Newton step
    res = {"workload": f"{which}: n={n} fp16 sign-Newton A-sequence ({k} inversions)", "ms": ms,
           "tflops": flops / (ms / 1e3) / 1e12}
    res["frac_of_fp16_peak"] = res["tflops"] / pk["bf16"]
    # per-class event times with the look-ahead stream off: with it the rank-512 update runs
    # beside the next block's panels, and events around a launch would time both
    classes = {}
    os.environ["LYAP_GJE_NO_LOOKAHEAD"] = "1"
    try:
        e0.record()
        s.newton_aseq(A)
        e1.record()
        torch.cuda.synchronize()
        res["ms_without_lookahead"] = e0.elapsed_time(e1)
        for name in ("tc_gemm", "gje_panel", "gje_update"):
            G.kernel_timing(name)
            s.newton_aseq(A)
            classes[name] = G.kernel_stats()
        G.kernel_timing(None)
    finally:
        os.environ.pop("LYAP_GJE_NO_LOOKAHEAD", None)
    ms_t, cnt, fl, _ = classes["tc_gemm"]
    ach = fl / (ms_t / 1e3) / 1e12 if ms_t > 0 else 0.0
    res["tc_gemm"] = {"bound": "tensor", "achieved": ach, "peak": pk["bf16_sus"], "unit": "TFLOP/s",
                      "frac": ach / pk["bf16_sus"], "launches": cnt, "ms": ms_t}
    res["class_ms"] = {k2: v[0] for k2, v in classes.items()}
    res["class_ms_note"] = "serial order (LYAP_GJE_NO_LOOKAHEAD=1); gje_panel = pivot panels + X rows, gje_update = all update GEMMs"
    # the fused Newton averaging update (HBM-streaming: read A_k and the inverse, write
    # A_{k+1} and the cached A_k^{-1}: 4 x 2 n^2 bytes per launch in fp16)
    G.kernel_timing("newton_update")
    s.newton_aseq(A)
    ms_u, cnt_u, _, by_u = G.kernel_stats()
    G.kernel_timing(None)
    gbs = by_u / (ms_u / 1e3) / 1e9 if ms_u > 0 else 0.0
    res["newton_update"] = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm"], "unit": "GB/s",
                            "frac": gbs / pk["hbm"], "launches": cnt_u, "ms": ms_u,
                            "algorithmic_bytes_per_launch": by_u / max(cnt_u, 1)}
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if which == "cfg3" and os.path.exists(tf):
        res["newton_update"]["traffic"] = json.load(open(tf)).get("newton_update_n16384")
    del s, A
    torch.cuda.empty_cache()
    return res


def run_batch(args):
    """configs[4]: independent equations (n=2048, m=4, Cholesky, fp16), sharded over the
    ranks; each rank solves --eq-per-gpu equations per step (a stratified sample over the
    four kappa groups, different members on every rank), --lanes of them concurrently
    (one host thread + solver handle + CUDA stream each)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2510_02126_b200 import batch as B
    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    importlib_build()
    import paper_2510_02126_b200 as G
    import problems as P
    # configs[4] at spec: the 256 equations (four kappa groups of 64) sharded evenly over the
    # ranks (256 / N each); --eq-per-gpu E < 256/N runs a stratified E-member sample instead
    full = B.shard(256, rank, world)
    E = args.eq_per_gpu if args.eq_per_gpu > 0 else len(full)
    if E >= len(full):
        idx = full
    else:
        per_group = max(1, E // 4)
        idx = [g * 64 + (rank * per_group + i) % 64 for g in range(4) for i in range(per_group)][:E]
    E = len(idx)
    probs = [P.cfg4_member(i) for i in idx]
    n = probs[0].n
    lanes = max(1, min(args.lanes, E))
    streams = [torch.cuda.Stream(device=dev) for _ in range(lanes)]
    solvers = []
    for ln in range(lanes):
        with torch.cuda.stream(streams[ln]):
            solvers.append(G.Solver(n, us="fp16", max_cols=args.max_cols))
    dA = [torch.tensor(p.A, dtype=torch.float64, device=dev) for p in probs]
    dL = [torch.tensor(np.ascontiguousarray(p.L.T), dtype=torch.float64, device=dev) for p in probs]
    torch.cuda.synchronize()

    def work(k, ln):
        with torch.cuda.stream(streams[ln]):
            r = solvers[ln].solve(dA[k], dL[k], None, tol=1e-14, maxit=30)
        rep = r.report
        return {"index": idx[k], "steps": rep["steps"], "res": rep["final_res"], "rank": rep["rank"],
                "ok": 1.0 if rep["status"] == "converged" else 0.0}

    items = list(range(E))
    # warm-up: every handle solves once (one-time setup, sequential), then W concurrent passes
    # over a stratified sample of at most 8 of this rank's equations (a full pass is ~1 min)
    warm = sorted(set(items[:: max(1, E // 8)]))[:8]
    for ln in range(lanes):
        work(warm[ln % len(warm)], ln)
    for _ in range(args.warmup):
        B.run_concurrent(work, warm, lanes)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = G.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            results = B.run_concurrent(work, items, lanes)
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
    launches = G.launch_count() - launches0
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    tmax = B.max_over_ranks(ms) if world > 1 else ms
    allres = B.gather_results(results, ["index", "steps", "res", "rank", "ok"]) if world > 1 else results
    # end to end: host (pinned) inputs, factors read back, same concurrency
    hA = [torch.tensor(p.A).pin_memory().numpy() for p in probs]
    hL = [torch.tensor(np.ascontiguousarray(p.L.T)).pin_memory().numpy() for p in probs]
    ranks_h = []

    def work_h(k, ln):
        with torch.cuda.stream(streams[ln]):
            Z, _, rep = solvers[ln].solve_host(hA[k], hL[k], None, tol=1e-14, maxit=30)
        return {"rank": rep["rank"]}
    t0 = time.perf_counter()
    rh = B.run_concurrent(work_h, items, lanes)
    te = time.perf_counter() - t0
    te = B.max_over_ranks(te) if world > 1 else te
    if rank != 0:
        dist.destroy_process_group()
        return 0
    value = world * E * args.steps / (tmax / 1e3)
    h2d = sum(8 * (n * n + n * p.m) for p in probs)
    d2h = sum(8 * n * r["rank"] for r in rh)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tmax / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp16", "data": "synthetic",
        "config": {"workload": f"configs[4] batch: n=2048 m=4 Cholesky fp16, {E} equations per GPU per step "
                               f"({world * E} of 256 per step, kappa groups 1e1..1e4), {lanes} concurrent "
                               f"solver handles/streams per GPU; warm-up = {args.warmup} passes over "
                               f"{len(warm)} of them",
                   "n": n, "equations_per_gpu": E, "lanes": lanes, "parallelism": f"dp{world}",
                   "l2": "inputs (32 MB A per equation) exceed L2 together; no flush"},
        "equations": allres, "all_converged": all(r["ok"] == 1.0 for r in allres),
        "e2e": {"value": world * E / te, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def importlib_build():
    import importlib
    b = importlib.import_module("paper_2510_02126_b200.build")
    b.build()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg1", choices=sorted(WORKLOADS) + ["cfg4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eq-per-gpu", type=int, default=0,
                    help="configs[4]: equations per GPU per step (0 = 256 / N, the full batch)")
    ap.add_argument("--lanes", type=int, default=6, help="configs[4]: concurrent solver handles per GPU")
    ap.add_argument("--max-cols", type=int, default=1536, help="configs[4]: factor capacity per handle")
    ap.add_argument("--cfg3", default="both", choices=["none", "fp16", "fp32", "both"],
                    help="also solve configs[3] end to end with these solver precisions (rank 0 of N=1)")
    ap.add_argument("--scale", default="both", choices=["none", "cfg2", "cfg3", "both"],
                    help="also time the fp16 sign-Newton A-sequence at this configuration's n (rank 0)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl != "reference":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "cfg4":
        return run_batch(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
