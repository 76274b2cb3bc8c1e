#!/usr/bin/env python3
"""Benchmark of the B200 preconditioned-GMRES path on BASELINE.json's workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

A step is one GMRES(50) solve (tol 1e-10, block-triangular preconditioner) of BASELINE config 1
(1D, M=4095 interior points, N=512 time steps; all-at-once dimension 2,100,735).  Setup
(operator assembly, preconditioner build, forward solve for mu, noise) is untimed.

  value  GMRES iterations/s, device-resident right-hand side (CUDA events on the library stream)
  e2e    the same metric through the reference-facing host call fi_gmres_host: pinned host b,
         H2D + solve + D2H of x inside the timed region
  roofline  the dominant kernel (K2, the preconditioner sweep, HBM-bound) timed live with CUDA
         events on the library stream; roofline_operator = K1 (FP64 DMMA-bound)
  cpu_baseline  the CPU oracle (numpy/scipy restatement of the reference) on a bounded sample

Multi-GPU: the solve does not shard — N ranks run N independent replicas
(weak scaling); value = all ranks' iterations / max-over-ranks time.
--impl reference times the reference algorithm's CPU restatement (the reference itself needs
Eigen/FFTW, absent here) on the host cores; under torchrun only rank 0 works.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GMRES time-to-solve & iters/s; operator-apply FP64 TFLOP/s as % of roofline"
FP64_DMMA_PEAK_TFLOPS = 37.0  # measured: profiles/fp64_peak_r01.jsonl (register-only DMMA loop, best of 10)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md 6.65 TB/s"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def replica_aggregate(ms, work, device=None):
    """(max over ranks of the timed milliseconds, sum over ranks of the work units).
    Identity on one process; any torch.distributed backend (nccl on GPUs, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(ms), float(work)
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    w = torch.tensor([float(work)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(w, op=dist.ReduceOp.SUM)
    return float(t.item()), float(w.item())


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------------------------- CPU baseline (oracle)
def cpu_reference_sample(cfg: int, iters_hint: int, seconds_budget: float = 20.0):
    """Time the reference algorithm's CPU restatement on a bounded sample of config `cfg` and
    extrapolate GMRES iterations/s (= 1 / (A-apply + P-apply + MGS step)).

    P-apply = S+1 dense LU solves + the O(S^2 N) history (krylov.cpp:48-70); its LU factors
    (68.8 GB for config 1) are built for a uniform sample of levels only and the per-level
    solve time is scaled to all levels.  A-apply is timed whole (FFT matvecs, system.cpp:144-174).
    """
    import scipy.linalg as sla

    from oracle import fracinv_oracle as O
    from paper_2507_02809_b200.configs import baseline_problem

    t_setup = time.perf_counter()
    A = O.SystemOperator(baseline_problem(O, cfg))
    N, S = A.N, A.steps
    rng = np.random.default_rng(0)
    v = rng.uniform(-1, 1, A.dim)
    A.apply(v)  # warm-up (plans, E matrix)
    t_apply = float("inf")
    for _ in range(2):
        t0 = time.perf_counter()
        A.apply(v)
        t_apply = min(t_apply, time.perf_counter() - t0)

    # sample of levels for the P-apply: factor + solve incl. history sums
    nsamp = 24 if S > 64 else S + 1
    levels = sorted(set(int(round(x)) for x in np.linspace(1, S + 1, nsamp)))
    Bd = A.laplacian.dense(N)
    e = A.weights.e
    Y = rng.uniform(-1, 1, (S, N))
    t_fact = t_solve = 0.0
    for s in levels:
        if s <= S:
            blk = A.scale_space * A.diags.D2[s - 1][:, None] * Bd
            blk[np.diag_indices(N)] += e[0] * A.diags.D1[s - 1]
        else:
            blk = A.scale_reg * A.diags.D2[S - 1][:, None] * Bd
        t0 = time.perf_counter()
        lu = sla.lu_factor(blk, check_finite=False)
        t_fact += time.perf_counter() - t0
        t0 = time.perf_counter()
        rhs = v[:N].copy()
        if 1 < s <= S:
            rhs -= A.diags.D1[s - 1] * (e[s - 1:0:-1] @ Y[: s - 1])
        sla.lu_solve(lu, rhs, check_finite=False)
        t_solve += time.perf_counter() - t0
    t_P = t_solve / len(levels) * (S + 1)
    t_build = t_fact / len(levels) * (S + 1)
    # one MGS step at k = iters_hint/2 (dots + axpys over the (S+1)N vector)
    k = max(1, iters_hint // 2)
    w = v.copy()
    V = rng.uniform(-1, 1, (2, A.dim))
    t0 = time.perf_counter()
    for i in range(k + 1):
        h = V[i % 2] @ w
        w -= h * V[i % 2]
    t_mgs = time.perf_counter() - t0
    t_iter = t_apply + t_P + t_mgs
    return {
        "iters_per_s": 1.0 / t_iter,
        "time_per_iteration_s": t_iter,
        "a_apply_s": t_apply,
        "p_apply_s_extrapolated": t_P,
        "p_build_s_extrapolated": t_build,
        "mgs_step_s": t_mgs,
        "cores": os.cpu_count(),
        "sample": (f"config {cfg}: 1 full A-apply (FFT), P-apply from {len(levels)} of {S + 1} levels' dense LU "
                   f"factor+solve scaled to all levels, 1 MGS step at k={k}; iters/s = 1/(A+P+MGS); "
                   f"wall {time.perf_counter() - t_setup:.1f}s"),
    }


# --------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from oracle import fracinv_oracle as O  # noqa: F401  (cpu_baseline leg only)
    from paper_2507_02809_b200 import fracinv as F
    from paper_2507_02809_b200.configs import NAMES, NOISE, RESTART, SEED_BASE, TOL, baseline_problem

    cfg = args.config
    ctx = F.Context(local if ws > 1 else 0)
    t0 = time.perf_counter()
    spec = baseline_problem(F, cfg)
    A = F.SystemOperator(spec, ctx=ctx)
    t_asm = time.perf_counter() - t0
    t0 = time.perf_counter()
    P = F.BlockTriangularPreconditioner(A)
    t_pbuild = time.perf_counter() - t0
    t0 = time.perf_counter()
    mu = F.forward_solve(A, P).mu
    t_fwd = time.perf_counter() - t0
    mu_eps = F.add_gaussian_noise(mu, NOISE[cfg], SEED_BASE + cfg + rank)
    z = F.build_rhs(A, mu_eps).z
    opts = F.GmresOptions(TOL[cfg], 0, RESTART)
    n = A.dim()

    stream = torch.cuda.ExternalStream(ctx.stream)
    b_dev = torch.from_numpy(z).to(f"cuda:{ctx.device}")
    torch.cuda.synchronize()

    def solve_dev():
        return F.gmres(A, P, b_dev, opts)

    # warm-up
    for _ in range(args.warmup):
        x, rep = solve_dev()
    f_star = spec.f_true
    recon_err = F.relative_error(f_star, x[-A.N:].cpu().numpy())

    # ---- timed region: device-resident value
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = ctx.kernel_launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    iters = []
    if args.profile:  # ncu --profile-from-start off captures exactly the timed region
        torch.cuda.cudart().cudaProfilerStart()
    ev0.record(stream)
    for _ in range(args.steps):
        x, rep = solve_dev()
        iters.append(rep.iterations)
    ev1.record(stream)
    torch.cuda.synchronize()
    if args.profile:
        torch.cuda.cudart().cudaProfilerStop()
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms_total = ev0.elapsed_time(ev1)
    launches = ctx.kernel_launches - launches0
    total_iters = sum(iters)

    # the same solves with the Arnoldi step in the reference's order (K1 operator apply, then P^{-1})
    # instead of the default split P^{-1} A v = v + P^{-1}((A - P) v)
    A.set_split_apply(False)
    solve_dev()
    torch.cuda.synchronize()
    ev0.record(stream)
    u_iters = 0
    for _ in range(args.steps):
        _, rep_u = solve_dev()
        u_iters += rep_u.iterations
    ev1.record(stream)
    torch.cuda.synchronize()
    ms_unsplit = ev0.elapsed_time(ev1)
    A.set_split_apply(True)

    # ---- e2e: host (pinned) b -> fi_gmres_host -> host x
    b_host = torch.from_numpy(z).pin_memory()
    x_host = torch.empty(n, dtype=torch.float64).pin_memory()
    import ctypes

    from paper_2507_02809_b200._lib import GmresOpts, GmresReport, last_error, lib
    o = GmresOpts(opts.tol, opts.maxit, opts.restart)
    r = GmresReport()
    hist = np.zeros(4096)
    dp = lambda t: ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_double))
    e_iters = 0
    for _ in range(max(1, args.warmup)):  # untimed: first-call staging allocation, warm caches
        rc = lib.fi_gmres_host(A.handle, P.handle, dp(b_host), None, dp(x_host), ctypes.byref(o), ctypes.byref(r),
                               hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 4096)
        assert rc == 0, last_error()
    # three timed passes of K solves each; the median pass is reported (a host-side hiccup in one
    # pass, e.g. the thread descheduled while it waits on the look-ahead event, would otherwise
    # decide the number)
    passes = []
    for _ in range(3):
        torch.cuda.synchronize()
        e_iters = 0
        ev0.record(stream)
        for _ in range(args.steps):
            rc = lib.fi_gmres_host(A.handle, P.handle, dp(b_host), None, dp(x_host), ctypes.byref(o), ctypes.byref(r),
                                   hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 4096)
            assert rc == 0, last_error()
            e_iters += r.iterations
        ev1.record(stream)
        torch.cuda.synchronize()
        passes.append((ev0.elapsed_time(ev1), e_iters))
    ms_e2e, e_iters = sorted(passes)[1]

    # ---- roofline: K2 preconditioner sweep (dominant) and K1 operator, live CUDA events
    reps = 5
    y = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).to(b_dev.device)
    out = torch.empty_like(y)
    ms = ctypes.c_double()
    form = P.form
    # P^{-1} as the solve uses it: the inverses are polished at build, so one
    # sweep (one hodlr_sweep_kernel or sweep_kernel launch) with refinement off; the refined apply
    # (second sweep + K1 residual) is reported beside it
    P.set_refine(True)
    assert lib.fi_precond_apply_timed(P.handle, y.data_ptr(), out.data_ptr(), reps, ctypes.byref(ms)) == 0
    ms_refined = ms.value
    P.set_refine(False)
    assert lib.fi_precond_apply_timed(P.handle, y.data_ptr(), out.data_ptr(), reps, ctypes.byref(ms)) == 0
    ms_papply = ms_sweep = ms.value
    assert lib.fi_system_apply_timed(A.handle, y.data_ptr(), out.data_ptr(), reps, ctypes.byref(ms)) == 0
    ms_op = ms.value
    # K3: one MGS round (w -= c x; h = y.w) over three Krylov-length vectors, L2 flushed before each
    mw, mx, my = (torch.from_numpy(np.random.default_rng(k).uniform(-1, 1, n)).to(b_dev.device) for k in (5, 6, 7))
    assert lib.fi_mgs_round_timed(ctx.handle, n, mw.data_ptr(), mx.data_ptr(), my.data_ptr(), reps,
                                  ctypes.byref(ms)) == 0
    ms_mgs = ms.value
    del mw, mx, my

    N, S = A.N, A.S
    Np = ((N + 63) // 64) * 64 if spec.sgrid.d == 1 else spec.sgrid.n[0] * ((spec.sgrid.n[1] + 63) // 64) * 64
    nb = Np // 64
    T = nb * (nb + 1) // 2
    if form == "hodlr":
        # algorithmic bytes of one sweep: every level's HODLR rows once
        # (fi_precond_bytes: 64 leaf + 32 per ancestor doubles per row) + z, D1, 1/D2 read, y written
        sweep_bytes = int(P.device_bytes()) + 4 * 8 * Np * (S + 1)
        sweep_kernel = "hodlr_sweep_kernel (K2: substitution over HODLR inverses; chain of S+1 dependent levels)"
    else:
        # the packed lower-triangular FP64 tiles of all S+1 levels once, plus per level row z, D1, 1/D2
        # read and y written
        sweep_bytes = (S + 1) * T * 64 * 64 * 8 + 4 * 8 * Np * (S + 1)
        sweep_kernel = "sweep_kernel (K2: FP64 substitution over packed tiles)"
    hbm_peak, peak_src = load_peaks()
    achieved = sweep_bytes / (ms_sweep * 1e-3) / 1e9
    op_flops = 2.0 * N * N * (S + 1)
    op_tflops = op_flops / (ms_op * 1e-3) / 1e12

    # max over ranks for times, sum over ranks for the work done (replicas)
    ms_total_max, iters_all = replica_aggregate(ms_total, total_iters, b_dev.device)
    ms_e2e_max, e_iters_all = replica_aggregate(ms_e2e, e_iters, b_dev.device)
    value = iters_all / (ms_total_max * 1e-3)
    e2e_value = e_iters_all / (ms_e2e_max * 1e-3)
    ms_unsplit_max, u_iters_all = replica_aggregate(ms_unsplit, u_iters, b_dev.device)
    value_unsplit = u_iters_all / (ms_unsplit_max * 1e-3)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_reference_sample(cfg, max(iters))

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "iters/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_total_max / args.steps, 3),
            "time_to_solve_s": round(ms_total_max / args.steps * 1e-3, 5),
            "iterations_per_solve": iters[-1],
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (BASELINE.json config, manufactured mu via forward solve, seeded Gaussian noise)",
            "config": {
                "workload": NAMES[cfg],
                "M": N, "N_t": S, "dim": n, "restart": RESTART, "tol": TOL[cfg], "precond": "block-triangular",
                "noise": f"{NOISE[cfg] * 100:g}% gaussian rel-L2 seed {SEED_BASE + cfg}",
                "l2": ("inputs larger than L2: each P apply streams the HODLR inverses once (%.1f GB)"
                       % (P.device_bytes() / 1e9) if form == "hodlr" else
                       "inputs larger than L2: each P apply streams the packed FP64 tiles once (%.1f GB)"
                       % ((S + 1) * T * 64 * 64 * 8 / 1e9)),
                "parallelism": f"replicas x{ws}",
                "recon_error_vs_fstar": recon_err,
                "final_true_residual": rep.final_true_residual,
                "setup_s": {"assembly": round(t_asm, 3), "precond_build": round(t_pbuild, 3),
                            "forward_solve": round(t_fwd, 3)},
            },
            "e2e": {"value": round(e2e_value, 3), "unit": "iters/s", "h2d_bytes_per_step": 8 * n,
                    "d2h_bytes_per_step": 8 * n, "timing": "median of 3 timed passes of K solves"},
            "gpu_launches": int(launches),
            "arnoldi_step": "split: P^-1 A v = v + P^-1((A - P) v), one preconditioner sweep per step (exact identity)",
            "value_operator_then_precond": {"value": round(value_unsplit, 3), "unit": "iters/s",
                                            "iterations_per_solve": rep_u.iterations,
                                            "note": "reference order: K1 operator apply, then P^-1, every Arnoldi step"},
            "roofline": {"bound": "hbm", "kernel": sweep_kernel,
                         "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4), "traffic": None,
                         "bytes_per_launch": sweep_bytes, "ms_per_launch": round(ms_sweep, 4),
                         "us_per_level": round(ms_sweep * 1e3 / (S + 1), 3),
                         # the level chain's floor: one all-to-all exchange round among the sweep's 128
                         # CTAs, 1785 cycles = 0.91 us at 1965 MHz (tools/xchg_latency.cu,
                         # profiles/xchg_latency_r01.txt)
                         "exchange_floor_us_per_level": 0.908, "precond_form": form,
                         "peak_source": peak_src},
            "roofline_arnoldi": {"bound": "hbm", "kernel": "reduce_kernel (K3: one MGS round, fused axpy + dot)",
                                 "achieved": round(32.0 * n / (ms_mgs * 1e-3) / 1e9, 1), "peak": hbm_peak,
                                 "unit": "GB/s", "frac": round(32.0 * n / (ms_mgs * 1e-3) / 1e9 / hbm_peak, 4),
                                 "bytes_per_launch": 32 * n, "ms_per_launch": round(ms_mgs, 5),
                                 "note": "w read + written, v_(i-1) and v_i read; L2 flushed before each timed round"},
            "roofline_operator": {"bound": "tensor", "kernel": "toeplitz_apply_kernel (K1, FP64 DMMA)",
                                  "achieved": round(op_tflops, 3), "peak": FP64_DMMA_PEAK_TFLOPS,
                                  "unit": "TFLOP/s", "frac": round(op_tflops / FP64_DMMA_PEAK_TFLOPS, 4),
                                  "flops_per_launch": op_flops, "ms_per_launch": round(ms_op, 4),
                                  "peak_source": "profiles/fp64_peak_r01.jsonl (measured DMMA loop)"},
            "precond_apply_ms": round(ms_papply, 4),
            "precond_apply_refined_ms": round(ms_refined, 4),
            "clocks": clocks,
        }
        if cpu is not None:
            line["cpu_baseline"] = {"value": round(cpu["iters_per_s"], 5), "unit": "iters/s", "cores": cpu["cores"],
                                    "kind": "port", "sample": cpu["sample"],
                                    "time_per_iteration_s": round(cpu["time_per_iteration_s"], 3),
                                    "p_build_s_extrapolated": round(cpu["p_build_s_extrapolated"], 1)}
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from paper_2507_02809_b200.configs import NAMES, RESTART, TOL
    samples = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference_sample(args.config, args.iters_hint)
        if i >= args.warmup:
            samples.append(r)
    v = float(np.mean([s["iters_per_s"] for s in samples]))
    t_iter = float(np.mean([s["time_per_iteration_s"] for s in samples]))
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 5),
        "unit": "iters/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_iter * 1e3, 1),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": NAMES[args.config], "restart": RESTART, "tol": TOL[args.config],
                   "note": "CPU restatement of the reference (oracle/, numpy+scipy); the reference needs "
                           "Eigen3/FFTW3 which are absent, so it cannot be built here"},
        "cpu_baseline": {"value": round(v, 5), "unit": "iters/s", "cores": samples[-1]["cores"], "kind": "port",
                         "sample": samples[-1]["sample"]},
        "e2e": {"value": round(v, 5), "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--iters-hint", type=int, default=12, help="GMRES iterations per solve assumed by the CPU arm")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="bracket the timed region with cudaProfilerStart/Stop")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: the contract requires >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
