#!/usr/bin/env python3
"""Benchmark of the B200 preconditioned-GMRES path on BASELINE.json's workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

A step is one GMRES(50) solve with the block-triangular preconditioner of BASELINE config 4 by
default — the largest single-GPU configuration (2D, 255 x 255 interior points, N = 512 time steps;
all-at-once dimension 33,357,825; tol 1e-8).  Setup (operator assembly, preconditioner build, forward
solve for mu, noise) is untimed.

  value  GMRES iterations/s of the device-resident solve (CUDA events on the library stream)
  e2e    the same metric through the reference-facing host call fi_gmres_host: pinned host b,
         H2D + solve + D2H of x inside the timed region
  roofline  the dominant kernel of the solve, timed live with CUDA events on the library stream:
         for the 2D configs the tau-PCG forward substitution (tau_pcg_fused, K5) on the input an
         Arnoldi step feeds it; roofline_operator = K1 (FP64 DMMA), roofline_arnoldi = one MGS round
  configs  time-to-solve and iterations/s of every BASELINE config (one solve each after a warm-up)
         and of the unpreconditioned config-4 solve (one GMRES(50) cycle timed)
  cpu_baseline  the CPU oracle (numpy/scipy restatement of the reference) on a bounded sample of
         the same workload, at 1 core (the reference is single-threaded) and at all cores

Multi-GPU: the solve does not shard — N ranks run N independent replicas
(weak scaling); value = all ranks' iterations / max-over-ranks time.
--impl reference times the reference algorithm's CPU restatement (the reference itself needs
Eigen/FFTW, absent here) on all host cores; under torchrun only rank 0 works.  It never imports the
product library (paper_2507_02809_b200.configs is pure Python and the package loads the .so lazily).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GMRES time-to-solve & iters/s; operator-apply FP64 TFLOP/s as % of roofline"
DEFAULT_CONFIG = 4


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md 6.65 TB/s"


def load_traffic(kernel, cfg):
    """DRAM bytes per launch of `kernel` from the committed ncu capture (profiles/r02/ncu_traffic.json) when it
    was taken on this configuration, else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")) as f:
            e = json.load(f).get(kernel)
        return (int(e["bytes"]), "profiles/r02/ncu_traffic.json: " + e["report"]) if e and e["config"] == cfg else (None, None)
    except Exception:
        return None, None


def load_fp64_peak():
    with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
        p = json.load(f)
    return float(p[p["roofline_peak"]]), "profiles/fp64_peak.json " + p["roofline_peak"] + " (measured DMMA loop)"


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


def workload_config(cfg: int, ws: int = 1) -> dict:
    """The config keys of the JSON line — identical in both arms (no measured quantities)."""
    from paper_2507_02809_b200.configs import NAMES, NOISE, RESTART, SEED_BASE, SHAPES, TOL
    n, S = SHAPES[cfg]
    N = int(np.prod(n))
    return {"workload": NAMES[cfg], "M": "x".join(str(v) for v in n), "N_t": S, "dim": (S + 1) * N,
            "restart": RESTART, "tol": TOL[cfg], "precond": "block-triangular",
            "noise": f"{NOISE[cfg] * 100:g}% gaussian rel-L2 seed {SEED_BASE + cfg}",
            "l2": ("inputs larger than L2: every solve streams Krylov vectors of %.0f MB and the operator's "
                   "%.0f MB of coefficient fields" % (8e-6 * (S + 1) * N, 8e-6 * 2 * S * N)
                   if 8 * (S + 1) * N > 126e6 else
                   "the working set is not flushed from L2 between solves (Krylov vectors of %.1f MB)"
                   % (8e-6 * (S + 1) * N)),
            "parallelism": f"replicas x{ws}"}


def golden_iterations(cfg: int, default: int = 12) -> int:
    try:
        return int(np.load(os.path.join(ROOT, "tests", "golden", f"oracle_config{cfg}.npz"))["iterations"])
    except Exception:
        return default


# --------------------------------------------------------------------------- CPU baseline (oracle)
def cpu_reference_sample(cfg: int, iters: int, threads: int, nlev: int = 12):
    """Time the reference algorithm's CPU restatement (oracle/) on a bounded sample of config `cfg`
    with `threads` host threads (BLAS pool and FFT workers) and extrapolate GMRES iterations/s
    (= 1 / (A-apply + P-apply + MGS step), the reference's order: krylov.cpp:123-132).

    A-apply: one whole apply (system.cpp:144-174).  P-apply (krylov.cpp:48-70): the first `nlev` time
    levels of the forward substitution on the input an Arnoldi step feeds P (A v with v the f-block
    direction), timed level by level with the oracle's own per-block solve (dense LU, or the
    substituted tau-PCG with its warm start); the remaining levels are extrapolated with the mean of the
    levels that already have the full warm start, plus the history sum at its true length.
    """
    import threadpoolctl

    from oracle import fracinv_oracle as O
    from paper_2507_02809_b200.configs import baseline_problem

    t_wall = time.perf_counter()
    O.FFT_WORKERS = threads
    with threadpoolctl.threadpool_limits(threads):
        A = O.SystemOperator(baseline_problem(O, cfg))
        N, S = A.N, A.steps
        rng = np.random.default_rng(0)
        v = rng.uniform(-1, 1, A.dim)
        A.apply(v)  # warm-up (E matrix)
        t0 = time.perf_counter()
        A.apply(v)
        t_apply = time.perf_counter() - t0
        dense = not (A.spec.sgrid.d == 2 and N > 4096)
        e = A.weights.e
        D1 = A.diags.D1
        t_build = 0.0
        if dense:
            P = O.BlockTriangularPreconditioner(A, cache=False, inner="lu") if N > 2048 else \
                O.BlockTriangularPreconditioner(A, inner="lu")
        else:
            P = O.BlockTriangularPreconditioner(A, inner="pcg")
        # the preconditioner's input in the first Arnoldi step: A v0 with v0 = P^{-1} b / |P^{-1} b|.  The
        # time rows of b are b_{s-1} D1 rho (zero for the 2D configs), so v0 is (nearly) the f-block solve
        # of the observation: v0 ~ [0; G_f^{-1} mu_eps]
        try:
            mu_eps = np.load(os.path.join(ROOT, "tests", "golden", f"oracle_config{cfg}.npz"))["mu_eps"]
        except Exception:
            mu_eps = A.spec.f_true
        fv = P.solve_block(S + 1, mu_eps)
        u = np.zeros(A.dim)
        u[S * N:] = fv / np.linalg.norm(fv)
        z = A.apply(u)
        if dense:
            # dense blocks: factor (untimed build) and time the solves of a uniform sample of levels
            levels = sorted(set(int(round(x)) for x in np.linspace(1, S + 1, min(nlev, S + 1))))
            Y = rng.uniform(-1, 1, (S, N))
            t_solve = 0.0
            for s in levels:
                t0 = time.perf_counter()
                lu = P._factor(s)
                t_build += time.perf_counter() - t0
                t0 = time.perf_counter()
                rhs = z[(s - 1) * N: s * N].copy()
                if 1 < s <= S:
                    rhs -= D1[s - 1] * (e[s - 1:0:-1] @ Y[: s - 1])
                O.sla.lu_solve(lu, rhs, check_finite=False)
                t_solve += time.perf_counter() - t0
            t_P = t_solve / len(levels) * (S + 1)
            t_build = t_build / len(levels) * (S + 1)
            how = f"P: {len(levels)} of {S + 1} levels' dense LU solves (factors built untimed) scaled to all levels"
        else:
            P.pcg.dropped = False
            P.pcg.iterations = []
            k = min(nlev, S)
            Y = np.zeros((k, N))
            t_solve, t_hist_l = [], []
            for s in range(1, k + 1):
                t0 = time.perf_counter()
                rhs = z[(s - 1) * N: s * N].copy()
                if s > 1:
                    rhs -= D1[s - 1] * (e[s - 1:0:-1] @ Y[: s - 1])
                t1 = time.perf_counter()
                Y[s - 1] = P.solve_block(s, rhs, [Y[s - 1 - j] for j in range(1, min(O.WARM_ORDER, s - 1) + 1)])
                t_solve.append(time.perf_counter() - t1)
                t_hist_l.append(t1 - t0)
            its = list(P.pcg.iterations[:k])
            # per-level solve time = b * (CG steps + 1): a level's fixed work (the warm start's B x0 and the first
            # tau solve) is one step's worth.  A two-parameter least-squares fit is ill-conditioned over the
            # narrow step range of the first levels (24 .. 17 on config 4) and, with many threads, traded the
            # per-step cost for a large spurious fixed cost that dominated the extrapolation.
            b_step = float(np.sum(t_solve)) / float(np.sum(np.array(its) + 1))
            a_fix = b_step
            # the oracle's own CG step counts of every level on this input (tests/golden/gen_pcg_steps.py)
            try:
                steps = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_pcg_steps.json")))[str(cfg)]
                counts = steps["steps_per_level"]
                src = "per-level CG step counts of the oracle's full apply (tests/golden/oracle_pcg_steps.json)"
            except Exception:
                counts = its + [its[-1]] * (S + 1 - k)
                src = "the last sampled level's CG step count for the unsampled levels"
            # the history sum at full depth (S - 1 previous levels), scaled linearly in s
            Yh = rng.uniform(-1, 1, (S - 1, N))
            t0 = time.perf_counter()
            _ = e[S - 1:0:-1] @ Yh
            t_hist = time.perf_counter() - t0
            del Yh
            t_P = sum(a_fix + b_step * c for c in counts) + sum(t_hist * s / S for s in range(2, S + 1))
            how = (f"P: the first {k} of {S} time levels of the tau-PCG substitution timed level by level "
                   f"(CG steps {its}; {b_step * 1e3:.2f} ms per CG step, a level's setup counted as one step), "
                   f"extrapolated to all {S + 1} levels with {src} ({sum(counts)} steps) plus the L1 history sum "
                   f"at its true length")
        # one MGS step at k = iters/2 (k+1 dots + axpys over the (S+1)N vector, krylov.cpp:127-132)
        kk = max(1, iters // 2)
        w = v.copy()
        V = rng.uniform(-1, 1, (2, A.dim))
        tmp = np.empty_like(w)
        t0 = time.perf_counter()
        for i in range(kk + 1):
            h = float(V[i % 2] @ w)
            np.multiply(V[i % 2], h, out=tmp)
            np.subtract(w, tmp, out=w)
        t_mgs = time.perf_counter() - t0
    t_iter = t_apply + t_P + t_mgs
    return {
        "iters_per_s": 1.0 / t_iter,
        "time_per_iteration_s": t_iter,
        # the reference's time-to-solve: iters Arnoldi steps + P^{-1} b + the final true residual's A x
        "time_to_solve_s_extrapolated": iters * t_iter + t_P + t_apply,
        "a_apply_s": t_apply,
        "p_apply_s_extrapolated": t_P,
        "p_build_s_extrapolated": t_build,
        "mgs_step_s": t_mgs,
        "cores": threads,
        "sample": (f"config {cfg} with {threads} host thread(s): 1 full A-apply (FFT); {how}; 1 MGS step at "
                   f"k={kk}; iters/s = 1/(A+P+MGS); wall {time.perf_counter() - t_wall:.1f}s"),
    }


def cpu_baseline_entry(cfg, iters):
    one = cpu_reference_sample(cfg, iters, 1)
    n = os.cpu_count() or 1
    alln = cpu_reference_sample(cfg, iters, n)
    return {"value": round(one["iters_per_s"], 6), "unit": "iters/s", "cores": 1, "kind": "port",
            "sample": one["sample"], "time_per_iteration_s": round(one["time_per_iteration_s"], 3),
            "time_to_solve_s_extrapolated": round(one["time_to_solve_s_extrapolated"], 2),
            "all_cores": {"value": round(alln["iters_per_s"], 6), "cores": n,
                          "time_per_iteration_s": round(alln["time_per_iteration_s"], 3),
                          "time_to_solve_s_extrapolated": round(alln["time_to_solve_s_extrapolated"], 2),
                          "sample": alln["sample"]}}


# --------------------------------------------------------------------------- GPU arm
def build_case(F, ctx, cfg, seed_offset=0):
    from paper_2507_02809_b200.configs import NOISE, SEED_BASE, baseline_problem
    t0 = time.perf_counter()
    spec = baseline_problem(F, cfg)
    A = F.SystemOperator(spec, ctx=ctx)
    t_asm = time.perf_counter() - t0
    t0 = time.perf_counter()
    P = F.BlockTriangularPreconditioner(A, inner="auto")
    ctx.synchronize()
    t_pb = time.perf_counter() - t0
    t0 = time.perf_counter()
    mu = F.forward_solve(A, P).mu
    t_fwd = time.perf_counter() - t0
    mu_eps = F.add_gaussian_noise(mu, NOISE[cfg], SEED_BASE + cfg + seed_offset)
    z = F.build_rhs(A, mu_eps).z
    return spec, A, P, z, {"assembly": round(t_asm, 3), "precond_build": round(t_pb, 3),
                           "forward_solve": round(t_fwd, 3)}


def time_solves(F, A, P, b_dev, opts, stream, steps):
    import torch
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    its = 0
    ev0.record(stream)
    for _ in range(steps):
        x, rep = F.gmres(A, P, b_dev, opts)
        its += rep.iterations
    ev1.record(stream)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1), its, x, rep


def run_ours(args):
    import ctypes

    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2507_02809_b200 import fracinv as F
    from paper_2507_02809_b200._lib import GmresOpts, GmresReport, last_error, lib
    from paper_2507_02809_b200.configs import NAMES, RESTART, TOL

    cfg = args.config
    ctx = F.Context(local if ws > 1 else 0)
    spec, A, P, z, setup_s = build_case(F, ctx, cfg, rank)
    opts = F.GmresOptions(TOL[cfg], 0, RESTART)
    n = A.dim()
    stream = torch.cuda.ExternalStream(ctx.stream)
    b_dev = torch.from_numpy(z).to(f"cuda:{ctx.device}")
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        x, rep = F.gmres(A, P, b_dev, opts)
    recon_err = F.relative_error(spec.f_true, x[-A.N:].cpu().numpy())

    # ---- timed region: device-resident value
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = ctx.kernel_launches
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    if args.profile:  # ncu --profile-from-start off captures exactly the timed region
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    ms_total, total_iters, x, rep = time_solves(F, A, P, b_dev, opts, stream, args.steps)
    if args.profile:
        torch.cuda.cudart().cudaProfilerStop()
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop()
    launches = ctx.kernel_launches - launches0

    # the same solve with the Arnoldi step in the reference's order (K1 operator apply, then P^{-1})
    # instead of the default split P^{-1} A v = v + P^{-1}((A - P) v)
    A.set_split_apply(False)
    F.gmres(A, P, b_dev, opts)
    ms_unsplit, u_iters, _, rep_u = time_solves(F, A, P, b_dev, opts, stream, max(1, min(2, args.steps)))
    A.set_split_apply(True)

    # ---- e2e: host (pinned) b -> fi_gmres_host -> host x
    b_host = torch.from_numpy(z).pin_memory()
    x_host = torch.empty(n, dtype=torch.float64).pin_memory()
    o = GmresOpts(opts.tol, opts.maxit, opts.restart)
    r = GmresReport()
    hist = np.zeros(4096)
    dp = lambda t: ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_double))
    hp = hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    for _ in range(max(1, min(args.warmup, 2))):  # untimed: first-call staging allocation
        assert lib.fi_gmres_host(A.handle, P.handle, dp(b_host), None, dp(x_host), ctypes.byref(o), ctypes.byref(r),
                                 hp, 4096) == 0, last_error()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    passes = []
    for _ in range(3):  # median of three timed passes of K solves
        torch.cuda.synchronize()
        e_iters = 0
        ev0.record(stream)
        for _ in range(args.steps):
            rc = lib.fi_gmres_host(A.handle, P.handle, dp(b_host), None, dp(x_host), ctypes.byref(o), ctypes.byref(r),
                                   hp, 4096)
            assert rc == 0, last_error()
            e_iters += r.iterations
        ev1.record(stream)
        torch.cuda.synchronize()
        passes.append((ev0.elapsed_time(ev1), e_iters))
    ms_e2e, e_iters = sorted(passes)[1]

    # ---- roofline: the dominant kernel, timed live with CUDA events on the library stream
    reps = 3
    ms = ctypes.c_double()
    hbm_peak, peak_src = load_peaks()
    N, S = A.N, A.S
    Np = ((N + 63) // 64) * 64 if spec.sgrid.d == 1 else spec.sgrid.n[0] * ((spec.sgrid.n[1] + 63) // 64) * 64
    # P^{-1} on the input an Arnoldi step feeds it: (A - P) v = (-eta q_s f_v)_s for the first basis vector
    v0 = P.apply(b_dev)
    v0 = v0 / torch.linalg.norm(v0)
    u = torch.zeros_like(v0)
    fv = v0[S * N:]
    qv = torch.from_numpy(A.q).to(u.device)
    u[: S * N] = (-spec.tgrid.eta * qv[:, None] * fv[None, :]).reshape(-1)
    out = torch.empty_like(u)
    if P.inner == "pcg":
        P.stats(reset=True)
    assert lib.fi_precond_apply_timed(P.handle, u.data_ptr(), out.data_ptr(), reps, ctypes.byref(ms)) == 0, last_error()
    ms_sweep = ms.value
    if P.inner == "pcg":
        st = P.stats(reset=True)
        applies = max(st["applies"], 1)
        steps_per_level = st["cg_steps"] / applies / (S + 1)
        # algorithmic HBM bytes of one apply: every level reads its right-hand side, D1 and 1/D2 rows and
        # writes its solution once, and the blocked L1 history reads each earlier level once per 8-level
        # block (sum over block starts B0 of B0 levels); the CG iterations themselves work on an
        # L2-resident set of ~10 MB per level (vectors and transform buffers), so the kernel is bound by
        # the latency of its dependent passes, not by HBM
        hist_levels = sum(b0 for b0 in range(8, S, 8))
        sweep_bytes = 8 * Np * (4 * (S + 1) + 8 + hist_levels)
        passes_per_level = 4 * steps_per_level + 3
        roof = {"bound": "hbm", "kernel": "tau_pcg_fused (K5: tau-preconditioned CG block solves, one cooperative "
                                          "kernel per P^-1; chain of S+1 dependent levels)",
                "achieved": round(sweep_bytes / (ms_sweep * 1e-3) / 1e9, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(sweep_bytes / (ms_sweep * 1e-3) / 1e9 / hbm_peak, 4),
                "traffic": load_traffic("tau_pcg_fused", cfg)[0], "traffic_source": load_traffic("tau_pcg_fused", cfg)[1],
                "bytes_per_launch": sweep_bytes, "ms_per_launch": round(ms_sweep, 4),
                "us_per_level": round(ms_sweep * 1e3 / (S + 1), 2), "cg_steps_per_level": round(steps_per_level, 2),
                "passes_per_level": round(passes_per_level, 1),
                "us_per_pass": round(ms_sweep * 1e3 / (S + 1) / passes_per_level, 2),
                "inner_nonconverged": st["nonconverged_blocks"], "input": "(A - P) v0, the first Arnoldi step's",
                # SURVEY 8(d), P-apply configs 2-4: "count the inner-solve vector traffic per level x inner
                # iterations": a textbook PCG step touches 17 length-N vectors (B p: 2, p.Bp: 2, x: 3, r: 3,
                # tau solve: 2, r.z: 2, p: 3); here they stay in shared memory / L2 (see `traffic`)
                "inner_solve_vector_bytes": int(17 * 8 * N * st["cg_steps"] / applies),
                "achieved_incl_inner_vectors": round((sweep_bytes + 17 * 8 * N * st["cg_steps"] / applies) /
                                                     (ms_sweep * 1e-3) / 1e9, 1),
                "note": "latency-bound: per CG step 4 grid-synchronised transform passes (rows, columns, rows, "
                        "columns) on an L2-resident working set; us_per_pass is the number to watch",
                "peak_source": peak_src}
    else:
        # HODLR / packed-tile sweep over the dense-block inverses (1D)
        form = P.form
        nb = Np // 64
        T = nb * (nb + 1) // 2
        sweep_bytes = (int(P.device_bytes()) + 4 * 8 * Np * (S + 1) if form == "hodlr" else
                       (S + 1) * T * 64 * 64 * 8 + 4 * 8 * Np * (S + 1))
        roof = {"bound": "hbm", "kernel": ("hodlr_sweep_kernel (K2h: substitution over HODLR inverses)" if form == "hodlr"
                                           else "sweep_kernel (K2: substitution over packed tiles)"),
                "achieved": round(sweep_bytes / (ms_sweep * 1e-3) / 1e9, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(sweep_bytes / (ms_sweep * 1e-3) / 1e9 / hbm_peak, 4),
                "traffic": load_traffic("hodlr_sweep_kernel", cfg)[0] if form == "hodlr" else None,
                "traffic_source": load_traffic("hodlr_sweep_kernel", cfg)[1] if form == "hodlr" else None,
                "bytes_per_launch": sweep_bytes, "ms_per_launch": round(ms_sweep, 4),
                "us_per_level": round(ms_sweep * 1e3 / (S + 1), 3), "precond_form": form, "peak_source": peak_src}
    del out
    y = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).to(b_dev.device)
    o2 = torch.empty_like(y)
    # K1 (the dense DMMA contraction) is timed in DMMA mode; the solve's own apply (K1f on 2D grids) beside it
    op_mode = A.apply_mode
    A.set_apply_mode("dmma")
    assert lib.fi_system_apply_timed(A.handle, y.data_ptr(), o2.data_ptr(), reps, ctypes.byref(ms)) == 0
    ms_op = ms.value
    A.set_apply_mode("auto")
    ms_fft = None
    if op_mode == "fft":
        assert lib.fi_system_apply_timed(A.handle, y.data_ptr(), o2.data_ptr(), reps, ctypes.byref(ms)) == 0
        ms_fft = ms.value
    del o2
    op_flops = 2.0 * N * N * (S + 1)
    op_tflops = op_flops / (ms_op * 1e-3) / 1e12
    fp64_peak, fp64_src = load_fp64_peak()
    # K3/K4: one Arnoldi step's MGS + Givens kernel at k = iterations / 2 (mgs_step_kernel), L2 flushed before each
    k_mgs = max(1, rep.iterations // 2)
    reorth = ctypes.c_int()
    assert lib.fi_mgs_step_timed(ctx.handle, n, k_mgs, reps, ctypes.byref(ms), ctypes.byref(reorth)) == 0, last_error()
    ms_mgs = ms.value
    # algorithmic bytes of MGS step k: 8 n (3 (k + 1) + 3), doubled when the second pass runs
    mgs_bytes = 8 * n * (3 * (k_mgs + 1) + 3) * (2 if reorth.value else 1)
    # the same at k = 25, the mean Arnoldi step of a GMRES(50) cycle (the unpreconditioned solve's regime)
    reorth25 = ctypes.c_int()
    assert lib.fi_mgs_step_timed(ctx.handle, n, 25, max(2, reps // 2), ctypes.byref(ms), ctypes.byref(reorth25)) == 0
    ms_mgs25 = ms.value
    mgs_bytes25 = 8 * n * (3 * 26 + 3) * (2 if reorth25.value else 1)
    del y
    # max over ranks for times, sum over ranks for the work done (replicas)
    ms_total_max, iters_all = replica_aggregate(ms_total, total_iters, b_dev.device)
    ms_e2e_max, e_iters_all = replica_aggregate(ms_e2e, e_iters, b_dev.device)
    value = iters_all / (ms_total_max * 1e-3)
    e2e_value = e_iters_all / (ms_e2e_max * 1e-3)

    # ---- the other configurations (rank 0, single process): time-to-solve of each
    configs = {}
    if rank == 0 and ws == 1 and not args.no_configs:
        # config 4 unpreconditioned (BASELINE: GMRES(50), max 2000 iterations): the whole solve, timed once
        # (with K1f a step is one FFT apply + the MGS step; with K1 alone it would be ~0.14 s per step)
        unprec_maxit = 2000 if cfg == 4 else RESTART
        ou = F.GmresOptions(TOL[cfg], unprec_maxit, RESTART)
        F.gmres(A, None, b_dev, F.GmresOptions(TOL[cfg], 1, RESTART))
        torch.cuda.synchronize()
        ev0.record(stream)
        _, rep_n = F.gmres(A, None, b_dev, ou)
        ev1.record(stream)
        torch.cuda.synchronize()
        t_n = ev0.elapsed_time(ev1) * 1e-3
        configs[NAMES[cfg] + "_unpreconditioned"] = {
            "time_to_solve_s": round(t_n, 3), "iterations": rep_n.iterations, "converged": rep_n.converged,
            "iters_per_s": round(rep_n.iterations / t_n, 3), "maxit": unprec_maxit,
            "final_true_residual": rep_n.final_true_residual, "last_history": rep_n.residual_history[-1],
            "note": "GMRES(50) without preconditioner (krylov.cpp:81-83), the full solve timed; parity against "
                    "tests/golden/oracle_config4_unprec.npz in tests/test_gpu_goldens.py"}
        del P, A, b_dev, x
        torch.cuda.empty_cache()
        for c in [c for c in (0, 1, 2, 3, 4) if c != cfg]:
            sp, Ac, Pc, zc, su = build_case(F, ctx, c)
            bc = torch.from_numpy(zc).to(f"cuda:{ctx.device}")
            oc = F.GmresOptions(TOL[c], 0, RESTART)
            F.gmres(Ac, Pc, bc, oc)
            msc, itc, xc, repc = time_solves(F, Ac, Pc, bc, oc, stream, 2)
            configs[NAMES[c]] = {"time_to_solve_s": round(msc * 1e-3 / 2, 5), "iterations": repc.iterations,
                                 "iters_per_s": round(itc / (msc * 1e-3), 3), "setup_s": su,
                                 "precond": Pc.inner if Pc.inner == "pcg" else Pc.form,
                                 "recon_error_vs_fstar": F.relative_error(sp.f_true, xc[-Ac.N:].cpu().numpy())}
            if not args.no_cpu_baseline:
                # the CPU restatement of the reference beside it, same box, all host threads (a bounded sample,
                # extrapolated as for the headline's cpu_baseline)
                nthr = os.cpu_count() or 1
                cs_ = cpu_reference_sample(c, repc.iterations, nthr)
                configs[NAMES[c]]["cpu_oracle"] = {
                    "iters_per_s": round(cs_["iters_per_s"], 6), "cores": nthr, "kind": "port",
                    "time_to_solve_s_extrapolated": round(cs_["time_to_solve_s_extrapolated"], 3),
                    "gpu_speedup": round((itc / (msc * 1e-3)) / cs_["iters_per_s"], 1)}
            del Ac, Pc, bc, xc
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_entry(cfg, golden_iterations(cfg, rep.iterations))

    if rank == 0:
        configs[NAMES[cfg]] = {"time_to_solve_s": round(ms_total_max / args.steps * 1e-3, 5),
                               "iterations": rep.iterations, "iters_per_s": round(value / ws, 3)}
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "iters/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_total_max / args.steps, 3),
            "time_to_solve_s": round(ms_total_max / args.steps * 1e-3, 5),
            "iterations_per_solve": rep.iterations,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (BASELINE.json config; observation by the forward solve of f* + seeded Gaussian noise)",
            "config": workload_config(cfg, ws),
            "setup_s": setup_s,
            "recon_error_vs_fstar": recon_err,
            "final_true_residual": rep.final_true_residual,
            "e2e": {"value": round(e2e_value, 3), "unit": "iters/s", "h2d_bytes_per_step": 8 * n,
                    "d2h_bytes_per_step": 8 * n, "timing": "median of 3 timed passes of K solves"},
            "gpu_launches": int(launches),
            "arnoldi_step": "split: P^-1 A v = v + P^-1((A - P) v), one preconditioner apply per step (exact identity)",
            "value_operator_then_precond": {"value": round(u_iters / (ms_unsplit * 1e-3), 3), "unit": "iters/s",
                                            "iterations_per_solve": rep_u.iterations,
                                            "note": "reference order: the operator apply, then P^-1, every Arnoldi step"},
            "roofline": roof,
            "roofline_operator": {"bound": "tensor", "kernel": "toeplitz_apply_kernel (K1, FP64 DMMA)",
                                  "achieved": round(op_tflops, 3), "peak": fp64_peak, "unit": "TFLOP/s",
                                  "frac": round(op_tflops / fp64_peak, 4), "flops_per_launch": op_flops,
                                  "ms_per_launch": round(ms_op, 4), "peak_source": fp64_src,
                                  "traffic": load_traffic("toeplitz_apply_kernel", cfg)[0],
                                  "note": "the dense contraction, timed in FI_APPLY_DMMA mode" +
                                          ("; the solve applies A by K1f (operator_fft)" if ms_fft else "")},
            "operator_fft": None if ms_fft is None else {
                "kernel": "K1f: fftop_rows_fwd + fftop_cols + fftop_rows_inv (batched 2D FFT Toeplitz products) "
                          "with K1's time convolution (conv-only DMMA) on a side stream",
                "ms_per_launch": round(ms_fft, 4), "speedup_vs_dmma": round(ms_op / ms_fft, 1)},
            "roofline_arnoldi": {"bound": "hbm", "kernel": "mgs_step_kernel (K3/K4: the MGS rounds, second pass, "
                                                          "h_(k+1), v_(k+1) and the Givens update of one Arnoldi step)",
                                 "achieved": round(mgs_bytes / (ms_mgs * 1e-3) / 1e9, 1), "peak": hbm_peak,
                                 "unit": "GB/s", "frac": round(mgs_bytes / (ms_mgs * 1e-3) / 1e9 / hbm_peak, 4),
                                 "bytes_per_launch": mgs_bytes, "ms_per_launch": round(ms_mgs, 5), "k": k_mgs,
                                 "second_pass": bool(reorth.value),
                                 "note": "algorithmic bytes 8 n (3 (k + 1) + 3) (SURVEY 8(d)); the kernel moves "
                                         "8 n (7 + 4 k) (w read and written every round); L2 flushed before each",
                                 "k25": {"ms_per_launch": round(ms_mgs25, 4),
                                         "achieved": round(mgs_bytes25 / (ms_mgs25 * 1e-3) / 1e9, 1),
                                         "frac": round(mgs_bytes25 / (ms_mgs25 * 1e-3) / 1e9 / hbm_peak, 4),
                                         "bytes_per_launch": mgs_bytes25, "second_pass": bool(reorth25.value)}},
            "configs": configs,
            "clocks": clocks,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    cfg = args.config
    iters = golden_iterations(cfg, args.iters_hint)
    threads = os.cpu_count() or 1
    samples = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference_sample(cfg, iters, threads)
        if i >= args.warmup:
            samples.append(r)
    v = float(np.mean([s["iters_per_s"] for s in samples]))
    t_iter = float(np.mean([s["time_per_iteration_s"] for s in samples]))
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 6),
        "unit": "iters/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_iter * 1e3, 1),
        "time_to_solve_s": round(float(np.mean([s["time_to_solve_s_extrapolated"] for s in samples])), 2),
        "iterations_per_solve": iters,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE.json config; observation by the forward solve of f* + seeded Gaussian noise)",
        "config": workload_config(cfg, ws),
        "note": "CPU restatement of the reference (oracle/, numpy+scipy, reference order of operations); the "
                "reference needs Eigen3/FFTW3, absent here, so it cannot be built; each step is a bounded sample "
                "(one A apply, sampled P levels, one MGS step) extrapolated to one GMRES iteration",
        "cpu_baseline": {"value": round(v, 6), "unit": "iters/s", "cores": threads, "kind": "port",
                         "sample": samples[-1]["sample"]},
        "e2e": {"value": round(v, 6), "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--iters-hint", type=int, default=12, help="GMRES iterations per solve if no golden exists")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config table")
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
