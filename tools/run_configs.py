#!/usr/bin/env python3
"""Solve every BASELINE config on the GPU and print one JSON line per config: setup times,
GMRES(50) iterations, time-to-solve, per-apply times of K1 (operator) and P, recovered-f error,
and — when tests/golden/oracle_config<i>.npz exists — parity against the oracle's solve on the
identical observation.   usage: python tools/run_configs.py [cfg ...] [--unprec4]"""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200._lib import lib  # noqa: E402
from paper_2507_02809_b200.configs import NAMES, NOISE, RESTART, SEED_BASE, TOL, baseline_problem  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    cfgs = [int(a) for a in args] or [0, 1, 2, 3, 4]
    for cfg in cfgs:
        out = {"config": NAMES[cfg]}
        t0 = time.perf_counter()
        A = F.SystemOperator(baseline_problem(F, cfg))
        out["assembly_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        P = F.BlockTriangularPreconditioner(A)
        F.default_context().synchronize()
        out["precond_build_s"] = time.perf_counter() - t0
        out["precond_inner"] = P.inner
        gpath = os.path.join(ROOT, "tests", "golden", f"oracle_config{cfg}.npz")
        g = np.load(gpath) if os.path.exists(gpath) else None
        t0 = time.perf_counter()
        if g is not None:
            mu_eps = g["mu_eps"]
        else:
            mu_eps = F.add_gaussian_noise(F.forward_solve(A, P).mu, NOISE[cfg], SEED_BASE + cfg)
        out["forward_solve_s"] = time.perf_counter() - t0
        z = F.build_rhs(A, mu_eps).z
        zt = torch.from_numpy(z).cuda()
        opts = F.GmresOptions(TOL[cfg], 0, RESTART)
        x, rep = F.gmres(A, P, zt, opts)  # warm-up (graph instantiation, workspaces)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = F.gmres(A, P, zt, opts)
        torch.cuda.synchronize()
        out["time_to_solve_s"] = time.perf_counter() - t0
        out["iterations"] = rep.iterations
        out["converged"] = rep.converged
        out["final_true_residual"] = rep.final_true_residual
        f = x[-A.N:].cpu().numpy()
        out["recon_error_vs_fstar"] = F.relative_error(A.spec.f_true, f)
        if g is not None:
            out["oracle_iterations"] = int(g["iterations"])
            out["f_parity_vs_oracle"] = float(np.linalg.norm(f - g["f"]) / np.linalg.norm(g["f"]))
        y = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, A.dim())).cuda()
        o = torch.empty_like(y)
        ms = ctypes.c_double()
        assert lib.fi_system_apply_timed(A.handle, y.data_ptr(), o.data_ptr(), 3, ctypes.byref(ms)) == 0
        out["operator_apply_ms"] = ms.value
        out["operator_tflops"] = 2.0 * A.N ** 2 * (A.S + 1) / (ms.value * 1e-3) / 1e12
        assert lib.fi_precond_apply_timed(P.handle, y.data_ptr(), o.data_ptr(), 2, ctypes.byref(ms)) == 0
        out["precond_apply_ms"] = ms.value
        print(json.dumps(out), flush=True)
        if cfg == 4 and "--unprec4" in sys.argv:
            opts = F.GmresOptions(1e-8, 2000, RESTART)
            t0 = time.perf_counter()
            x, rep = F.gmres(A, None, zt, opts)
            torch.cuda.synchronize()
            print(json.dumps({"config": NAMES[4] + "_unpreconditioned", "iterations": rep.iterations,
                              "converged": rep.converged, "time_to_solve_s": time.perf_counter() - t0,
                              "final_true_residual": rep.final_true_residual}), flush=True)
        del P, A
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
