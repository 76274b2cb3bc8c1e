#!/usr/bin/env python3
"""Run the CPU oracle once per BASELINE config and store its GMRES(50) solve as a golden file.

For each config: the observation mu_eps (forward solve of f* + seeded Gaussian noise), the
oracle's iteration count, residual history, final true residual and recovered f.  The GPU tests
feed the same mu_eps to the device path and compare against these (iterations +-1, f <= 1e-8).
1D blocks use the reference's dense LU (config 1: refactored per apply, 68.8 GB of factors do not
fit in host RAM); 2D blocks use the substituted tau-PCG solve.
Usage: python tests/golden/gen_oracle_solutions.py [--keep-observation] 2 3 4u ...
(writes tests/golden/oracle_config<i>.npz; <i>u: the unpreconditioned solve, resumable)
"""
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
warnings.filterwarnings("ignore")

from oracle import fracinv_oracle as O  # noqa: E402
from paper_2507_02809_b200.configs import NOISE, RESTART, SEED_BASE, TOL, baseline_problem  # noqa: E402


def run(cfg, precond=True):
    t0 = time.time()
    A = O.SystemOperator(baseline_problem(O, cfg))
    P = O.BlockTriangularPreconditioner(A, cache=(cfg != 1))
    prec_file = os.path.join(HERE, f"oracle_config{cfg}.npz")
    if (not precond or KEEP_OBSERVATION) and os.path.exists(prec_file):
        # the unpreconditioned solve runs on the same observation as the preconditioned golden;
        # --keep-observation: a regenerated golden keeps its observation (the unpreconditioned golden's input)
        mu_eps = np.load(prec_file)["mu_eps"]
    else:
        Pfs = P if P.inner == "pcg" else None
        mu = O.forward_solve(A, P=Pfs).mu if cfg != 1 else O.forward_solve(A, P=P).mu
        mu_eps = O.add_gaussian_noise(mu, NOISE[cfg], SEED_BASE + cfg)
    z = O.build_rhs(A, mu_eps).z
    t1 = time.time()
    calls = [0]

    def apply_A(v):
        calls[0] += 1
        if calls[0] % 50 == 0:
            print(f"  config {cfg}: {calls[0]} operator applies, {time.time() - t1:.0f}s", flush=True)
        return A.apply(v)

    x, rep = O.gmres(apply_A, P.apply if precond else None, z, tol=TOL[cfg], restart=RESTART,
                     maxit=0 if precond else 2000)
    t2 = time.time()
    f = x[-A.N:]
    name = f"oracle_config{cfg}{'' if precond else '_unprec'}.npz"
    np.savez_compressed(os.path.join(HERE, name), mu_eps=mu_eps, f=f, iterations=rep.iterations,
                        history=np.array(rep.residual_history), final_true_residual=rep.final_true_residual,
                        converged=rep.converged, recon_error=O.relative_error(A.spec.f_true, f),
                        setup_s=t1 - t0, solve_s=t2 - t1, inner=P.inner)
    print(f"config {cfg}: {rep.iterations} iterations, converged {rep.converged}, setup {t1 - t0:.1f}s, "
          f"solve {t2 - t1:.1f}s -> {name}", flush=True)


def run_unprec_resumable(cfg, maxit=2000):
    """The unpreconditioned GMRES(50) solve, one restart cycle per oracle call.

    O.gmres(x0=x, maxit=RESTART, restart=RESTART) is exactly one cycle of the oracle's GMRES(m): the same
    r = b - A x at the start, the same Arnoldi loop and x update (the first history entry of a
    continued call repeats the restart residual and is dropped).  After every cycle x and the history
    go to scratch/unprec<cfg>_ckpt.npz, so an interrupted run resumes; every 10 cycles and at the end the
    golden tests/golden/oracle_config<cfg>_unprec.npz is (re)written with `maxit` = the iterations it
    covers (the GPU test runs the device solve to the same maxit).
    """
    A = O.SystemOperator(baseline_problem(O, cfg))
    mu_eps = np.load(os.path.join(HERE, f"oracle_config{cfg}.npz"))["mu_eps"]
    z = O.build_rhs(A, mu_eps).z
    os.makedirs(os.path.join(ROOT, "scratch"), exist_ok=True)
    ckpt = os.path.join(ROOT, "scratch", f"unprec{cfg}_ckpt.npz")
    x, hist, iters, spent = None, [], 0, 0.0
    if os.path.exists(ckpt):
        c = np.load(ckpt)
        x, hist, iters, spent = c["x"], list(c["history"]), int(c["iterations"]), float(c["solve_s"])
        print(f"resuming at {iters} iterations ({spent:.0f}s so far)", flush=True)
    converged = False
    ftr = float("nan")
    while iters < maxit and not converged:
        t1 = time.time()
        x, rep = O.gmres(A.apply, None, z, tol=TOL[cfg], restart=RESTART, maxit=min(RESTART, maxit - iters), x0=x)
        hist += rep.residual_history if not hist else rep.residual_history[1:]
        iters += rep.iterations
        converged, ftr = rep.converged, rep.final_true_residual
        spent += time.time() - t1
        np.savez(ckpt, x=x, history=np.array(hist), iterations=iters, solve_s=spent)
        print(f"  config {cfg} unpreconditioned: {iters} iterations, history {hist[-1]:.6e}, true residual "
              f"{ftr:.6e}, {spent:.0f}s", flush=True)
        if converged or iters >= maxit or (iters // RESTART) % 10 == 0:
            np.savez_compressed(os.path.join(HERE, f"oracle_config{cfg}_unprec.npz"), mu_eps=mu_eps, f=x[-A.N:],
                                iterations=iters, maxit=iters, history=np.array(hist), final_true_residual=ftr,
                                converged=converged, recon_error=O.relative_error(A.spec.f_true, x[-A.N:]),
                                setup_s=0.0, solve_s=spent, inner="none")


KEEP_OBSERVATION = "--keep-observation" in sys.argv

if __name__ == "__main__":
    for arg in [a for a in sys.argv[1:] if not a.startswith("--")]:
        if arg.endswith("u"):
            run_unprec_resumable(int(arg[:-1]))
        else:
            run(int(arg))
