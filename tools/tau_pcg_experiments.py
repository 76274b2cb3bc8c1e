"""Oracle-only experiments behind the K5 / TauPCG choices of DESIGN 4 (CPU; no GPU, no product code):
CG steps of one preconditioner apply on the first Arnoldi step's input (tests/golden/gen_pcg_steps.py's input)
under variants of the oracle's per-block solve.

  python tools/tau_pcg_experiments.py shift [cfg=4]   the tau preconditioner's shift: arithmetic / geometric /
                                                      harmonic mean of delta, median, multiples of the mean
  python tools/tau_pcg_experiments.py guess [cfg=4]   initial guesses: one fixed kind on every level against the
                                                      choice by measurement; the previous stopping rule
"""
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from oracle import fracinv_oracle as O  # noqa: E402
from paper_2507_02809_b200.configs import baseline_problem  # noqa: E402
import gen_pcg_steps as G  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "shift"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
A = O.SystemOperator(baseline_problem(O, cfg))
P = O.BlockTriangularPreconditioner(A, inner="pcg")
z = G.bench_input(A, P, cfg)


def run(name):
    P.pcg.iterations = []
    t = time.time()
    y = P.apply(z)
    its = P.pcg.iterations
    bwd = np.linalg.norm(A.apply_precond_matrix(y) - z) / np.linalg.norm(z)
    print(f"config {cfg} {name}: {sum(its)} CG steps; per 64 levels "
          f"{[round(sum(its[i:i + 64]) / 64, 1) for i in range(0, len(its), 64)]}; backward error {bwd:.2e}; "
          f"{time.time() - t:.0f}s", flush=True)


if mode == "shift":
    hmean = O._hmean
    variants = [("harmonic mean (the oracle's)", hmean), ("arithmetic mean", lambda d: float(d.mean())),
                ("geometric mean", lambda d: float(np.exp(np.log(d).mean())) if np.all(d > 0) else 0.0),
                ("median", lambda d: float(np.median(d))), ("0.3 x mean", lambda d: 0.3 * float(d.mean())),
                ("0.1 x mean", lambda d: 0.1 * float(d.mean())), ("min", lambda d: float(d.min()))]
    for name, fn in variants:
        O._hmean = fn
        run("shift = " + name)
    O._hmean = hmean
else:
    run("guesses chosen by measurement, floor rule (the oracle's)")
    ww = O.TauPCG.warm_weights
    for kind, label in ((0, "6-point polynomial"), (1, "8-point polynomial"), (2, "10-point polynomial"),
                        (3, "least squares (degree 5, 10 points)")):
        def fixed(self, nprev, level=0, kind=kind):
            self.kind = kind if nprev >= O.LS_WINDOW else 0
            if self.kind == 3:
                return O.LS_COEF
            k = min(nprev, (O.WARM_ORDER, 8, 10)[self.kind])
            return [float((-1) ** (j + 1) * math.comb(k, j)) for j in range(1, k + 1)]
        O.TauPCG.warm_weights = fixed
        run("every level: " + label)
    O.TauPCG.warm_weights = ww
    P.pcg.theta, P.pcg.lswin = 0.0, 0
    run("previous rule: tol ||b|| alone, 6-point polynomial")
