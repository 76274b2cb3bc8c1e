#!/usr/bin/env python3
"""Per-level CG step counts of the oracle's tau-PCG preconditioner apply (configs 2-4) on the input the
first Arnoldi step feeds P: u = A v0, v0 = [0; G_f^{-1} mu_eps] / norm (mu_eps of the golden solve).

bench.py's CPU baseline (both arms) times the oracle's per-level fixed cost and its cost per CG step on
the first levels and multiplies them with these counts for all S + 1 levels, so that the bounded CPU
sample extrapolates with the oracle's own operation counts instead of the (slower) first levels'.
Usage: python tests/golden/gen_pcg_steps.py 2 3 4   (writes tests/golden/oracle_pcg_steps.json)
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import fracinv_oracle as O  # noqa: E402
from paper_2507_02809_b200.configs import baseline_problem  # noqa: E402


def bench_input(A, P, cfg):
    N, S = A.N, A.steps
    mu_eps = np.load(os.path.join(HERE, f"oracle_config{cfg}.npz"))["mu_eps"]
    fv = P.solve_block(S + 1, mu_eps)
    u = np.zeros(A.dim)
    u[S * N:] = fv / np.linalg.norm(fv)
    return A.apply(u)


def main():
    path = os.path.join(HERE, "oracle_pcg_steps.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for cfg in [int(a) for a in sys.argv[1:]]:
        t0 = time.time()
        A = O.SystemOperator(baseline_problem(O, cfg))
        P = O.BlockTriangularPreconditioner(A, inner="pcg")
        z = bench_input(A, P, cfg)
        P.pcg.iterations = []
        y = P.apply(z)
        its = [int(v) for v in P.pcg.iterations]
        out[str(cfg)] = {"steps_per_level": its, "total": int(sum(its)), "levels": len(its),
                         "y_norm": float(np.linalg.norm(y)), "seconds": round(time.time() - t0, 1)}
        print(f"config {cfg}: {sum(its)} CG steps over {len(its)} levels ({sum(its) / len(its):.2f}/level), "
              f"{time.time() - t0:.0f}s", flush=True)
        json.dump(out, open(path, "w"), indent=0)


if __name__ == "__main__":
    main()
