"""P^{-1} applied to the split Arnoldi step's input u = (-eta q_s f)_s (smooth in time), the input a
solve actually feeds the preconditioner, against a random vector (diagnostic; FI_ITER_TRACE=1 prints
the tau-PCG phase split).  usage: CFG=3 python tools/smooth_papply.py"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200.configs import baseline_problem  # noqa: E402

cfg = int(os.environ.get("CFG", "3"))
A = F.SystemOperator(baseline_problem(F, cfg))
P = F.BlockTriangularPreconditioner(A)
N, S = A.N, A.S
f = np.random.default_rng(2).uniform(-1, 1, N)
u = np.zeros(A.dim())
for s in range(S):
    u[s * N:(s + 1) * N] = -A.spec.tgrid.eta * A.q[s] * f
r = np.random.default_rng(3).uniform(-1, 1, A.dim())
out = {"cfg": cfg}
for name, v in (("smooth", u), ("random", r)):
    P.apply(v)
    t = time.perf_counter()
    P.apply(v)
    out[name + "_ms"] = round((time.perf_counter() - t) * 1e3, 2)
print(json.dumps(out))
