"""Local forward error per time level of the device P^{-1} (refinement off / on) against the
reference's per-block LU solve (oracle), using the device's own history of earlier levels:
err_s = |y_s - G_s^{-1}(z_s - D1_s o sum_m e_{s-m} y_m)| / |G_s^{-1}(...)|.
usage: CFG=1 python tools/level_errors.py"""
import os
import sys

import numpy as np
import scipy.linalg as sla

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import fracinv_oracle as O  # noqa: E402
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200.configs import baseline_problem  # noqa: E402

cfg = int(os.environ.get("CFG", "1"))


def problem(M):
    # CFG, or the reference's 1D problem with BETA, OMEGA, N, S from the environment
    if "OMEGA" in os.environ:
        return M.make_problem("paper1d", float(os.environ["BETA"]), float(os.environ["OMEGA"]),
                              [int(os.environ.get("N", "1023"))], int(os.environ.get("S", "48")), 5e-3, 0.01)
    return baseline_problem(M, cfg)


A = F.SystemOperator(problem(F))
P = F.BlockTriangularPreconditioner(A)
z = np.random.default_rng(3).uniform(-1, 1, A.dim())
P.set_refine(False)
y0 = P.apply(z)
P.set_refine(True)
y1 = P.apply(z)
Ao = O.SystemOperator(problem(O))
Po = O.BlockTriangularPreconditioner(Ao, cache=False)
N, S = Ao.space_dim, Ao.steps
e = Ao.weights.e
levels = sorted({1, 2, 3, S // 4, S // 2, S - 1, S, S + 1})
print(f"config {cfg} form {P.form}: N={N} S={S}", flush=True)
for s in levels:
    out = []
    for name, y in (("y0", y0), ("y1", y1)):
        Y = y[: S * N].reshape(S, N)
        if s <= S:
            rhs = z[(s - 1) * N: s * N].copy()
            if s > 1:
                rhs -= Ao.diags.D1[s - 1] * (e[s - 1:0:-1] @ Y[: s - 1])
        else:
            rhs = z[S * N:] - Y[S - 1]
        ref = sla.lu_solve(sla.lu_factor(Po.block(s), check_finite=False), rhs, check_finite=False)
        got = y[(s - 1) * N: s * N]
        out.append(f"{name} {np.linalg.norm(got - ref) / np.linalg.norm(ref):.2e}")
    print(f"level {s:4d}: " + ", ".join(out), flush=True)
