"""Small invocations of every kernel family for compute-sanitizer (memcheck / initcheck / racecheck /
synccheck): K1, the HODLR sweep (K2h), the packed-tile sweeps (K2, merged K2 with refinement), the tau-PCG
solve (K5), the forward solve, and GMRES through the CUDA-graph driver and the host-driven loop.
usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02809_b200 import fracinv as F  # noqa: E402


def problem(n, S, d=1):
    grid = F.SpaceGrid([n] * d, [0.0] * d, [1.0] * d)
    X = grid.nodes()
    return F.make_custom_problem(F.FractionalOrders(0.5, 1.5), grid, S, 1.0,
                                 lambda X, t: 1 + 0.5 * np.sin(np.pi * X[:, 0]) * np.exp(-t),
                                 lambda X, t: 1 + X[:, 0] * (1 - X[:, 0]) * (1 + t), lambda t: 1 + t,
                                 np.zeros(X.shape[0]), np.sin(np.pi * X[:, 0]), 1e-3, 0.01)


rng = np.random.default_rng(0)
# 1D: K1, HODLR sweep (default), forward solve, GMRES (graph driver and host loop)
A = F.SystemOperator(problem(127, 16))
P = F.BlockTriangularPreconditioner(A)
y = rng.uniform(-1, 1, A.dim())
A.apply(y)
P.apply(y)
mu = F.forward_solve(A, P).mu
z = F.build_rhs(A, mu).z
F.gmres(A, P, z, F.GmresOptions(1e-10, 0, 50))
F.gmres(A, P, z, F.GmresOptions(1e-10, 0, 0))  # full GMRES: host-driven loop, growing basis
P.set_refine(True)
P.apply(y)
# 1D packed tiles (FI_HODLR=0 is read once per process: use inner="lu" on a size HODLR refuses)
A2 = F.SystemOperator(problem(31, 8))
P2 = F.BlockTriangularPreconditioner(A2)
P2.apply(rng.uniform(-1, 1, A2.dim()))
P2.set_refine(True)
P2.apply(rng.uniform(-1, 1, A2.dim()))
# 2D tau-PCG (K5), smooth and random inputs, and a solve
A3 = F.SystemOperator(problem(15, 8, d=2))
P3 = F.BlockTriangularPreconditioner(A3, inner="pcg")
P3.apply(rng.uniform(-1, 1, A3.dim()))
z3 = F.build_rhs(A3, F.forward_solve(A3, P3).mu).z
F.gmres(A3, P3, z3, F.GmresOptions(1e-10, 0, 50))
print("sanitize run done", A.ctx.kernel_launches)
