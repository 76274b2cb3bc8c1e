"""Where a config-1 GMRES solve spends its time: the solve (device path) against the same number of
bare P and A applies back to back (diagnostic).  usage: python tools/solve_breakdown.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200._lib import lib  # noqa: E402
from paper_2507_02809_b200.configs import NOISE, RESTART, SEED_BASE, TOL, baseline_problem  # noqa: E402

ctx = F.Context(0)
A = F.SystemOperator(baseline_problem(F, 1), ctx=ctx)
P = F.BlockTriangularPreconditioner(A)
mu = F.forward_solve(A, P).mu
z = F.build_rhs(A, F.add_gaussian_noise(mu, NOISE[1], SEED_BASE + 1)).z
b = torch.from_numpy(z).cuda()
opts = F.GmresOptions(TOL[1], 0, RESTART)
stream = torch.cuda.ExternalStream(ctx.stream)
for _ in range(3):
    _, rep = F.gmres(A, P, b, opts)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(5):
    _, rep = F.gmres(A, P, b, opts)
e1.record(stream)
torch.cuda.synchronize()
t_solve = e0.elapsed_time(e1) / 5
n = A.dim()
# padded-layout device vectors for the bare applies (fi_precond_apply / fi_system_apply take padded? use host-facing)
y = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
w = torch.empty_like(y)
k = rep.iterations + 1
torch.cuda.synchronize()
e0.record(stream)
for _ in range(5):
    for _ in range(k):
        assert lib.fi_system_apply(A.handle, y.data_ptr(), w.data_ptr()) == 0
        assert lib.fi_precond_apply(P.handle, w.data_ptr(), y.data_ptr()) == 0
e1.record(stream)
torch.cuda.synchronize()
t_bare = e0.elapsed_time(e1) / 5
print(f"iterations {rep.iterations}: solve {t_solve:.3f} ms, {k} x (A + P) bare {t_bare:.3f} ms, "
      f"overhead {t_solve - t_bare:.3f} ms ({100 * (t_solve - t_bare) / t_solve:.1f}%)")
