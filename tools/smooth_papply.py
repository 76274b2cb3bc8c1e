"""P^{-1} applied to the split Arnoldi step's input u = (-eta q_s f)_s (smooth in time), the input a
solve actually feeds the preconditioner, against a random vector: device time per apply (CUDA events,
fi_precond_apply_timed) and the inner CG steps (FI_ITER_TRACE=1 also prints the tau-PCG phase split).
usage: CFG=3 python tools/smooth_papply.py"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200._lib import lib  # noqa: E402
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
ms = ctypes.c_double()
for name, v in (("smooth", u), ("random", r)):
    vt = torch.from_numpy(v).cuda()
    o = torch.empty_like(vt)
    if P.inner == "pcg":
        P.stats(reset=True)
    assert lib.fi_precond_apply_timed(P.handle, vt.data_ptr(), o.data_ptr(), 3, ctypes.byref(ms)) == 0
    out[name + "_ms"] = round(ms.value, 3)
    if P.inner == "pcg":
        st = P.stats(reset=True)
        out[name + "_cg_steps_per_level"] = round(st["cg_steps"] / max(st["applies"], 1) / (S + 1), 2)
print(json.dumps(out))
