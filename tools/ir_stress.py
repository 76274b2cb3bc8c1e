"""Repeat one preconditioner apply many times on the same input and count runs whose bits differ
from the first (race detector for the persistent sweep kernels).
usage: FI_HODLR=0 CFG=1 REPS=40 python tools/ir_stress.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200._lib import lib  # noqa: E402
from paper_2507_02809_b200.configs import baseline_problem  # noqa: E402

cfg = int(os.environ.get("CFG", "1"))
reps = int(os.environ.get("REPS", "40"))
A = F.SystemOperator(baseline_problem(F, cfg))
P = F.BlockTriangularPreconditioner(A)
P.set_refine(os.environ.get("REFINE", "1") == "1")
n = A.dim()
z = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, n)).cuda()
ref = torch.empty_like(z)
out = torch.empty_like(z)
ms = ctypes.c_double()
assert lib.fi_precond_apply_timed(P.handle, z.data_ptr(), ref.data_ptr(), 1, ctypes.byref(ms)) == 0
bad, worst = 0, 0.0
for r in range(reps):
    assert lib.fi_precond_apply_timed(P.handle, z.data_ptr(), out.data_ptr(), 1, ctypes.byref(ms)) == 0
    if not torch.equal(out, ref):
        bad += 1
        d = float((out - ref).norm() / ref.norm())
        worst = max(worst, d)
        lv = ((out - ref).abs().view(A.S + 1, A.N).amax(1) > 0).nonzero()
        print(f"rep {r}: rel diff {d:.3e}, first differing level {int(lv[0])} of {A.S + 1}", flush=True)
print(f"form {P.form}: {bad}/{reps} runs differ, worst {worst:.3e}", flush=True)
