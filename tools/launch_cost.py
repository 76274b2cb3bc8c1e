"""Host-side cost of enqueueing one P apply / one A apply (no synchronisation in the timed loop)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200._lib import lib  # noqa: E402
from paper_2507_02809_b200.configs import baseline_problem  # noqa: E402

cfg = int(os.environ.get("CFG", "1"))
ctx = F.Context(0)
A = F.SystemOperator(baseline_problem(F, cfg), ctx=ctx)
P = F.BlockTriangularPreconditioner(A)
n = A.dim()
y = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
w = torch.empty_like(y)
for _ in range(3):
    lib.fi_precond_apply(P.handle, y.data_ptr(), w.data_ptr())
torch.cuda.synchronize()
for name, fn in (("P", lambda: lib.fi_precond_apply(P.handle, y.data_ptr(), w.data_ptr())),
                 ("A", lambda: lib.fi_system_apply(A.handle, y.data_ptr(), w.data_ptr()))):
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t) * 1e3)
        torch.cuda.synchronize()
    print(name, "host enqueue ms:", " ".join(f"{v:.3f}" for v in ts))
