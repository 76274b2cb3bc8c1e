"""Time the K2 sweep / P-apply / K1 on BASELINE config 1 for a few environment settings
(used to tune the preconditioner kernel; prints one JSON line per setting)."""
import ctypes
import json
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
A = F.SystemOperator(baseline_problem(F, cfg))
P = F.BlockTriangularPreconditioner(A)
n = A.dim()
y = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
out = torch.empty_like(y)
ms = ctypes.c_double()
res = {"cfg": cfg, "pf": os.environ.get("FI_PF_TILES", "default")}
P.set_refine(False)
assert lib.fi_precond_apply_timed(P.handle, y.data_ptr(), out.data_ptr(), 5, ctypes.byref(ms)) == 0
res["sweep_ms"] = ms.value
P.set_refine(True)
rc = lib.fi_precond_apply_timed(P.handle, y.data_ptr(), out.data_ptr(), 5, ctypes.byref(ms))
assert rc == 0, lib.fi_last_error()
res["papply_ms"] = ms.value
assert lib.fi_system_apply_timed(A.handle, y.data_ptr(), out.data_ptr(), 5, ctypes.byref(ms)) == 0
res["op_ms"] = ms.value
print(json.dumps(res), flush=True)
if os.environ.get("BWD"):
    # backward error of P^{-1} y against the oracle's P (and a dump for cross-setting comparisons)
    from oracle import fracinv_oracle as O  # noqa: E402
    Ao = O.SystemOperator(baseline_problem(O, cfg))
    yh = y.cpu().numpy()
    x = P.apply(yh)
    r = Ao.apply_precond_matrix(x) - yh
    N = A.N
    res2 = {"cfg": cfg, "ir": os.environ.get("FI_SWEEP_IR", "1"),
            "bwd": float(np.linalg.norm(r) / np.linalg.norm(yh)),
            "bwd_f": float(np.linalg.norm(r[-N:]) / np.linalg.norm(yh[-N:]))}
    os.makedirs("gpurun_out", exist_ok=True)
    np.save(f"gpurun_out/papply_cfg{cfg}_ir{res2['ir']}.npy", x)
    print(json.dumps(res2), flush=True)
