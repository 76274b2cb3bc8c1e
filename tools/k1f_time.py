"""Time the operator apply (K1f on 2D configs) with fi_system_apply_timed.  usage: CFG=4 python tools/k1f_time.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200._lib import lib  # noqa: E402
from paper_2507_02809_b200.configs import baseline_problem  # noqa: E402

A = F.SystemOperator(baseline_problem(F, int(os.environ.get("CFG", "4"))))
y = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, A.dim())).cuda()
o = torch.empty_like(y)
ms = ctypes.c_double()
assert lib.fi_system_apply_timed(A.handle, y.data_ptr(), o.data_ptr(), 10, ctypes.byref(ms)) == 0
print({"cfg": os.environ.get("CFG", "4"), "mode": A.apply_mode, "ms": round(ms.value, 4)})
