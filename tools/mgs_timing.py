"""Time one MGS round (fi_mgs_round_timed, L2 flushed) on config-1-length vectors (tuning aid)."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200._lib import lib  # noqa: E402

n = 513 * 4096
ctx = F.Context(0)
w, x, y = (torch.from_numpy(np.random.default_rng(k).uniform(-1, 1, n)).cuda() for k in (5, 6, 7))
ms = ctypes.c_double()
assert lib.fi_mgs_round_timed(ctx.handle, n, w.data_ptr(), x.data_ptr(), y.data_ptr(), 20, ctypes.byref(ms)) == 0
print(json.dumps({"mgs_round_us": ms.value * 1e3, "GBps": 32.0 * n / (ms.value * 1e-3) / 1e9}))
