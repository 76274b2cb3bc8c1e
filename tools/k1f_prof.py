import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes, numpy as np, torch
from paper_2507_02809_b200 import fracinv as F
from paper_2507_02809_b200._lib import lib
from paper_2507_02809_b200.configs import baseline_problem
A = F.SystemOperator(baseline_problem(F, 4))
y = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, A.dim())).cuda(); o = torch.empty_like(y)
ms = ctypes.c_double()
assert lib.fi_system_apply_timed(A.handle, y.data_ptr(), o.data_ptr(), 3, ctypes.byref(ms)) == 0
print("fft apply ms", ms.value)
