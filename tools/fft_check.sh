set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fft_smoke.log 2>&1
timeout 900 python -m pytest -x -q -s -m gpu tests/test_gpu_fft_apply.py > gpurun_out/fft_tests.log 2>&1
for c in 2 3 4; do CFG=$c timeout 300 python - >> gpurun_out/fft_timing.log 2>&1 <<'PY'
import ctypes, os, json, numpy as np, torch
from paper_2507_02809_b200 import fracinv as F
from paper_2507_02809_b200._lib import lib
from paper_2507_02809_b200.configs import baseline_problem
cfg = int(os.environ["CFG"])
A = F.SystemOperator(baseline_problem(F, cfg))
y = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, A.dim())).cuda(); o = torch.empty_like(y)
ms = ctypes.c_double(); out = {"cfg": cfg}
for m in ("fft", "dmma"):
    A.set_apply_mode(m)
    assert lib.fi_system_apply_timed(A.handle, y.data_ptr(), o.data_ptr(), 5, ctypes.byref(ms)) == 0
    out[m + "_ms"] = round(ms.value, 4)
print(json.dumps(out))
PY
done
