"""Compare the HODLR preconditioner sweep with the packed-tile sweep (refinement off and on) on a
BASELINE config: relative difference of P^{-1} z and backward error against the oracle's P.
usage: CFG=0 python tools/hodlr_check.py   (runs itself twice, FI_HODLR=1 and 0)"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cfg = int(os.environ.get("CFG", "0"))
if os.environ.get("HODLR_CHILD"):
    from paper_2507_02809_b200 import fracinv as F
    from paper_2507_02809_b200.configs import baseline_problem
    A = F.SystemOperator(baseline_problem(F, cfg))
    P = F.BlockTriangularPreconditioner(A)
    z = np.random.default_rng(3).uniform(-1, 1, A.dim())
    P.set_refine(False)
    y0 = P.apply(z)
    P.set_refine(True)
    y1 = P.apply(z)
    np.savez(os.environ["HODLR_CHILD"], y0=y0, y1=y1, z=z)
    sys.exit(0)
out = {}
for flag in ("1", "0"):
    fn = f"/tmp/hodlr_{cfg}_{flag}.npz"
    env = dict(os.environ, FI_HODLR=flag, HODLR_CHILD=fn)
    subprocess.run([sys.executable, __file__], env=env, check=True)
    out[flag] = np.load(fn)
from oracle import fracinv_oracle as O  # noqa: E402
from paper_2507_02809_b200.configs import baseline_problem  # noqa: E402
Ao = O.SystemOperator(baseline_problem(O, cfg))
z = out["1"]["z"]
N = Ao.N
for k in ("y0", "y1"):
    a, b = out["1"][k], out["0"][k]
    rel = np.linalg.norm(a - b) / np.linalg.norm(b)
    lev = [float(np.linalg.norm(a[s * N:(s + 1) * N] - b[s * N:(s + 1) * N]) / np.linalg.norm(b[s * N:(s + 1) * N]))
           for s in (0, 1, 2, Ao.steps - 1, Ao.steps)]
    bwd_h = np.linalg.norm(Ao.apply_precond_matrix(a) - z) / np.linalg.norm(z)
    bwd_d = np.linalg.norm(Ao.apply_precond_matrix(b) - z) / np.linalg.norm(z)
    print(f"cfg {cfg} {k}: hodlr vs tiles {rel:.3e}, per level {['%.1e' % v for v in lev]}, "
          f"backward error hodlr {bwd_h:.3e} tiles {bwd_d:.3e}", flush=True)
