"""Uninitialised device memory (the sanitizer is closed on this GPU pool): with FI_POISON=1 every device
allocation starts as 0xff bytes (NaN doubles, ~0 counters).  A 2D preconditioned GMRES(50) solve (tau-PCG
block solves, K1f, the GMRES engine's scratch) must give the same iterations and solution as without
poisoning.  Regression test for round 2's finding: the tau-PCG kernel left the pad columns of its output
unwritten, so an output buffer's previous contents leaked into the Krylov vectors (tools/poison_run.sh runs
the whole GPU suite this way)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, %r)
from paper_2507_02809_b200 import fracinv as F
g = F.SpaceGrid([31, 31], [0.0, 0.0], [1.0, 1.0])
X = g.nodes()
spec = F.make_custom_problem(F.FractionalOrders(0.3, 1.2), g, 24, 1.0,
    lambda X, t: 1 + 0.5 * np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1]),
    lambda X, t: 1 + X[:, 0] * X[:, 1] * (1 + t), lambda t: 1 + t * t, np.zeros(X.shape[0]),
    np.sin(np.pi * X[:, 0]) * np.sin(2 * np.pi * X[:, 1]), 1e-3, 0.01)
A = F.SystemOperator(spec)
P = F.BlockTriangularPreconditioner(A, inner="pcg")
mu = F.add_gaussian_noise(F.forward_solve(A, P).mu, 0.01, 7)
z = F.build_rhs(A, mu).z
x, r = F.gmres(A, P, z, F.GmresOptions(1e-10, 500, 50))
print(json.dumps({"it": r.iterations, "conv": r.converged, "f": x[-A.N:].tolist(), "finite": bool(np.isfinite(x).all())}))
""" % ROOT


def _run(poison):
    env = dict(os.environ)
    env.pop("FI_POISON", None)
    if poison:
        env["FI_POISON"] = "1"
    out = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, timeout=240, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_poisoned_allocations_change_nothing():
    import numpy as np
    clean, poisoned = _run(False), _run(True)
    assert clean["finite"] and poisoned["finite"] and clean["conv"] and poisoned["conv"]
    assert poisoned["it"] == clean["it"]
    f0, f1 = np.array(clean["f"]), np.array(poisoned["f"])
    assert np.linalg.norm(f1 - f0) <= 1e-12 * np.linalg.norm(f0)
