"""Diagnostic: device tau-PCG P^{-1} on the first Arnoldi step's input vs the oracle, per level: forward
error and true residual (backward error) of every block.  usage: CFG=3 python tools/tau_parity_diag.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import fracinv_oracle as O  # noqa: E402
from paper_2507_02809_b200 import fracinv as F  # noqa: E402
from paper_2507_02809_b200.configs import baseline_problem  # noqa: E402

cfg = int(os.environ.get("CFG", "3"))
A = F.SystemOperator(baseline_problem(F, cfg))
if os.environ.get("SAME_SYMBOL", "1") == "1":  # the oracle on the product's generating vector
    Ao = O.SystemOperator(baseline_problem(O, cfg),
                          symbol=O.SymbolCoefficients(A.symbol.omega, A.symbol.n, np.asarray(A.symbol.coeffs)))
else:
    Ao = O.SystemOperator(baseline_problem(O, cfg))
P, Po = F.BlockTriangularPreconditioner(A), O.BlockTriangularPreconditioner(Ao)
N, S = Ao.N, Ao.steps
mu = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                          f"oracle_config{cfg}.npz"))["mu_eps"]
fv = Po.solve_block(S + 1, mu)
u = np.zeros(Ao.dim)
u[S * N:] = fv / np.linalg.norm(fv)
z = Ao.apply(u) if os.environ.get("INPUT", "arnoldi") == "arnoldi" else np.random.default_rng(5).uniform(-1, 1, Ao.dim)
y = P.apply(z)
r = Ao.apply_precond_matrix(y) - z
print(f"config {cfg}: device backward error {np.linalg.norm(r) / np.linalg.norm(z):.3e} "
      f"(time rows {np.linalg.norm(r[:S * N]) / np.linalg.norm(z):.3e}, f rows {np.linalg.norm(r[S * N:]) / np.linalg.norm(z):.3e})")
lv = [np.linalg.norm(r[s * N:(s + 1) * N]) / max(np.linalg.norm(z[s * N:(s + 1) * N]), 1e-300) for s in range(S + 1)]
worst = np.argsort(lv)[-5:]
print("worst levels (rel residual of the block row):", [(int(i), f"{lv[i]:.2e}") for i in worst])
print("levels 0..7:", [f"{v:.1e}" for v in lv[:8]], " f-block:", f"{lv[-1]:.2e}")
if os.environ.get("ORACLE", "1") == "1":
    yo = Po.apply(z)
    fe = [np.linalg.norm(y[s * N:(s + 1) * N] - yo[s * N:(s + 1) * N]) / max(np.linalg.norm(yo[s * N:(s + 1) * N]), 1e-300)
          for s in range(S + 1)]
    print(f"forward parity whole {np.linalg.norm(y - yo) / np.linalg.norm(yo):.3e}; worst levels",
          [(int(i), f"{fe[i]:.2e}") for i in np.argsort(fe)[-5:]], "first", [f"{v:.1e}" for v in fe[:6]])
