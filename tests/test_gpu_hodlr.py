"""GPU tests of the HODLR form of the dense-block inverses (precond_hodlr.cu): which shapes use it,
and parity of P^{-1} against the packed-tile form (FI_HODLR=0, a separate process) and the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import fracinv_oracle as O
from paper_2507_02809_b200.configs import baseline_problem

pytestmark = pytest.mark.gpu
F = pytest.importorskip("paper_2507_02809_b200.fracinv")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
from paper_2507_02809_b200 import fracinv as F
from paper_2507_02809_b200.configs import baseline_problem
A = F.SystemOperator(baseline_problem(F, int(os.environ["CFG"])))
P = F.BlockTriangularPreconditioner(A)
z = np.random.default_rng(3).uniform(-1, 1, A.dim())
P.set_refine(False)
y0 = P.apply(z)
P.set_refine(True)
y1 = P.apply(z)
np.savez(os.environ["OUT"], y0=y0, y1=y1, z=z, form=P.form)
"""


def _run(cfg, hodlr, tmp_path):
    out = str(tmp_path / f"p{cfg}_{hodlr}.npz")
    env = dict(os.environ, FI_HODLR=str(hodlr), CFG=str(cfg), OUT=out, ROOT=ROOT)
    subprocess.run([sys.executable, "-c", _CHILD], env=env, check=True, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("cfg", [0, 1])
def test_hodlr_matches_tiles_and_oracle(cfg, tmp_path):
    h, t = _run(cfg, 1, tmp_path), _run(cfg, 0, tmp_path)
    assert str(h["form"]) == "hodlr" and str(t["form"]) == "tiles"
    rel = float(np.linalg.norm(h["y1"] - t["y1"]) / np.linalg.norm(t["y1"]))
    Ao = O.SystemOperator(baseline_problem(O, cfg))
    z = h["z"]
    bwd = float(np.linalg.norm(Ao.apply_precond_matrix(h["y1"]) - z) / np.linalg.norm(z))
    print(f"config{cfg}: HODLR vs tiles {rel:.3e}, backward error {bwd:.3e}")
    assert rel <= 1e-11 and bwd <= 1e-12


_CHILD_PAPER = r"""
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
from paper_2507_02809_b200 import fracinv as F
beta, omega = float(os.environ["BETA"]), float(os.environ["OMEGA"])
A = F.SystemOperator(F.make_problem("paper1d", beta, omega, [1023], 48, 5e-3, 0.01))
P = F.BlockTriangularPreconditioner(A)
z = np.random.default_rng(4).uniform(-1, 1, A.dim())
y = P.apply(z)
P.set_refine(True)
np.savez(os.environ["OUT"], y=y, y1=P.apply(z), z=z, form=P.form)
"""


@pytest.mark.parametrize("beta,omega", [(0.1, 1.9), (0.5, 1.5), (0.9, 1.1)])
def test_hodlr_paper_orders(beta, omega, tmp_path):
    """The reference's three (beta, omega) pairs at n = 1023 (16 leaves): the rank-32 probe passes;
    the default P^{-1} (polished inverses, one sweep) matches the oracle's LU solves to 1e-12 and the
    packed tiles; with the refinement sweep the residual is LU-grade (backward error 1e-12)."""
    res = {}
    for flag in (1, 0):
        out = str(tmp_path / f"o{flag}.npz")
        env = dict(os.environ, FI_HODLR=str(flag), BETA=str(beta), OMEGA=str(omega), OUT=out, ROOT=ROOT)
        subprocess.run([sys.executable, "-c", _CHILD_PAPER], env=env, check=True, timeout=600)
        res[flag] = np.load(out)
    assert str(res[1]["form"]) == "hodlr"
    rel = float(np.linalg.norm(res[1]["y"] - res[0]["y"]) / np.linalg.norm(res[0]["y"]))
    Ao = O.SystemOperator(O.make_problem("paper1d", beta, omega, [1023], 48, 5e-3, 0.01))
    z = res[1]["z"]
    yo = O.BlockTriangularPreconditioner(Ao).apply(z)
    fwd = float(np.linalg.norm(res[1]["y"] - yo) / np.linalg.norm(yo))
    bwd = float(np.linalg.norm(Ao.apply_precond_matrix(res[1]["y1"]) - z) / np.linalg.norm(z))
    print(f"(beta, omega) = ({beta}, {omega}): HODLR vs tiles {rel:.3e}, vs oracle LU {fwd:.3e}, "
          f"backward error (refined) {bwd:.3e}")
    assert rel <= 1e-11 and fwd <= 1e-12 and bwd <= 1e-12


def test_hodlr_form_selection():
    # 1D with >= 2 leaves -> HODLR; one leaf -> tiles; 2D dense blocks fail the rank-32 probe -> tiles
    A1 = F.SystemOperator(baseline_problem(F, 0))
    assert F.BlockTriangularPreconditioner(A1).form == "hodlr"
    small = F.make_problem("paper1d", 0.5, 1.5, [32], 8, 5e-3, 0.01)
    assert F.BlockTriangularPreconditioner(F.SystemOperator(small)).form == "tiles"
    grid = F.SpaceGrid([15, 15], [0.0, 0.0], [1.0, 1.0])
    X = grid.nodes()
    spec2 = F.make_custom_problem(F.FractionalOrders(0.3, 1.2), grid, 8, 1.0, lambda X, t: 1 + X[:, 0] * X[:, 1],
                                  lambda X, t: 1 + X[:, 0] * (1 + t), lambda t: 1 + t * t, np.zeros(X.shape[0]),
                                  np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1]), 1e-3, 0.01)
    assert F.BlockTriangularPreconditioner(F.SystemOperator(spec2), inner="lu").form == "tiles"


def test_hodlr_apply_is_bit_reproducible():
    # fixed-order reductions and level-tagged exchange: two applies give identical bits
    A = F.SystemOperator(baseline_problem(F, 0))
    P = F.BlockTriangularPreconditioner(A)
    z = np.random.default_rng(8).uniform(-1, 1, A.dim())
    y1, y2 = P.apply(z), P.apply(z)
    assert P.form == "hodlr" and np.array_equal(y1, y2)


_CHILD_REPEAT = r"""
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
from paper_2507_02809_b200 import fracinv as F
from paper_2507_02809_b200.configs import baseline_problem
A = F.SystemOperator(baseline_problem(F, 1))
P = F.BlockTriangularPreconditioner(A)
z = np.random.default_rng(5).uniform(-1, 1, A.dim())
y0 = P.apply(z)
bad = sum(not np.array_equal(P.apply(z), y0) for _ in range(int(os.environ["REPS"])))
print(P.form, bad)
"""


@pytest.mark.parametrize("hodlr", [1, 0])
def test_persistent_sweeps_repeat_bit_exactly(hodlr):
    """Race check of both persistent P^{-1} kernels (hodlr_sweep_kernel; sweep_ir_kernel, whose
    B-tile steps run ahead of their consumer): repeated applies on BASELINE config 1 are identical."""
    env = dict(os.environ, FI_HODLR=str(hodlr), REPS="40", ROOT=ROOT)
    out = subprocess.run([sys.executable, "-c", _CHILD_REPEAT], env=env, check=True, timeout=900,
                         capture_output=True, text=True).stdout.split()
    assert out[-2] == ("hodlr" if hodlr else "tiles") and out[-1] == "0", out


@pytest.mark.parametrize("cfg", [0, 1])
def test_hodlr_build_check(cfg):
    """The build's a-posteriori check of every level's compressed inverse on 4 probe vectors: the forward
    error against the uncompressed inverse and the normwise backward error in the block matrix itself."""
    A = F.SystemOperator(baseline_problem(F, cfg))
    P = F.BlockTriangularPreconditioner(A)
    chk = P.build_check()
    print(f"config{cfg} HODLR build check: forward {chk['forward']:.3e}, backward {chk['backward']:.3e}")
    assert P.form == "hodlr"
    assert 0.0 < chk["forward"] <= 1e-12 and 0.0 < chk["backward"] <= 1e-13


_CHILD_ZSKIP = r"""
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
from oracle import fracinv_oracle as O
from paper_2507_02809_b200 import fracinv as F
from paper_2507_02809_b200.configs import baseline_problem
A, Ao = F.SystemOperator(baseline_problem(F, 0)), O.SystemOperator(baseline_problem(O, 0))
P, Po = F.BlockTriangularPreconditioner(A), O.BlockTriangularPreconditioner(Ao)
assert P.form == "hodlr"
N, S = Ao.N, Ao.steps
for first in (0, 1, 15, 16, 37, 64):
    z = np.random.default_rng(21).uniform(-1, 1, A.dim())
    z[: first * N] = 0.0
    y, yo = P.apply(z), Po.apply(z)
    assert float(np.linalg.norm(y - yo) / np.linalg.norm(yo)) <= 1e-12, first
    # exact zeros below the 16-level block the sweep starts at; the zero levels it does run carry the level tag
    # in the last mantissa bit of the exchanged values (denormals)
    assert not np.any(y[: (first & ~15) * N]) and np.all(np.abs(y[: first * N]) <= 1e-300), first
    if first >= 16:  # one tiny entry on level 0 disables the skip: the sweep from level 0 gives the same result
        z2 = z.copy()
        z2[0] = 1e-300
        y2 = P.apply(z2)
        assert float(np.linalg.norm(y - y2) / np.linalg.norm(y2)) <= 1e-14, first
print("ok")
"""


def test_hodlr_sweep_skips_leading_zero_levels():
    """FI_HODLR_ZSKIP=1 (opt-in; a separate process, the switch is read once): GMRES's first apply is
    P^-1 [0; ..; mu] when the initial state is zero, and the sweep then starts at the 16-level block of the first
    nonzero time level (first = 64: only the f-block is nonzero).  Same result as the oracle's LU substitution
    (krylov.cpp:48-70), exact zeros below, and as the sweep run from level 0."""
    env = dict(os.environ, FI_HODLR_ZSKIP="1", ROOT=ROOT)
    r = subprocess.run([sys.executable, "-c", _CHILD_ZSKIP], env=env, timeout=600, capture_output=True, text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
