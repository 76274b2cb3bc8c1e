"""The oracle's substituted per-block solve (TauPCG: tau-preconditioned CG, extrapolated initial guesses chosen
by measurement, rounding-floor stopping rule) against the reference's dense LU block solve (krylov.cpp:48-70) on
an input that is smooth in time, and the guess weights against the device's literals."""
import math
import os
import re
import warnings

import numpy as np

from oracle import fracinv_oracle as O

warnings.filterwarnings("ignore", module="scipy")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def smooth_problem(M, n=(15, 15), S=64, beta=0.7, omega=1.5):
    grid = M.SpaceGrid(list(n), [0.0, 0.0], [1.0, 1.0])
    X = grid.nodes()
    return M.make_custom_problem(
        M.FractionalOrders(beta, omega), grid, S, 1.0,
        lambda X, t: 1.0 + 0.5 * np.sin(math.pi * X[:, 0]) * np.exp(-t) + X[:, 1],
        lambda X, t: 1.0 + X[:, 0] * X[:, 1] * (1.0 + t),
        lambda t: 1.0 + t * t, np.zeros(X.shape[0]), np.sin(math.pi * X[:, 0]) * np.sin(2 * math.pi * X[:, 1]),
        1e-3, 0.01)


def arnoldi_like_input(A):
    """(A - P) [0; g]: -eta q_s g on every time level (what the split Arnoldi step feeds P^-1), 0 in the f-block."""
    N, S = A.N, A.steps
    g = np.random.default_rng(3).uniform(-1, 1, N)
    u = np.zeros(A.dim)
    u[: S * N] = (-A.spec.tgrid.eta * A.q[:, None] * g[None, :]).reshape(-1)
    return u


def test_ls_weights_reproduce_polynomials_and_match_device_literals():
    w = O.LS_COEF
    assert len(w) == O.LS_WINDOW == 10
    for d in range(O.WARM_ORDER):  # exact for degree <= 5: sum_j w_j (-j)^d = 0^d
        assert abs(sum(wj * float(-(j + 1)) ** d for j, wj in enumerate(w)) - (1.0 if d == 0 else 0.0)) <= 1e-9
    assert abs(math.sqrt(sum(v * v for v in w)) - 6.0937) < 1e-3
    src = open(os.path.join(ROOT, "paper_2507_02809_b200", "csrc", "precond_iter.cu")).read()
    lit = re.search(r"kLsCoef\[kLsWindow\] = \{([^}]*)\}", src).group(1)
    assert [float(v) for v in lit.split(",")] == w  # the same doubles on both sides
    rows = re.search(r"kWarmCoef\[kLsWindow \+ 1\]\[kLsWindow \+ 1\] = \{(.*?)\};", src, re.S).group(1)
    table = [[float(v) for v in r.split(",")] for r in re.findall(r"\{([^{}]*)\}", rows)]
    assert len(table) == 11
    for k in range(11):
        assert table[k] == [float((-1) ** (j + 1) * math.comb(k, j)) if 1 <= j <= k else 0.0 for j in range(11)]


def test_tau_pcg_with_guesses_matches_lu_on_a_smooth_input():
    A = O.SystemOperator(smooth_problem(O))
    Pp = O.BlockTriangularPreconditioner(A, inner="pcg")
    Pl = O.BlockTriangularPreconditioner(A, inner="lu")
    u = arnoldi_like_input(A)
    kinds = []
    ww = Pp.pcg.warm_weights
    Pp.pcg.warm_weights = lambda nprev, level=0: (ww(nprev, level), kinds.append(Pp.pcg.kind))[0]
    y, yl = Pp.apply(u), Pl.apply(u)
    steps_new = sum(Pp.pcg.iterations)
    assert _rel(y, yl) <= 1e-12
    assert not Pp.pcg.dropped and {1, 2, 3} <= set(kinds)  # the trial levels ran every kind
    # the previous rule (tol ||b|| alone, six-point interpolation everywhere): the same solution, more steps
    Pold = O.BlockTriangularPreconditioner(A, inner="pcg")
    Pold.pcg.theta, Pold.pcg.lswin = 0.0, 0
    yo = Pold.apply(u)
    assert _rel(yo, yl) <= 1e-12 and _rel(y, yo) <= 1e-12
    assert steps_new <= sum(Pold.pcg.iterations)


def test_tau_pcg_random_input_drops_the_guess():
    A = O.SystemOperator(smooth_problem(O, S=24))
    Pp = O.BlockTriangularPreconditioner(A, inner="pcg")
    Pl = O.BlockTriangularPreconditioner(A, inner="lu")
    z = np.random.default_rng(8).uniform(-1, 1, A.dim)
    assert _rel(Pp.apply(z), Pl.apply(z)) <= 1e-12
    assert Pp.pcg.dropped
