"""GPU parity of the substituted per-block solve (tau-preconditioned CG, precond_iter.cu) used for the
2D configurations whose blocks exceed the reference's dense cap (BASELINE configs 2-4)."""
import math
import os
import warnings

import numpy as np
import pytest

from helpers import RandomVectors
from oracle import fracinv_oracle as O
from paper_2507_02809_b200.configs import NOISE, RESTART, SEED_BASE, TOL, baseline_problem

pytestmark = pytest.mark.gpu
warnings.filterwarnings("ignore", module="scipy")
F = pytest.importorskip("paper_2507_02809_b200.fracinv")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def _problem2d(M, n, S, beta=0.5, omega=1.5):
    h = math.pi / (n[0] + 1)
    grid = M.SpaceGrid(n, [0.0, 0.0], [math.pi, h * (n[1] + 1)])
    X = grid.nodes()
    return M.make_custom_problem(
        M.FractionalOrders(beta, omega), grid, S, 1.0,
        lambda X, t: t * np.exp(X[:, 0]) * (1.0 + 0.5 * X[:, 1]),
        lambda X, t: t * t * (X[:, 0] + 0.25 * X[:, 1] + 0.1),
        lambda t: t * t, np.zeros(X.shape[0]), X[:, 0] * np.sin(X[:, 0]) * np.sin(X[:, 1]), 5e-3, 0.01)


@pytest.mark.parametrize("n,S,beta,omega", [([7, 7], 8, 0.5, 1.5), ([15, 15], 8, 0.1, 1.9), ([15, 7], 6, 0.9, 1.1)])
def test_tau_pcg_matches_dense_and_oracle(n, S, beta, omega):
    A, Ao = F.SystemOperator(_problem2d(F, n, S, beta, omega)), O.SystemOperator(_problem2d(O, n, S, beta, omega))
    Pi = F.BlockTriangularPreconditioner(A, inner="pcg")
    Pd = F.BlockTriangularPreconditioner(A, inner="lu")
    assert Pi.inner == "pcg" and Pd.inner == "lu"
    Po = O.BlockTriangularPreconditioner(Ao, inner="pcg")
    Pl = O.BlockTriangularPreconditioner(Ao, inner="lu")
    rng = RandomVectors(5)
    for _ in range(3):
        z = rng.vector(A.dim())
        yi = Pi.apply(z)
        assert _rel(yi, Po.apply(z)) <= 1e-12
        assert _rel(yi, Pl.apply(z)) <= 1e-12
        assert _rel(yi, Pd.apply(z)) <= 1e-12


def test_config2_uses_tau_pcg_and_matches_oracle():
    A, Ao = F.SystemOperator(baseline_problem(F, 2)), O.SystemOperator(baseline_problem(O, 2))
    P = F.BlockTriangularPreconditioner(A)
    assert P.inner == "pcg"  # N = 16129 > cap 4096: the reference itself would raise here
    Po = O.BlockTriangularPreconditioner(Ao)
    assert Po.inner == "pcg"
    z = RandomVectors(9).vector(A.dim())
    y = P.apply(z)
    par = _rel(y, Po.apply(z))
    bwd = _rel(Ao.apply_precond_matrix(y), z)
    print(f"config2 tau-PCG P: parity {par:.3e}, backward error {bwd:.3e}, oracle CG steps max "
          f"{max(Po.pcg.iterations)}")
    assert par <= 1e-12 and bwd <= 1e-12


def test_config3_backward_error():
    A, Ao = F.SystemOperator(baseline_problem(F, 3)), O.SystemOperator(baseline_problem(O, 3))
    P = F.BlockTriangularPreconditioner(A)
    z = RandomVectors(10).vector(A.dim())
    y = P.apply(z)
    bwd = _rel(Ao.apply_precond_matrix(y), z)
    print(f"config3 tau-PCG P: backward error {bwd:.3e}")
    assert bwd <= 1e-12


def test_config2_end_to_end_vs_golden():
    path = os.path.join(GOLDEN, "oracle_config2.npz")
    if not os.path.exists(path):
        pytest.skip("oracle golden for config 2 not generated")
    g = np.load(path)
    A = F.SystemOperator(baseline_problem(F, 2))
    P = F.BlockTriangularPreconditioner(A)
    z = F.build_rhs(A, g["mu_eps"]).z
    x, rep = F.gmres(A, P, z, F.GmresOptions(TOL[2], 0, RESTART))
    print(f"config2: {rep.iterations} iterations (oracle {int(g['iterations'])}), "
          f"f parity {_rel(x[-A.N:], g['f']):.3e}")
    assert rep.converged and abs(rep.iterations - int(g["iterations"])) <= 1
    assert _rel(x[-A.N:], g["f"]) <= 1e-8


def test_config2_forward_solve_parity():
    A, Ao = F.SystemOperator(baseline_problem(F, 2)), O.SystemOperator(baseline_problem(O, 2))
    P = F.BlockTriangularPreconditioner(A)
    Po = O.BlockTriangularPreconditioner(Ao)
    mu, muo = F.forward_solve(A, P).mu, O.forward_solve(Ao, P=Po).mu
    print(f"config2 forward solve parity {_rel(mu, muo):.3e}")
    assert _rel(mu, muo) <= 1e-12


def test_tau_pcg_guesses_and_floor_on_a_smooth_input():
    """The input a solve feeds P^-1 (smooth in time: the guesses are used, every kind is tried on the trial
    levels, levels stop at the rounding floor): device against the oracle's tau-PCG and the reference's LU block
    solves (krylov.cpp:48-70); CG steps as the oracle's."""
    from test_oracle_taupcg import arnoldi_like_input, smooth_problem
    A, Ao = F.SystemOperator(smooth_problem(F)), O.SystemOperator(smooth_problem(O))
    P = F.BlockTriangularPreconditioner(A, inner="pcg")
    Po, Pl = O.BlockTriangularPreconditioner(Ao, inner="pcg"), O.BlockTriangularPreconditioner(Ao, inner="lu")
    u = arnoldi_like_input(Ao)
    P.stats(reset=True)
    y = P.apply(u)
    st = P.stats()
    yo, yl = Po.apply(u), Pl.apply(u)
    so = sum(Po.pcg.iterations)
    print(f"smooth input: device vs oracle tau-PCG {_rel(y, yo):.3e}, vs LU {_rel(y, yl):.3e}, CG steps device "
          f"{st['cg_steps']} / oracle {so}")
    assert _rel(y, yo) <= 1e-12 and _rel(y, yl) <= 1e-12
    assert st["nonconverged_blocks"] == 0 and not Po.pcg.dropped
    assert abs(st["cg_steps"] - so) <= max(3, 0.05 * so)
    # leading zero levels (GMRES's first apply: b = [0; ..; mu]) are skipped: same result as the oracle
    z = np.zeros(A.dim())
    z[40 * Ao.N:] = u[40 * Ao.N:]
    z[-Ao.N:] = np.random.default_rng(4).uniform(-1, 1, Ao.N)
    yz, yzo = P.apply(z), Pl.apply(z)
    assert _rel(yz, yzo) <= 1e-12 and not np.any(yz[: 40 * Ao.N])
