"""End-to-end parity against the CPU oracle's GMRES(50) solves of the BASELINE configurations
(tests/golden/oracle_config<i>.npz, made by tests/golden/gen_oracle_solutions.py on the identical
seeded observation mu_eps).  The north star's bar: iteration count +-1, recovered f <= 1e-8."""
import os

import numpy as np
import pytest

from paper_2507_02809_b200.configs import RESTART, TOL, baseline_problem

pytestmark = pytest.mark.gpu
F = pytest.importorskip("paper_2507_02809_b200.fracinv")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_solve_matches_oracle_golden(cfg):
    path = os.path.join(GOLDEN, f"oracle_config{cfg}.npz")
    if not os.path.exists(path):
        pytest.skip(f"oracle golden for config {cfg} not generated")
    g = np.load(path)
    A = F.SystemOperator(baseline_problem(F, cfg))
    P = F.BlockTriangularPreconditioner(A)
    z = F.build_rhs(A, g["mu_eps"]).z
    x, rep = F.gmres(A, P, z, F.GmresOptions(TOL[cfg], 0, RESTART))
    f = x[-A.N:]
    print(f"config{cfg} ({P.inner}): {rep.iterations} iterations (oracle {int(g['iterations'])}), "
          f"f parity {_rel(f, g['f']):.3e}, recon error {F.relative_error(A.spec.f_true, f):.3e} "
          f"(oracle {float(g['recon_error']):.3e})")
    assert rep.converged == bool(g["converged"])
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    assert _rel(f, g["f"]) <= 1e-8
    # the residual history follows the oracle's step by step (same Krylov space, same arithmetic order)
    h, ho = np.asarray(rep.residual_history), np.asarray(g["history"])
    k = min(len(h), len(ho))
    assert np.allclose(h[:k], ho[:k], rtol=1e-4, atol=1e-14)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_split_apply_matches_operator_then_precond(cfg):
    """The default Arnoldi step P^-1 A v = v + P^-1((A - P) v) against the reference's order (K1, then
    P^-1): same iteration count, residual histories to 1e-6, solutions to 1e-10."""
    g = np.load(os.path.join(GOLDEN, f"oracle_config{cfg}.npz"))
    A = F.SystemOperator(baseline_problem(F, cfg))
    P = F.BlockTriangularPreconditioner(A)
    z = F.build_rhs(A, g["mu_eps"]).z
    opts = F.GmresOptions(TOL[cfg], 0, RESTART)
    x1, r1 = F.gmres(A, P, z, opts)
    A.set_split_apply(False)
    x2, r2 = F.gmres(A, P, z, opts)
    A.set_split_apply(True)
    print(f"config{cfg} split vs reference order: iterations {r1.iterations} / {r2.iterations}, solution "
          f"{_rel(x1, x2):.3e}, history max rel diff "
          f"{max(abs(a - b) / max(abs(b), 1e-300) for a, b in zip(r1.residual_history, r2.residual_history)):.3e}")
    assert r1.iterations == r2.iterations
    assert np.allclose(r1.residual_history, r2.residual_history, rtol=1e-6, atol=1e-15)
    assert _rel(x1, x2) <= 1e-10


def test_full_gmres_reference_defaults_grow_the_basis():
    """maxit = 0, restart = 0 are the reference's defaults (krylov.hpp:54-57): full GMRES with maxit = n.
    For config 1 (n = 2.1M) a basis of n + 1 vectors up front would be 35 TB; the basis grows on demand
    and the solve converges in the same iterations as GMRES(50) (fewer than 50 steps)."""
    g = np.load(os.path.join(GOLDEN, "oracle_config1.npz"))
    A = F.SystemOperator(baseline_problem(F, 1))
    P = F.BlockTriangularPreconditioner(A)
    z = F.build_rhs(A, g["mu_eps"]).z
    x, rep = F.gmres(A, P, z, F.GmresOptions(TOL[1], 0, 0))
    assert rep.converged and abs(rep.iterations - int(g["iterations"])) <= 1
    assert _rel(x[-A.N:], g["f"]) <= 1e-8


def test_unpreconditioned_config4_matches_oracle_golden():
    """BASELINE configs[4] is solved twice; this is the unpreconditioned GMRES(50) solve (max 2000
    iterations, tol 1e-8): no preconditioner = the reference's empty apply_M_inv (krylov.cpp:81-83), the
    loop of krylov.cpp:123-186 with the restart extension.  Golden: the oracle's run on the
    same observation (tests/golden/oracle_config4_unprec.npz, gen_oracle_solutions.py 4u)."""
    path = os.path.join(GOLDEN, "oracle_config4_unprec.npz")
    if not os.path.exists(path):
        pytest.skip("oracle golden for the unpreconditioned config-4 solve not generated")
    g = np.load(path)
    A = F.SystemOperator(baseline_problem(F, 4))
    z = F.build_rhs(A, g["mu_eps"]).z
    # the golden records how many iterations the oracle's run covers (2000 = BASELINE's cap)
    maxit = int(g["maxit"]) if "maxit" in g.files else 2000
    x, rep = F.gmres(A, None, z, F.GmresOptions(TOL[4], maxit, RESTART))
    f = x[-A.N:]
    h, ho = np.asarray(rep.residual_history), np.asarray(g["history"])
    print(f"config4 unpreconditioned: {rep.iterations} iterations (oracle {int(g['iterations'])}), converged "
          f"{rep.converged} (oracle {bool(g['converged'])}), f parity {_rel(f, g['f']):.3e}, last history "
          f"{h[-1]:.6e} (oracle {ho[-1]:.6e}), final true residual {rep.final_true_residual:.6e} "
          f"(oracle {float(g['final_true_residual']):.6e})")
    assert rep.converged == bool(g["converged"])
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    assert _rel(f, g["f"]) <= 1e-8
    k = min(len(h), len(ho))
    assert np.allclose(h[:k], ho[:k], rtol=1e-4, atol=1e-14)
    assert abs(rep.final_true_residual - float(g["final_true_residual"])) <= 1e-4 * float(g["final_true_residual"])
