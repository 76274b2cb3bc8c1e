"""Oracle pins: preconditioner and GMRES (test_krylov.cpp, acceptance.cpp criterion 5)."""
import math
import warnings

import numpy as np
import pytest

from helpers import RandomVectors, paper_problem
from oracle import fracinv_oracle as O

warnings.filterwarnings("ignore", category=Warning, module="scipy")


def _mat(M):
    return lambda v: M @ v


def test_preconditioner_inverts_dense_realisation():
    A = O.SystemOperator(paper_problem(0.5, 1.5, 8, 4))
    P = O.BlockTriangularPreconditioner(A)
    Pd = O.assemble_dense_system(A, O.PRECONDITIONER_P)
    rng = RandomVectors(3)
    for _ in range(20):
        y = rng.vector(A.dim)
        assert np.linalg.norm(P.apply(Pd @ y) - y) <= 1e-10 * np.linalg.norm(y)
        z = rng.vector(A.dim)
        assert np.linalg.norm(Pd @ P.apply(z) - z) <= 1e-10 * np.linalg.norm(z)
    A = O.SystemOperator(O.make_problem("constant", 0.5, 1.5, [4], 2, 1e-2, 0.0))
    P = O.BlockTriangularPreconditioner(A)
    Pd = O.assemble_dense_system(A, O.PRECONDITIONER_P)
    y = RandomVectors(31).vector(A.dim)
    assert np.linalg.norm(P.apply(Pd @ y) - y) <= 1e-12 * np.linalg.norm(y)
    # uncached (refactor per apply) is the same arithmetic
    Pu = O.BlockTriangularPreconditioner(A, cache=False)
    assert np.array_equal(Pu.apply(y), P.apply(y))


def test_preconditioner_singular_final_block_and_cap():
    one = lambda X, t: np.ones(X.shape[0])
    spec = O.make_custom_problem(O.FractionalOrders(0.5, 1.5), O.SpaceGrid([4], [0.0], [math.pi]), 2, 1.0,
                                 one, lambda X, t: np.full(X.shape[0], 1.0 - t), lambda t: 1.0,
                                 np.zeros(4), np.zeros(4), 1e-2, 0.0)
    with pytest.raises(O.SingularBlockError) as ex:
        O.BlockTriangularPreconditioner(O.SystemOperator(spec))
    assert ex.value.time_index == 3
    with pytest.raises(O.ResourceLimitError):
        O.BlockTriangularPreconditioner(O.SystemOperator(paper_problem(0.5, 1.5, 16, 4)), 8)


def test_precond_zero_dims_and_scalar_reduction():
    A = O.SystemOperator(paper_problem(0.5, 1.5, 6, 3))
    P = O.BlockTriangularPreconditioner(A)
    assert np.linalg.norm(P.apply(np.zeros(A.dim))) == 0.0
    with pytest.raises(O.DimensionError):
        P.apply(np.zeros(A.dim - 1))
    spec = O.make_custom_problem(O.FractionalOrders(0.5, 1.5), O.SpaceGrid([1], [0.0], [2.0]), 1, 1.0,
                                 lambda X, t: np.full(X.shape[0], 2.0), lambda X, t: np.full(X.shape[0], 3.0),
                                 lambda t: 1.0, np.zeros(1), np.zeros(1), 7e-3, 0.0)
    A = O.SystemOperator(spec)
    P = O.BlockTriangularPreconditioner(A)
    a0, eta = A.laplacian.sym.at(0), A.spec.tgrid.eta
    z = np.array([0.8, -1.1])
    y = P.apply(z)
    y1 = z[0] / (2.0 + eta * 3.0 * a0)
    assert y[0] == pytest.approx(y1, rel=1e-14)
    assert y[1] == pytest.approx((z[1] - y1) / (7e-3 * 3.0 * a0), rel=1e-14)


def test_gmres_known_answers():
    b = RandomVectors(2).vector(12)
    y, rep = O.gmres(_mat(np.eye(12)), None, b)
    assert rep.converged and rep.iterations == 1 and np.linalg.norm(y - b) <= 1e-12 * np.linalg.norm(b)
    y, rep = O.gmres(_mat(np.diag([2.0, 3.0])), None, np.array([2.0, 3.0]))
    assert rep.converged and rep.iterations <= 2 and np.linalg.norm(y - 1) <= 1e-10
    diag = np.array([1.0, 2.5, 4.0, 7.5, 10.0])[np.arange(60) % 5]
    b = RandomVectors(8).vector(60)
    y, rep = O.gmres(_mat(np.diag(diag)), None, b, tol=1e-12)
    assert rep.converged and rep.iterations <= 5
    assert np.linalg.norm(diag * y - b) <= 1e-10 * np.linalg.norm(b)
    y, rep = O.gmres(_mat(np.eye(5)), None, np.zeros(5))
    assert rep.converged and rep.iterations == 0 and np.linalg.norm(y) == 0.0
    assert rep.residual_history == [0.0]


def test_gmres_monotone_history_random_dense():
    rng = RandomVectors(13)
    for trial in range(20):
        n = 20 + 4 * trial
        M = np.array([rng.next_double() for _ in range(n * n)]).reshape(n, n)
        M += 2.0 * math.sqrt(n) * np.eye(n)
        b = rng.vector(n)
        y, rep = O.gmres(_mat(M), None, b, tol=1e-10)
        assert rep.converged
        h = rep.residual_history
        assert all(h[i] <= h[i - 1] * (1 + 1e-15) for i in range(1, len(h)))
        assert rep.final_true_residual <= 1e-8


def test_gmres_maxit_and_breakdown():
    A = O.SystemOperator(paper_problem(0.1, 1.9, 8, 4))
    rhs = O.build_rhs(A, O.add_noise(O.forward_solve(A).mu, 0.01, 1))
    y, rep = O.gmres(A.apply, None, rhs.z, tol=1e-8, maxit=3)
    assert not rep.converged and rep.iterations == 3 and len(rep.residual_history) == 4
    M = np.diag([1.0, 1.0, 0.0])
    y, rep = O.gmres(_mat(M), None, np.ones(3), tol=1e-8)
    assert rep.breakdown and not rep.converged and rep.residual_history[-1] > 1e-8
    assert rep.final_true_residual == pytest.approx(1 / math.sqrt(3), rel=1e-10)


def test_gmres_restart_semantics():
    rng = RandomVectors(21)
    n = 80
    M = np.array([rng.next_double() for _ in range(n * n)]).reshape(n, n) + 3.0 * math.sqrt(n) * np.eye(n)
    b = rng.vector(n)
    yf, rf = O.gmres(_mat(M), None, b, tol=1e-10)
    yr, rr = O.gmres(_mat(M), None, b, tol=1e-10, restart=5)
    assert rr.converged and rr.iterations >= rf.iterations
    assert len(rr.residual_history) == rr.iterations + 1
    assert np.linalg.norm(M @ yr - b) <= 1e-8 * np.linalg.norm(b)
    # restart >= iterations needed is the full method, bit for bit
    y2, r2 = O.gmres(_mat(M), None, b, tol=1e-10, restart=rf.iterations)
    assert r2.iterations == rf.iterations and np.array_equal(y2, yf)
    # maxit bounds the total across cycles
    y3, r3 = O.gmres(_mat(M), None, b, tol=1e-14, maxit=7, restart=3)
    assert r3.iterations == 7 and len(r3.residual_history) == 8 and not r3.converged


def test_preconditioned_iterations_bounded():
    for S in (8, 16):
        A = O.SystemOperator(paper_problem(0.5, 1.5, 16, S))
        P = O.BlockTriangularPreconditioner(A)
        rhs = O.build_rhs(A, O.add_noise(O.forward_solve(A).mu, 0.01, 1))
        y, rep = O.gmres(A.apply, P.apply, rhs.z)
        assert rep.converged and rep.iterations <= 17


TABLE2 = [  # acceptance.cpp:175-180: (n, S, unprec[3], prec[3]) for (0.1,1.9),(0.5,1.5),(0.9,1.1)
    (16, 16, (174, 117, 112), (8, 10, 13)),
    (16, 32, (257, 146, 154), (8, 11, 13)),
    (32, 16, (320, 181, 151), (9, 11, 15)),
    (32, 32, (475, 217, 199), (8, 11, 15)),
]
ORDERS = [(0.1, 1.9), (0.5, 1.5), (0.9, 1.1)]


@pytest.mark.parametrize("n,S,unprec,prec", TABLE2)
def test_table2_iteration_counts(n, S, unprec, prec):
    """Paper Table 2 with the reference's tolerances: P-preconditioned +-2,
    unpreconditioned +-10 % (acceptance.cpp:199-204)."""
    for k, (beta, omega) in enumerate(ORDERS):
        A = O.SystemOperator(paper_problem(beta, omega, n, S, 5e-3, 0.01))
        P = O.BlockTriangularPreconditioner(A)
        rhs = O.build_rhs(A, O.add_noise(O.forward_solve(A).mu, 0.01, 1))
        yu, ru = O.gmres(A.apply, None, rhs.z, tol=1e-8)
        yp, rp = O.gmres(A.apply, P.apply, rhs.z, tol=1e-8)
        assert ru.converged and rp.converged
        assert abs(rp.iterations - prec[k]) <= 2, (beta, omega, rp.iterations)
        assert abs(ru.iterations - unprec[k]) <= 0.10 * unprec[k], (beta, omega, ru.iterations)


def test_inverse_crime():
    A = O.SystemOperator(paper_problem(0.1, 1.9, 32, 32, 1e-8, 0.0))
    rhs = O.build_rhs(A, O.forward_solve(A).mu)
    y = np.linalg.solve(O.assemble_dense_system(A, O.SYSTEM_A), rhs.z)
    assert O.relative_error(A.spec.f_true, O.extract_reconstruction(y, 32)) <= 1e-3
