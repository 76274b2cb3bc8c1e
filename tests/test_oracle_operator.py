"""Oracle pins: Toeplitz / system operator / noise / forward solve
(test_toeplitz.cpp, test_system.cpp of the reference)."""
import math

import numpy as np
import pytest

from helpers import RandomVectors, paper_problem, test_problem_2d
from oracle import fracinv_oracle as O


def _grid1(n):
    return O.SpaceGrid([n], [0.0], [math.pi])


def test_toeplitz_identity_and_stencil():
    n = 13
    coeffs = np.zeros(2 * n - 1)
    coeffs[n - 1] = 1.0
    op = O.ToeplitzOperator(_grid1(n), O.SymbolCoefficients(1.5, [n], coeffs))
    x = RandomVectors(1).vector(n)
    assert np.linalg.norm(op.apply(x) - x) <= 1e-14 * np.linalg.norm(x)
    op = O.ToeplitzOperator(_grid1(8), O.symbol_coeffs_1d(2.0, 8))
    y = op.apply(np.ones(8))
    assert y[0] == pytest.approx(1.0, rel=1e-13) and y[-1] == pytest.approx(1.0, rel=1e-13)
    assert np.all(np.abs(y[1:-1]) <= 1e-13)


@pytest.mark.parametrize("omega", [1.1, 1.5, 1.9])
def test_toeplitz_fft_vs_dense(omega):
    for n in (16, 32):
        op = O.ToeplitzOperator(_grid1(n), O.symbol_coeffs_1d(omega, n))
        B = op.dense()
        X = RandomVectors(7).vector(100 * n).reshape(100, n)
        ref = X @ B.T
        err = np.linalg.norm(op.apply(X) - ref, axis=1) / np.linalg.norm(ref, axis=1)
        assert err.max() <= 1e-12
    grid = O.SpaceGrid([5, 2], [0.0, 0.0], [math.pi, math.pi / 2])
    op = O.ToeplitzOperator(grid, O.symbol_coeffs_md(omega, [5, 2]))
    B = op.dense()
    X = RandomVectors(11).vector(1000).reshape(100, 10)
    ref = X @ B.T
    assert (np.linalg.norm(op.apply(X) - ref, axis=1) / np.linalg.norm(ref, axis=1)).max() <= 1e-12


def test_toeplitz_dense_layout_spd_and_cap():
    sym = O.symbol_coeffs_1d(1.5, 2)
    B = O.ToeplitzOperator(_grid1(2), sym).dense()
    assert B[0, 0] == sym.at(0) and B[0, 1] == sym.at(-1) and B[1, 0] == sym.at(1)
    B16 = O.ToeplitzOperator(_grid1(16), O.symbol_coeffs_1d(1.5, 16)).dense()
    assert np.array_equal(B16, B16.T)
    assert np.linalg.eigvalsh(B16).min() > 0
    op = O.ToeplitzOperator(_grid1(8), O.symbol_coeffs_1d(1.5, 8))
    with pytest.raises(O.DimensionError):
        op.apply(np.zeros(9))
    with pytest.raises(O.ResourceLimitError):
        O.ToeplitzOperator(_grid1(5000), O.symbol_coeffs_1d(1.5, 5000)).dense()


def test_sample_fields_points():
    spec = paper_problem(0.5, 1.5, 15, 4)
    diags = O.sample_fields(spec)
    assert diags.D1[3, 7] == pytest.approx(math.exp(math.pi / 2), rel=1e-14)
    assert diags.D2[1, 7] == pytest.approx(0.25 * math.pi / 2, rel=1e-14)


def test_apply_zero_linear_and_scalar_reduction():
    A = O.SystemOperator(paper_problem(0.5, 1.5, 8, 4))
    assert np.linalg.norm(A.apply(np.zeros(A.dim))) == 0.0
    rng = RandomVectors(5)
    y1, y2 = rng.vector(A.dim), rng.vector(A.dim)
    lhs, rhs = A.apply(0.37 * y1 + y2), 0.37 * A.apply(y1) + A.apply(y2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)
    with pytest.raises(O.DimensionError):
        A.apply(np.zeros(A.dim + 1))
    # test_system.cpp:154-171
    one = lambda X, t: np.ones(X.shape[0])
    spec = O.make_custom_problem(O.FractionalOrders(0.5, 1.5), O.SpaceGrid([1], [0.0], [2.0]), 1, 1.0,
                                 one, one, lambda t: 1.0, np.zeros(1), np.zeros(1), 7e-3, 0.0)
    A = O.SystemOperator(spec)
    a0, eta = A.laplacian.sym.at(0), A.spec.tgrid.eta
    y = np.array([1.25, -0.5])
    z = A.apply(y)
    assert z[0] == pytest.approx((1 + eta * a0) * y[0] - eta * y[1], rel=1e-14)
    assert z[1] == pytest.approx(y[0] + 7e-3 * a0 * y[1], rel=1e-14)


@pytest.mark.parametrize("beta,omega", [(0.1, 1.9), (0.5, 1.5), (0.9, 1.1)])
def test_apply_vs_dense(beta, omega):
    rng = RandomVectors(17)
    for A in (O.SystemOperator(paper_problem(beta, omega, 32, 16)),
              O.SystemOperator(test_problem_2d(beta, omega, [4, 3], 8)),
              O.SystemOperator(test_problem_2d(beta, omega, [6, 5], 16))):
        M = O.assemble_dense_system(A, O.SYSTEM_A)
        for _ in range(20):
            y = rng.vector(A.dim)
            ref = M @ y
            assert np.linalg.norm(A.apply(y) - ref) <= 1e-12 * np.linalg.norm(ref)
        P = O.assemble_dense_system(A, O.PRECONDITIONER_P)
        y = rng.vector(A.dim)
        assert np.linalg.norm(A.apply_precond_matrix(y) - P @ y) <= 1e-12 * np.linalg.norm(P @ y)


def test_build_rhs():
    A = O.SystemOperator(paper_problem(0.1, 1.9, 6, 3))
    mu = RandomVectors(9).vector(6)
    z = O.build_rhs(A, mu).z
    assert np.linalg.norm(z[:-6]) == 0.0 and np.array_equal(z[-6:], mu)
    one = lambda X, t: np.ones(X.shape[0])
    spec = O.make_custom_problem(O.FractionalOrders(0.5, 1.5), O.SpaceGrid([3], [0.0], [math.pi]), 2, 1.0,
                                 one, one, lambda t: 1.0, np.ones(3), np.zeros(3), 1e-2, 0.0)
    A = O.SystemOperator(spec)
    z = O.build_rhs(A, np.full(3, 2.5)).z
    b = A.weights.b
    assert np.allclose(z[:3], b[0], rtol=1e-15) and np.allclose(z[3:6], b[1], rtol=1e-15)
    assert np.all(z[6:] == 2.5)
    with pytest.raises(O.DimensionError):
        O.build_rhs(A, np.zeros(4))


def test_forward_solve():
    spec = paper_problem(0.5, 1.5, 8, 4)
    spec.f_true = np.zeros(8)
    sol = O.forward_solve(O.SystemOperator(spec))
    assert np.linalg.norm(sol.mu) == 0.0
    for n, S in ((4, 2), (8, 4)):
        A = O.SystemOperator(paper_problem(0.1, 1.9, n, S))
        sol = O.forward_solve(A)
        Ahat = O.assemble_dense_system(A, O.FORWARD_AHAT)
        v = np.concatenate(sol.states)
        zhat = np.concatenate([A.spec.tgrid.eta * A.q[s] * A.spec.f_true for s in range(S)])
        assert np.linalg.norm(Ahat @ v - zhat) <= 1e-12 * np.linalg.norm(zhat)
        vref = np.linalg.solve(Ahat, zhat)
        assert np.linalg.norm(v - vref) <= 1e-10 * np.linalg.norm(vref)


def test_forward_solve_singular_index():
    spec = O.make_custom_problem(O.FractionalOrders(0.5, 1.5), _grid1(4), 2, 1.0,
                                 lambda X, t: np.zeros(X.shape[0]), lambda X, t: np.full(X.shape[0], t - 0.5),
                                 lambda t: 1.0, np.zeros(4), np.ones(4), 1e-2, 0.0)
    with pytest.raises(O.SingularBlockError) as ex:
        O.forward_solve(O.SystemOperator(spec))
    assert ex.value.time_index == 1


def test_add_noise_uniform():
    mu = RandomVectors(23).vector(32)
    assert np.array_equal(O.add_noise(mu, 0.0, 7), mu)
    a, b, c = O.add_noise(mu, 0.01, 1), O.add_noise(mu, 0.01, 1), O.add_noise(mu, 0.01, 2)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert np.all(np.abs(a - mu) < 0.01)
    with pytest.raises(ValueError):
        O.add_noise(mu, -0.1, 1)
    mean = np.mean([np.linalg.norm(O.add_noise(np.zeros(256), 0.1, s)) for s in range(100)])
    expected = 0.1 * math.sqrt(256 / 3)
    assert 0.8 * expected <= mean <= 1.2 * expected


def test_add_gaussian_noise_relative_l2():
    mu = np.sin(np.linspace(0, 3, 1001))
    for eps in (0.005, 0.01, 0.05):
        out = O.add_gaussian_noise(mu, eps, 1000)
        assert abs(np.linalg.norm(out - mu) - eps * np.linalg.norm(mu)) <= 1e-14 * np.linalg.norm(mu)
    d = O.gaussian_stream(200000, 3)
    assert abs(d.mean()) < 0.01 and abs(d.std() - 1) < 0.01
    assert np.array_equal(O.gaussian_stream(10, 3), O.gaussian_stream(11, 3)[:10])


def test_extract_reconstruction_and_error():
    y = np.array([9, 8, 7, 6, 5, 4, 1, 2, 3.0])
    assert list(O.extract_reconstruction(y, 3)) == [1, 2, 3]
    with pytest.raises(O.DimensionError):
        O.extract_reconstruction(y, 4)
    assert O.relative_error(y, y) == 0.0


def test_q_and_preset_validation():
    one = lambda X, t: np.ones(X.shape[0])
    spec = O.make_custom_problem(O.FractionalOrders(0.5, 1.5), _grid1(4), 2, 1.0, one, one, lambda t: t - 0.5,
                                 np.zeros(4), np.zeros(4), 1e-2, 0.0)
    with pytest.raises(ValueError):
        O.SystemOperator(spec)
    with pytest.raises(O.ConfigError):
        O.make_problem("nope", 0.5, 1.5, [8], 4, 1e-2, 0.0)
    with pytest.raises(O.ConfigError):
        O.make_problem("paper1d", 0.5, 1.5, [4, 4], 4, 1e-2, 0.0)
    O.make_problem("constant", 0.5, 1.5, [4, 4], 4, 1e-2, 0.0)
    with pytest.raises(ValueError):
        O.make_problem("paper1d", 0.5, 1.5, [8], 4, 0.0, 0.0)
