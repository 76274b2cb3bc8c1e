"""K1f — the operator apply with the spatial Toeplitz products by batched 2D FFTs (toeplitz_fft.cu) —
against the CPU oracle (whose apply is the reference's FFT algorithm, toeplitz.cpp:68-114 inside
system.cpp:144-174), against the dense realisation and against K1 (the dense DMMA contraction), on the
reference's test pattern: matrix-free vs reference on random vectors to <= 1e-12 (test_system.cpp:80-99)."""
import math
import warnings

import numpy as np
import pytest

from helpers import RandomVectors
from oracle import fracinv_oracle as O
from paper_2507_02809_b200.configs import RESTART, TOL, baseline_problem

pytestmark = pytest.mark.gpu
warnings.filterwarnings("ignore", module="scipy")
F = pytest.importorskip("paper_2507_02809_b200.fracinv")


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def _problem2d(M, beta, omega, n, S, lam=5e-3):
    grid = M.SpaceGrid(n, [0.0, 0.0], [1.0, (n[1] + 1) / (n[0] + 1)])  # common mesh width
    X = grid.nodes()
    f = np.sin(math.pi * X[:, 0]) * np.sin(2 * math.pi * X[:, 1])
    return M.make_custom_problem(
        M.FractionalOrders(beta, omega), grid, S, 1.0,
        lambda X, t: 1.0 + 0.5 * np.sin(math.pi * X[:, 0]) * np.cos(X[:, 1]) * np.exp(-t),
        lambda X, t: 1.0 + X[:, 0] * X[:, 1] * (1.0 + t),
        lambda t: 1.0 + t * t, np.zeros(X.shape[0]), f, lam, 0.01)


@pytest.mark.parametrize("n,S,beta,omega", [([3, 3], 4, 0.5, 1.5), ([7, 7], 8, 0.1, 1.9), ([15, 7], 6, 0.9, 1.1),
                                            ([7, 31], 5, 0.3, 1.2), ([15, 15], 17, 0.7, 1.5), ([31, 31], 70, 0.7, 1.5)])
def test_fft_apply_matches_oracle_dense_and_dmma(n, S, beta, omega):
    mk = lambda M: _problem2d(M, beta, omega, n, S)
    A, Ao = F.SystemOperator(mk(F)), O.SystemOperator(mk(O))
    assert A.apply_mode == "fft"  # AUTO on a 2D grid with n_i + 1 a power of two
    rng = RandomVectors(29)
    ys = [rng.vector(A.dim()) for _ in range(4)]
    zf = [A.apply(y) for y in ys]
    for y, z in zip(ys, zf):
        assert _rel(z, Ao.apply(y)) <= 1e-12
    if A.dim() <= 4096:  # the dense realisation's cap (spectra.cpp)
        Md = O.assemble_dense_system(Ao, O.SYSTEM_A)
        assert _rel(zf[0], Md @ ys[0]) <= 1e-12
    A.set_apply_mode("dmma")
    assert A.apply_mode == "dmma"
    for y, z in zip(ys, zf):
        assert _rel(A.apply(y), z) <= 1e-13
    A.set_apply_mode("auto")
    assert A.apply_mode == "fft"
    # zero -> zero, linearity (test_system.cpp:49-59)
    assert np.linalg.norm(A.apply(np.zeros(A.dim()))) == 0.0
    assert _rel(A.apply(0.37 * ys[0] + ys[1]), 0.37 * zf[0] + zf[1]) <= 1e-13


def test_fft_mode_refused_where_unsupported():
    one = lambda X, t: np.ones(X.shape[0])
    spec1d = F.make_problem("paper1d", 0.5, 1.5, [32], 8, 5e-3, 0.01)
    A = F.SystemOperator(spec1d)
    assert A.apply_mode == "dmma"
    with pytest.raises(ValueError):
        A.set_apply_mode("fft")
    grid = F.SpaceGrid([6, 5], [0.0, 0.0], [1.0, 6.0 / 7.0])  # n_i + 1 not a power of two
    spec2d = F.make_custom_problem(F.FractionalOrders(0.5, 1.5), grid, 4, 1.0, one, one, lambda t: 1.0,
                                   np.zeros(30), np.zeros(30), 1e-3, 0.0)
    B = F.SystemOperator(spec2d)
    assert B.apply_mode == "dmma"
    with pytest.raises(ValueError):
        B.set_apply_mode("fft")


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_fft_apply_baseline_configs(cfg):
    """Configs 2-4 (the 2D BASELINE grids): K1f against the oracle on the product's coefficient tensor
    (test_gpu_parity_large.py explains why) and against K1, random and smooth inputs."""
    A = F.SystemOperator(baseline_problem(F, cfg))
    sym = O.SymbolCoefficients(A.symbol.omega, A.symbol.n, np.asarray(A.symbol.coeffs))
    Ao = O.SystemOperator(baseline_problem(O, cfg), symbol=sym)
    assert A.apply_mode == "fft"
    y = np.random.default_rng(70 + cfg).uniform(-1, 1, A.dim())
    X = A.spec.sgrid.nodes()
    smooth = np.concatenate([np.sin(math.pi * X[:, 0]) * np.sin(math.pi * X[:, 1]) * (1 + 0.1 * s)
                             for s in range(A.S + 1)])
    for kind, v in (("random", y), ("smooth", smooth)):
        zf = A.apply(v)
        zo = Ao.apply(v)
        A.set_apply_mode("dmma")
        zd = A.apply(v)
        A.set_apply_mode("auto")
        ef, ed = _rel(zf, zo), _rel(zd, zo)
        print(f"config{cfg} {kind}: fft vs oracle {ef:.3e}, dmma vs oracle {ed:.3e}, fft vs dmma {_rel(zf, zd):.3e}")
        if kind == "random":
            assert ef <= 1e-12 and _rel(zf, zd) <= 1e-12
        else:
            # on a vector smooth in space and time A v cancels (||A v|| << |A| |v|): every realisation's
            # rounding shows at ~1e-12 relative; the transforms must be no worse than the dense contraction
            assert ef <= max(1e-12, 1.5 * ed)


def test_gmres_same_with_either_apply():
    """Config 2 (21 iterations): the preconditioned GMRES(50) solve with K1f and with K1 as A (the final
    true residual, and every step in the reference's Arnoldi order) — same iterations, same solution."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_config2.npz"))
    A = F.SystemOperator(baseline_problem(F, 2))
    P = F.BlockTriangularPreconditioner(A)
    z = F.build_rhs(A, g["mu_eps"]).z
    opts = F.GmresOptions(TOL[2], 0, RESTART)
    A.set_split_apply(False)
    x1, r1 = F.gmres(A, P, z, opts)
    A.set_apply_mode("dmma")
    x2, r2 = F.gmres(A, P, z, opts)
    A.set_apply_mode("auto")
    A.set_split_apply(True)
    print(f"config2 reference order: fft {r1.iterations} / dmma {r2.iterations} iterations, solution "
          f"{_rel(x1, x2):.3e}, true residual {r1.final_true_residual:.6e} / {r2.final_true_residual:.6e}")
    assert r1.iterations == r2.iterations == int(g["iterations"])
    assert _rel(x1, x2) <= 1e-10
    assert abs(r1.final_true_residual - r2.final_true_residual) <= 1e-6 * r2.final_true_residual
