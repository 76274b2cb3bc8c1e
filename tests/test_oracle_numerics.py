"""Oracle pins: numerics.cpp / symbol.cpp restatements vs golden vectors
(test_numerics.cpp, test_symbol.cpp of the reference)."""
import math
import os
from collections import defaultdict

import numpy as np
import pytest

from helpers import GOLDEN, REFERENCE_FIXTURES, RandomVectors, load_csv
from oracle import fracinv_oracle as O


def test_golden_tables_match_reference_fixtures():
    # our regenerated mpmath tables equal the reference's fixtures row for row
    if not os.path.isdir(REFERENCE_FIXTURES):
        pytest.skip("reference tree absent (GPU box)")
    for name in ("gamma_reference.csv", "symbol_coeffs_reference.csv"):
        ours = open(os.path.join(GOLDEN, name)).read().splitlines()
        ref = open(os.path.join(REFERENCE_FIXTURES, name)).read().splitlines()
        assert ours[: len(ref)] == ref


def test_gamma_exact_values():
    assert O.gamma_fn(1.0) == pytest.approx(1.0, rel=1e-14)
    assert O.gamma_fn(5.0) == pytest.approx(24.0, rel=1e-14)
    assert O.gamma_fn(1.5) == pytest.approx(0.8862269254527580, rel=1e-13)
    assert O.gamma_fn(2.0) == pytest.approx(1.0, rel=1e-14)
    for bad in (0.0, -1.5):
        with pytest.raises(ValueError):
            O.gamma_fn(bad)


def test_gamma_matches_60_digit_table():
    for x, expected in load_csv("gamma_reference.csv"):
        assert abs(O.gamma_fn(x) - expected) <= 1e-13 * expected


def test_gamma_recurrence_random_points():
    rng = RandomVectors(42)
    for _ in range(1000):
        x = 0.1 + (0.5 + 0.5 * rng.next_double()) * 39.9
        lhs = O.gamma_fn(x + 1.0)
        assert abs(lhs - x * O.gamma_fn(x)) <= 1e-13 * abs(lhs)


def test_l1_weights_closed_forms_and_telescoping():
    w = O.l1_weights(0.5, 3)
    assert w.b[0] == pytest.approx(1.0, rel=1e-15)
    assert w.b[1] == pytest.approx(math.sqrt(2) - 1, rel=1e-14)
    assert w.e[1] == pytest.approx(math.sqrt(2) - 2, rel=1e-14)
    assert w.e[2] == pytest.approx(math.sqrt(3) - 2 * math.sqrt(2) + 1, rel=1e-12)
    for beta in np.arange(1, 10) / 10:
        w = O.l1_weights(beta, 512)
        assert w.b[0] == 1.0
        assert np.all(w.b > 0) and np.all(np.diff(w.b) < 0) and np.all(w.e[1:] < 0)
        assert np.max(np.abs(np.cumsum(w.e) - w.b)) <= 1e-14
    for beta, S in ((0.0, 4), (1.0, 4), (1.2, 4), (0.5, 0)):
        with pytest.raises(ValueError):
            O.l1_weights(beta, S)


def test_time_grid():
    g = O.time_grid(0.5, 10, 1.0)
    assert g.dt == pytest.approx(0.1, rel=1e-15)
    assert g.eta == pytest.approx(math.sqrt(0.1) * 0.8862269254527580, rel=1e-13)
    assert O.time_grid(0.1, 16, 1.0).eta == pytest.approx(0.7288822022628409628243493, rel=1e-14)
    for args in ((1.0, 10, 1.0), (0.0, 10, 1.0), (0.5, 0, 1.0), (0.5, 10, 0.0), (0.5, 10, -2.0)):
        with pytest.raises(ValueError):
            O.time_grid(*args)


def test_fractional_orders_validation():
    O.FractionalOrders(0.5, 1.5)
    for b, w in ((0.0, 1.5), (0.5, 1.0), (0.5, 2.0)):
        with pytest.raises(ValueError):
            O.FractionalOrders(b, w)


def _symbol_table():
    table = defaultdict(list)
    for omega, l, a in load_csv("symbol_coeffs_reference.csv"):
        table[omega].append(a)
    return table


def test_symbol_1d_omega2_stencil_and_seed():
    sym = O.symbol_coeffs_1d(2.0, 8)
    assert sym.at(0) == pytest.approx(2.0, rel=1e-15)
    assert sym.at(1) == pytest.approx(-1.0, rel=1e-15) and sym.at(-1) == pytest.approx(-1.0, rel=1e-15)
    assert all(sym.at(l) == 0.0 for l in range(2, 8))
    sym = O.symbol_coeffs_1d(1.5, 4)
    assert abs(sym.at(0) - 1.573787465354794968) <= 1e-13 * 1.574
    assert abs(sym.at(1) + 0.6744803422949121292) <= 1e-13
    for args in ((0.0, 4), (-1.0, 4), (2.5, 4), (1.5, 0)):
        with pytest.raises(ValueError):
            O.symbol_coeffs_1d(*args)


def test_symbol_1d_matches_golden_table():
    for omega, a in _symbol_table().items():
        a = np.array(a)
        sym = O.symbol_coeffs_1d(omega, a.size)
        got = sym.coeffs[a.size - 1:]
        # 5e-13 is the reference's bound on l<=255 (test_symbol.cpp:190-201); the 4094-step
        # recursion for omega=1.8 (config 1) accumulates ~l ulps
        tol = np.where(np.arange(a.size) < 256, 5e-13, 2e-12)
        assert np.all(np.abs(got - a) <= tol * np.abs(a)), omega
        assert np.all(got[1:] < 0) and got[0] > 0
        assert np.array_equal(sym.coeffs[: a.size - 1][::-1], got[1:])


def test_symbol_md_matches_1d_closed_form():
    for omega in (1.1, 1.5, 1.9):
        ref = O.symbol_coeffs_1d(omega, 16)
        fft = O.symbol_coeffs_md(omega, [16])
        assert np.max(np.abs(fft.coeffs - ref.coeffs)) <= 1e-10


def test_symbol_2d_symmetry_and_quadrature():
    sym = O.symbol_coeffs_md(1.9, [4, 4])
    T = sym.tensor()
    assert T[3, 3] > 0
    assert np.allclose(T, T[::-1, ::-1], rtol=1e-13, atol=0)
    assert np.allclose(T, T.T, rtol=1e-13, atol=0)
    for l in range(1, 4):
        assert sym.at([l, 0]) < 0 and sym.at([0, l]) < 0 and sym.at([-l, 0]) < 0
    # test_symbol.cpp:122-165: brute-force rectangle rule at M=2048 per direction
    M = 2048
    th = 2 * math.pi * np.arange(M) / M
    s2 = 4 * np.sin(th / 2) ** 2
    g = np.power(s2[:, None] + s2[None, :], 1.9 / 2)
    for l1, l2 in ((0, 0), (1, 0), (1, 1), (2, 1)):
        quad = float(np.sum(g * np.cos(l1 * th[:, None] + l2 * th[None, :]))) / (M * M)
        assert abs(sym.at([l1, l2]) - quad) <= 1e-8
    with pytest.raises(O.ResourceLimitError):
        O.symbol_coeffs_md(1.5, [5000, 5000])


def test_space_grid():
    g = O.SpaceGrid([3], [0.0], [math.pi])
    assert g.h == pytest.approx(math.pi / 4, rel=1e-15)
    assert np.allclose(g.nodes()[:, 0], [math.pi / 4, math.pi / 2, 3 * math.pi / 4])
    with pytest.raises(ValueError):
        O.SpaceGrid([0], [0.0], [1.0])
    with pytest.raises(ValueError):
        O.SpaceGrid([4], [1.0], [0.0])
    with pytest.raises(ValueError):
        O.SpaceGrid([4, 4], [0.0, 0.0], [1.0, 2.0])
    O.SpaceGrid([4, 9], [0.0, 0.0], [1.0, 2.0])
    nodes2 = O.SpaceGrid([2, 3], [0.0, 0.0], [1.0, 4.0 / 3.0]).nodes()
    assert nodes2.shape == (6, 2)
    assert nodes2[0] == pytest.approx([1 / 3, 1 / 3]) and nodes2[1, 1] == pytest.approx(2 / 3)
    assert nodes2[3, 0] == pytest.approx(2 / 3)
