"""Shared test helpers (restating tests/test_helpers.hpp of the reference)."""
import math
import os

import numpy as np

from oracle import fracinv_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
REFERENCE_FIXTURES = "/root/reference/proj/tests/fixtures"


def load_csv(name, directory=GOLDEN):
    """test_helpers.hpp:24-40 — numeric rows, header skipped."""
    rows = []
    with open(os.path.join(directory, name)) as f:
        next(f)
        for line in f:
            line = line.strip()
            if line:
                rows.append([float(c) for c in line.split(",")])
    return rows


class RandomVectors:
    """test_helpers.hpp:43-65: sequential SplitMix64 mapped to (-1, 1)."""

    M = (1 << 64) - 1

    def __init__(self, seed):
        self.state = seed & self.M

    def next_double(self):
        self.state = (self.state + 0x9E3779B97F4A7C15) & self.M
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        z ^= z >> 31
        return 2.0 * (((z >> 11) + 0.5) / 9007199254740992.0) - 1.0

    def vector(self, n):
        # vectorised form of n sequential next_double() calls
        idx = np.arange(1, n + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + idx * np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + n * 0x9E3779B97F4A7C15) & self.M
        return 2.0 * (((z >> np.uint64(11)).astype(np.float64) + 0.5) / 9007199254740992.0) - 1.0


def paper_problem(beta, omega, n, S, lam=5e-3, eps=0.01):
    """test_helpers.hpp:68-71."""
    return O.make_problem("paper1d", beta, omega, [n], S, lam, eps)


def test_problem_2d(beta, omega, n, S, lam=5e-3, eps=0.01):
    """test_helpers.hpp:75-91: variable-coefficient 2D problem with a shared h."""
    pi = math.pi
    h = pi / (n[0] + 1)
    grid = O.SpaceGrid(n, [0.0, 0.0], [pi, h * (n[1] + 1)])
    X = grid.nodes()
    f = X[:, 0] * np.sin(X[:, 0]) * np.sin(X[:, 1])
    return O.make_custom_problem(
        O.FractionalOrders(beta, omega), grid, S, 1.0,
        lambda X, t: t * np.exp(X[:, 0]) * (1.0 + 0.5 * X[:, 1]),
        lambda X, t: t * t * (X[:, 0] + 0.25 * X[:, 1] + 0.1),
        lambda t: t * t, np.zeros(X.shape[0]), f, lam, eps)


test_problem_2d.__test__ = False
