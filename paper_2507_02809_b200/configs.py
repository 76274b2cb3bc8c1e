"""BASELINE.json configurations 0-4 as problem specifications.

`baseline_problem(M, cfg)` builds the ProblemSpec through the API module `M` — either the
product (`paper_2507_02809_b200.fracinv`) or, in tests and the CPU baseline, the oracle —
so both sides assemble identical inputs.  Data are synthetic by construction: the
observation mu is manufactured by the forward solve of f* and perturbed with seeded
Gaussian noise of the stated relative L2 level (`NOISE[cfg]`, seed `SEED_BASE + cfg`).
"""
import math

import numpy as np

# (relative L2 noise, GMRES tol, restart) per config (BASELINE.json configs[i])
NOISE = {0: 0.01, 1: 0.005, 2: 0.01, 3: 0.01, 4: 0.05}
TOL = {0: 1e-10, 1: 1e-10, 2: 1e-10, 3: 1e-10, 4: 1e-8}
RESTART = 50
SEED_BASE = 1000
# (interior points per direction, time steps) per config: the shapes both bench arms report
SHAPES = {0: ((255,), 64), 1: ((4095,), 512), 2: ((127, 127), 128), 3: ((255, 255), 256), 4: ((255, 255), 512)}
NAMES = {0: "config0_1d_M255_N64", 1: "config1_1d_M4095_N512", 2: "config2_2d_M127x127_N128",
         3: "config3_2d_M255x255_N256", 4: "config4_2d_M255x255_N512"}


def baseline_problem(M, cfg: int):
    pi = math.pi
    if cfg == 0:
        n, S, beta, omega, lam = 255, 64, 0.5, 1.5, 1e-3
        g1 = lambda X, t: 1 + 0.5 * np.sin(pi * X[:, 0]) * np.exp(-t)
        g2 = lambda X, t: 1 + X[:, 0] * (1 - X[:, 0]) * (1 + t)
        q = lambda t: 1 + t
        rho = lambda X: X[:, 0] ** 2 * (1 - X[:, 0]) ** 2
        f = lambda X: np.sin(pi * X[:, 0])
        grid = M.SpaceGrid([n], [0.0], [1.0])
    elif cfg == 1:
        n, S, beta, omega, lam = 4095, 512, 0.9, 1.8, 1e-4
        g1 = lambda X, t: 2 + np.cos(2 * pi * X[:, 0])
        g2 = lambda X, t: 1 + 0.5 * X[:, 0] * t
        q = lambda t: math.exp(-t)
        rho = lambda X: X[:, 0] ** 2 * (1 - X[:, 0]) ** 2  # "same functional setup as config 0"
        f = lambda X: X[:, 0] * (1 - X[:, 0]) * np.exp(X[:, 0])
        grid = M.SpaceGrid([n], [0.0], [1.0])
    elif cfg == 2:
        n, S, beta, omega, lam = 127, 128, 0.3, 1.2, 1e-3
        g1 = lambda X, t: 1 + 0.5 * np.sin(pi * X[:, 0]) * np.sin(pi * X[:, 1])
        g2 = lambda X, t: 1 + X[:, 0] * X[:, 1] * (1 + t)
        q = lambda t: 1 + t * t
        rho = lambda X: np.zeros(X.shape[0])
        f = lambda X: np.sin(pi * X[:, 0]) * np.sin(2 * pi * X[:, 1])
        grid = M.SpaceGrid([n, n], [0.0, 0.0], [1.0, 1.0])
    elif cfg in (3, 4):
        n = 255
        if cfg == 3:
            S, beta, omega, lam = 256, 0.7, 1.5, 1e-4
            g1 = lambda X, t: 1 + X[:, 0] ** 2 + X[:, 1] ** 2
            g2 = lambda X, t: 2 + np.sin(pi * X[:, 0] * X[:, 1]) * np.exp(-t)
            q = lambda t: math.exp(-t)
            f = lambda X: 16 * X[:, 0] * (1 - X[:, 0]) * X[:, 1] * (1 - X[:, 1])
        else:
            S, beta, omega, lam = 512, 0.95, 1.9, 1e-2
            g1 = lambda X, t: 1 + 0.9 * np.sin(3 * pi * X[:, 0]) * np.sin(3 * pi * X[:, 1])
            g2 = lambda X, t: 1 + 10 * X[:, 0] * X[:, 1] * (1 + t)
            q = lambda t: 1.0  # BASELINE.json states no q for config 4
            f = lambda X: (((X[:, 0] >= 0.25) & (X[:, 0] <= 0.75) & (X[:, 1] >= 0.25) & (X[:, 1] <= 0.75))
                           .astype(np.float64))
        rho = lambda X: np.zeros(X.shape[0])
        grid = M.SpaceGrid([n, n], [0.0, 0.0], [1.0, 1.0])
    else:
        raise ValueError(f"unknown BASELINE config {cfg}")
    X = grid.nodes()
    return M.make_custom_problem(M.FractionalOrders(beta, omega), grid, S, 1.0, g1, g2, q, rho(X), f(X), lam,
                                 NOISE[cfg])
