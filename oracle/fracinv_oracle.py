"""CPU oracle for the fracinv preconditioned-GMRES path — TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference C++ library
(`/root/reference/proj`, "fracinv", arXiv 2507.02809).  It exists to check the
B200 product (`paper_2507_02809_b200`) and to time a CPU baseline.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import it; the product never does.

Every function cites the reference file:line it restates.  Third-party
arithmetic of the reference (FFTW3 for the circulant matvec, Eigen's
PartialPivLU) is replaced by numpy.fft (pocketfft) and LAPACK getrf via
scipy; those boundaries are pinned only to tolerance in the reference's own
tests as well (test_toeplitz.cpp:51-79, test_krylov.cpp:25-47).

Parity pins (see tests/test_oracle_*.py):
  * Gamma vs the 60-digit mpmath table (tests/golden/gamma_reference.csv),
  * 1D generating vector vs the mpmath direct-quotient table,
  * operator vs dense assembly, preconditioner vs dense inverse,
  * GMRES known-answer tests and the paper's Table 2 iteration counts
    (acceptance.cpp:175-205) on the `paper1d` preset.

Extensions over the reference (each marked "EXTENSION"):
  * `gmres(..., restart=m)` — restarted GMRES(m), BASELINE.json asks for GMRES(50);
  * `add_gaussian_noise` — BASELINE.json's i.i.d. Gaussian relative-L2 noise;
  * `BlockTriangularPreconditioner(..., solver="pcg")` — the substituted
    per-block solve for 2D configurations whose dense factors do not fit.
"""
from __future__ import annotations

import dataclasses
import math
import time
from typing import Callable, List, Optional, Sequence

import os

import numpy as np
import scipy.fft as _sfft
import scipy.linalg as sla

# Threads for the oracle's batched FFTs (scipy.fft / pocketfft; the arithmetic does not depend on
# the thread count).  The reference's FFTW plans are single-threaded (fft.cpp:47-50): set
# FI_ORACLE_WORKERS=1 for a reference-faithful 1-core timing.
FFT_WORKERS = int(os.environ.get("FI_ORACLE_WORKERS", "0")) or (os.cpu_count() or 1)
_POOL = None


def _sub_scaled(w: np.ndarray, v: np.ndarray, h: float, tmp: np.ndarray) -> None:
    """w -= h * v as two separately rounded elementwise passes (multiply, then subtract: the
    arithmetic of krylov.cpp:130).  Long vectors are cut into FFT_WORKERS slices handled by host
    threads (numpy releases the GIL); every element sees the same two operations, so the result does
    not depend on the thread count."""
    global _POOL
    n = w.size
    if FFT_WORKERS == 1 or n < (1 << 22):
        np.multiply(v, h, out=tmp)
        np.subtract(w, tmp, out=w)
        return
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(FFT_WORKERS)
    step = -(-n // FFT_WORKERS)

    def part(a):
        b = min(n, a + step)
        np.multiply(v[a:b], h, out=tmp[a:b])
        np.subtract(w[a:b], tmp[a:b], out=w[a:b])

    list(_POOL.map(part, range(0, n, step)))

# --------------------------------------------------------------------------- errors
# errors.hpp:9-43


class DimensionError(ValueError):
    pass


class ResourceLimitError(RuntimeError):
    pass


class SingularBlockError(RuntimeError):
    def __init__(self, what: str, time_index: int):
        super().__init__(what)
        self.time_index = time_index


class EigensolverError(RuntimeError):
    pass


class ConfigError(RuntimeError):
    pass


# --------------------------------------------------------------------------- numerics
# numerics.cpp:20-35 — Lanczos g=7, 9-term (Godfrey) coefficients
_LANCZOS_G = 7.0
_LANCZOS_P = (
    0.99999999999980993,
    676.5203681218851,
    -1259.1392167224028,
    771.32342877765313,
    -176.61502916214059,
    12.507343278686905,
    -0.13857109526572012,
    9.9843695780195716e-6,
    1.5056327351493116e-7,
)
_SQRT_TWO_PI = 2.5066282746310002


def _lanczos_gamma(x: float) -> float:
    # numerics.cpp:37-53
    if x < 0.5:
        return _lanczos_gamma(x + 1.0) / x
    z = x - 1.0
    s = _LANCZOS_P[0]
    for k in range(1, 9):
        s += _LANCZOS_P[k] / (z + k)
    t = z + _LANCZOS_G + 0.5
    if x < 140.0:
        return _SQRT_TWO_PI * math.pow(t, z + 0.5) * math.exp(-t) * s
    return _SQRT_TWO_PI * math.exp((z + 0.5) * math.log(t) - t) * s


def gamma_fn(x: float) -> float:
    """numerics.cpp:57-61."""
    if not (x > 0.0):
        raise ValueError(f"gamma_fn requires x > 0, got {x}")
    return _lanczos_gamma(float(x))


@dataclasses.dataclass
class FractionalOrders:
    """numerics.cpp:10-16."""

    beta: float
    omega: float

    def __post_init__(self):
        if not (0.0 < self.beta < 1.0):
            raise ValueError(f"time order beta must lie in (0,1), got {self.beta}")
        if not (1.0 < self.omega < 2.0):
            raise ValueError(f"space order omega must lie in (1,2), got {self.omega}")


@dataclasses.dataclass
class L1Weights:
    b: np.ndarray
    e: np.ndarray


def l1_weights(beta: float, S: int) -> L1Weights:
    """numerics.cpp:63-80: b_m=(m+1)^{1-beta}-m^{1-beta}, e_0=b_0, e_m=b_m-b_{m-1}."""
    if not (0.0 < beta < 1.0):
        raise ValueError(f"l1_weights requires beta in (0,1), got {beta}")
    if S < 1:
        raise ValueError(f"l1_weights requires S >= 1, got {S}")
    p = 1.0 - beta
    b = np.array([math.pow(m + 1.0, p) - math.pow(float(m), p) for m in range(S)])
    e = np.empty(S)
    e[0] = b[0]
    e[1:] = b[1:] - b[:-1]
    return L1Weights(b, e)


@dataclasses.dataclass
class TimeGrid:
    S: int
    T: float
    dt: float
    eta: float


def time_grid(beta: float, S: int, T: float) -> TimeGrid:
    """numerics.cpp:82-96: dt=T/S, eta=dt^beta*Gamma(2-beta)."""
    if not (0.0 < beta < 1.0):
        raise ValueError(f"time_grid requires beta in (0,1), got {beta}")
    if S < 1:
        raise ValueError(f"time_grid requires S >= 1, got {S}")
    if not (T > 0.0):
        raise ValueError(f"time_grid requires T > 0, got {T}")
    dt = T / S
    return TimeGrid(S, T, dt, math.pow(dt, beta) * gamma_fn(2.0 - beta))


# --------------------------------------------------------------------------- grid / symbol
class SpaceGrid:
    """symbol.cpp:16-57 (h=(hi-lo)/(n+1), nodes lo+j*h, last direction fastest)."""

    def __init__(self, n: Sequence[int], lo: Sequence[float], hi: Sequence[float]):
        self.n = [int(v) for v in n]
        self.d = len(self.n)
        self.box_lo = [float(v) for v in lo]
        self.box_hi = [float(v) for v in hi]
        if self.d < 1:
            raise ValueError("SpaceGrid requires at least one direction")
        if len(self.box_lo) != self.d or len(self.box_hi) != self.d:
            raise DimensionError("SpaceGrid: box bounds must match the number of directions")
        for i in range(self.d):
            if self.n[i] < 1:
                raise ValueError("SpaceGrid requires n_i >= 1")
            if not (self.box_hi[i] > self.box_lo[i]):
                raise ValueError("SpaceGrid requires box_hi > box_lo in every direction")
        self.h = (self.box_hi[0] - self.box_lo[0]) / (self.n[0] + 1)
        for i in range(1, self.d):
            hi_ = (self.box_hi[i] - self.box_lo[i]) / (self.n[i] + 1)
            if abs(hi_ - self.h) > 1e-12 * abs(self.h):
                raise ValueError("SpaceGrid: mesh width must be common to all directions")

    def total(self) -> int:
        t = 1
        for v in self.n:
            t *= v
        return t

    def node(self, direction: int, j: int) -> float:
        return self.box_lo[direction] + j * self.h

    def nodes(self) -> np.ndarray:
        """(N, d) array, lexicographic multi-index order, last direction fastest."""
        axes = [self.box_lo[i] + np.arange(1, self.n[i] + 1, dtype=np.float64) * self.h for i in range(self.d)]
        mesh = np.meshgrid(*axes, indexing="ij")
        return np.stack([m.reshape(-1) for m in mesh], axis=1)


class SymbolCoefficients:
    """symbol.cpp:59-77: full d-level tensor over l_i=-(n_i-1)..(n_i-1), lexicographic."""

    def __init__(self, omega: float, n: Sequence[int], coeffs: np.ndarray):
        self.omega = omega
        self.n = [int(v) for v in n]
        self.d = len(self.n)
        self.coeffs = np.asarray(coeffs, dtype=np.float64)

    def tensor_size(self) -> int:
        t = 1
        for v in self.n:
            t *= 2 * v - 1
        return t

    def tensor(self) -> np.ndarray:
        return self.coeffs.reshape([2 * v - 1 for v in self.n])

    def at(self, l) -> float:
        if np.isscalar(l):
            l = [int(l)]
        if len(l) != self.d:
            raise DimensionError("SymbolCoefficients::at: multi-index has wrong dimension")
        idx = 0
        for i in range(self.d):
            ni, li = self.n[i], int(l[i])
            if li <= -ni or li >= ni:
                raise DimensionError("SymbolCoefficients::at: index out of range")
            idx = idx * (2 * ni - 1) + (li + ni - 1)
        return float(self.coeffs[idx])


def _check_omega(omega: float):
    if not (0.0 < omega <= 2.0):
        raise ValueError(f"symbol coefficients require omega in (0,2], got {omega}")


def symbol_coeffs_1d(omega: float, n: int) -> SymbolCoefficients:
    """symbol.cpp:88-110: a_0=Gamma(w+1)/Gamma(w/2+1)^2, a_{l+1}=(1-(w+1)/(w/2+l+1)) a_l."""
    _check_omega(omega)
    if n < 1:
        raise ValueError("symbol_coeffs_1d requires n >= 1")
    a = [0.0] * n
    g1 = gamma_fn(omega / 2.0 + 1.0)
    a[0] = gamma_fn(omega + 1.0) / (g1 * g1)
    for l in range(n - 1):
        a[l + 1] = (1.0 - (omega + 1.0) / (omega / 2.0 + l + 1.0)) * a[l]
    a = np.array(a)
    coeffs = np.concatenate([a[:0:-1], a])  # index l+n-1 holds a_|l|
    return SymbolCoefficients(omega, [n], coeffs)


def symbol_coeffs_md(omega: float, n: Sequence[int], sample_cap: int = 1 << 26) -> SymbolCoefficients:
    """symbol.cpp:112-191: rectangle-rule DFT of g(theta)=(sum 4 sin^2(theta_i/2))^{w/2}.

    Sampling extent M_i = max(4 n_i, 1024) for d>=2, max(4n, 131072) for d=1.
    """
    _check_omega(omega)
    n = [int(v) for v in n]
    d = len(n)
    if d < 1:
        raise ValueError("symbol_coeffs_md requires at least one direction")
    if any(v < 1 for v in n):
        raise ValueError("symbol_coeffs_md requires n_i >= 1")
    M = []
    total = 1
    for i in range(d):
        base = 131072 if d == 1 else 1024
        M.append(max(4 * n[i], base))
        total *= M[-1]
        if total > sample_cap:
            raise ResourceLimitError(
                f"symbol_coeffs_md: sample tensor of {total} points exceeds cap {sample_cap}")
    # symbol.cpp:142-160 — per-direction 4 sin^2(pi k / M_i), summed, raised to omega/2
    acc = np.zeros(M, dtype=np.float64)
    for i in range(d):
        s = np.sin(math.pi * np.arange(M[i], dtype=np.float64) / M[i])
        shape = [1] * d
        shape[i] = M[i]
        acc = acc + (4.0 * s * s).reshape(shape)
    samples = np.power(acc, omega / 2.0)
    X = np.fft.fftn(samples.astype(np.complex128))
    # symbol.cpp:165-189 — a_l ~ Re X_l / prod M_i; negative l wraps to M_i - |l_i|
    idx = [np.array([(l if l >= 0 else M[i] + l) for l in range(-(n[i] - 1), n[i])]) for i in range(d)]
    sub = X.real[np.ix_(*idx)] * (1.0 / float(total))
    return SymbolCoefficients(omega, n, sub.reshape(-1))


# --------------------------------------------------------------------------- Toeplitz operator
class ToeplitzOperator:
    """toeplitz.cpp:20-143: multilevel symmetric Toeplitz B via a 2n_i circulant embedding."""

    kDefaultDenseCap = 4096

    def __init__(self, grid: SpaceGrid, sym: SymbolCoefficients):
        if sym.d != grid.d or sym.n != grid.n:
            raise DimensionError("ToeplitzOperator: symbol tensor does not match the grid")
        self.grid = grid
        self.sym = sym
        self.dim = grid.total()
        self.embed = [2 * v for v in grid.n]
        # toeplitz.cpp:30-57 — k_i<n_i -> l_i=k_i, k_i==n_i gap (0), k_i>n_i -> l_i=k_i-2n_i
        T = sym.tensor()
        col = np.zeros(self.embed)
        src = []
        dst = []
        for i, ni in enumerate(grid.n):
            k = np.arange(2 * ni)
            valid = k != ni
            l = np.where(k < ni, k, k - 2 * ni)
            dst.append(k[valid])
            src.append(l[valid] + ni - 1)
        col[np.ix_(*dst)] = T[np.ix_(*src)]
        self.spectrum = np.fft.rfftn(col)  # real, even column -> spectrum of the circulant

    def apply(self, x: np.ndarray) -> np.ndarray:
        """toeplitz.cpp:75-114. Accepts (..., N) batches; returns B x for each."""
        x = np.asarray(x, dtype=np.float64)
        if x.shape[-1] != self.dim:
            raise DimensionError(
                f"ToeplitzOperator::apply: vector length {x.shape[-1]} does not match operator dimension {self.dim}")
        batch = x.shape[:-1]
        d = self.grid.d
        xs = x.reshape(batch + tuple(self.grid.n))
        axes = tuple(range(len(batch), len(batch) + d))
        X = _sfft.rfftn(xs, s=self.embed, axes=axes, workers=FFT_WORKERS)
        y = _sfft.irfftn(X * self.spectrum, s=self.embed, axes=axes, workers=FFT_WORKERS)
        sl = (Ellipsis,) + tuple(slice(0, v) for v in self.grid.n)
        return np.ascontiguousarray(y[sl]).reshape(batch + (self.dim,))

    def dense(self, cap: int = kDefaultDenseCap) -> np.ndarray:
        """toeplitz.cpp:116-143: entry (r,c) = a_{m_r - m_c} in lexicographic multi-index order."""
        if self.dim > cap:
            raise ResourceLimitError(f"ToeplitzOperator::dense: dimension {self.dim} exceeds cap {cap}")
        T = self.sym.tensor()
        mi = np.stack(np.unravel_index(np.arange(self.dim), self.grid.n), axis=1)  # (N,d)
        idx = []
        for i, ni in enumerate(self.grid.n):
            idx.append(mi[:, i][:, None] - mi[:, i][None, :] + ni - 1)
        return T[tuple(idx)]


# --------------------------------------------------------------------------- problem / system
SpaceTimeField = Callable[[np.ndarray, float], np.ndarray]  # (nodes (N,d), t) -> (N,)
TimeField = Callable[[float], float]


@dataclasses.dataclass
class ProblemSpec:
    """system.hpp:26-38."""

    orders: FractionalOrders
    sgrid: SpaceGrid
    tgrid: TimeGrid
    gamma1: SpaceTimeField
    gamma2: SpaceTimeField
    q: TimeField
    rho: np.ndarray
    f_true: np.ndarray
    lam: float = 5e-3
    noise_eps: float = 0.0
    preset: str = "custom"


def make_problem(preset: str, beta: float, omega: float, n: Sequence[int], S: int, lam: float,
                 noise_eps: float) -> ProblemSpec:
    """system.cpp:31-78 (presets 'paper1d' and 'constant' on (0,pi)^d, T=1)."""
    d = len(n)
    grid = SpaceGrid(n, [0.0] * d, [math.pi] * d)
    if preset == "paper1d":
        if d != 1:
            raise ConfigError("preset 'paper1d' is one-dimensional")
        g1 = lambda X, t: t * np.exp(X[:, 0])
        g2 = lambda X, t: t * t * X[:, 0]
        q = lambda t: t * t
        f = lambda X: X[:, 0] * np.sin(X[:, 0])
    elif preset == "constant":
        g1 = lambda X, t: np.ones(X.shape[0])
        g2 = lambda X, t: np.ones(X.shape[0])
        q = lambda t: 1.0
        f = lambda X: X.sum(axis=1) * np.sin(X.sum(axis=1))
    else:
        raise ConfigError(f"unknown preset '{preset}' (expected 'paper1d' or 'constant')")
    N = grid.total()
    spec = ProblemSpec(FractionalOrders(beta, omega), grid, time_grid(beta, S, 1.0), g1, g2, q,
                       np.zeros(N), f(grid.nodes()), lam, noise_eps, preset)
    if not (lam > 0.0):
        raise ValueError("regularization parameter lambda must be positive")
    if noise_eps < 0.0:
        raise ValueError("noise level eps must be nonnegative")
    return spec


def make_custom_problem(orders: FractionalOrders, sgrid: SpaceGrid, S: int, T: float, gamma1, gamma2, q,
                        rho, f_true, lam: float, noise_eps: float) -> ProblemSpec:
    """system.cpp:80-102."""
    N = sgrid.total()
    rho = np.asarray(rho, dtype=np.float64)
    f_true = np.asarray(f_true, dtype=np.float64)
    if rho.size != N or f_true.size != N:
        raise DimensionError("make_custom_problem: rho/f_true must have length N(n)")
    if not (lam > 0.0):
        raise ValueError("regularization parameter lambda must be positive")
    if noise_eps < 0.0:
        raise ValueError("noise level eps must be nonnegative")
    return ProblemSpec(orders, sgrid, time_grid(orders.beta, S, T), gamma1, gamma2, q, rho, f_true, lam,
                       noise_eps, "custom")


@dataclasses.dataclass
class CoefficientDiagonals:
    D1: np.ndarray  # (S, N), row s-1 = level s
    D2: np.ndarray


def sample_fields(spec: ProblemSpec) -> CoefficientDiagonals:
    """system.cpp:104-119: D_k(s-1, j) = gamma_k(x_j, t_s), t_s = s*dt."""
    N = spec.sgrid.total()
    S = spec.tgrid.S
    X = spec.sgrid.nodes()
    D1 = np.empty((S, N))
    D2 = np.empty((S, N))
    for s in range(1, S + 1):
        t = s * spec.tgrid.dt
        D1[s - 1] = np.broadcast_to(np.asarray(spec.gamma1(X, t), dtype=np.float64), (N,))
        D2[s - 1] = np.broadcast_to(np.asarray(spec.gamma2(X, t), dtype=np.float64), (N,))
    return CoefficientDiagonals(D1, D2)


class SystemOperator:
    """system.cpp:121-174: matrix-free all-at-once operator of dimension (S+1)N."""

    def __init__(self, spec: ProblemSpec, symbol: Optional[SymbolCoefficients] = None):
        self.spec = spec
        self.diags = sample_fields(spec)
        self.weights = l1_weights(spec.orders.beta, spec.tgrid.S)
        self.N = spec.sgrid.total()
        if symbol is None:
            symbol = (symbol_coeffs_1d(spec.orders.omega, spec.sgrid.n[0]) if spec.sgrid.d == 1
                      else symbol_coeffs_md(spec.orders.omega, spec.sgrid.n))
        self.laplacian = ToeplitzOperator(spec.sgrid, symbol)
        S = spec.tgrid.S
        self.q = np.array([float(spec.q(s * spec.tgrid.dt)) for s in range(1, S + 1)])
        for s in range(1, S + 1):
            if not (self.q[s - 1] > 0.0):
                raise ValueError(f"q(t) must be positive at every time level, violated at s = {s}")
        if spec.rho.size != self.N or spec.f_true.size != self.N:
            raise DimensionError("SystemOperator: rho/f_true must have length N(n)")
        hw = math.pow(spec.sgrid.h, spec.orders.omega)
        self.scale_space = spec.tgrid.eta / hw
        self.scale_reg = spec.lam / hw
        self._E = None

    @property
    def space_dim(self) -> int:
        return self.N

    @property
    def steps(self) -> int:
        return self.spec.tgrid.S

    @property
    def dim(self) -> int:
        return (self.steps + 1) * self.N

    def time_matrix(self) -> np.ndarray:
        """Lower-triangular Toeplitz E with E[s-1, m-1] = e_{s-m} (system.cpp:161-163)."""
        if self._E is None:
            S = self.steps
            e = self.weights.e
            k = np.arange(S)[:, None] - np.arange(S)[None, :]
            self._E = np.where(k >= 0, e[np.clip(k, 0, S - 1)], 0.0)
        return self._E

    def apply(self, y: np.ndarray) -> np.ndarray:
        """system.cpp:144-174.

        z^(s) = D1^(s) o sum_{m<=s} e_{s-m} y^(m) + (eta/h^w) D2^(s) o (B y^(s)) - eta q_s y^(S+1)
        z^(S+1) = y^(S) + (lambda/h^w) D2^(S) o (B y^(S+1))
        """
        y = np.asarray(y, dtype=np.float64)
        if y.shape[-1] != self.dim:
            raise DimensionError(
                f"SystemOperator::apply: vector length {y.shape[-1]} does not match operator dimension {self.dim}")
        S, N = self.steps, self.N
        Y = y[: S * N].reshape(S, N)
        f = y[S * N:]
        D1, D2 = self.diags.D1, self.diags.D2
        W = (self.time_matrix() @ Y) * D1
        BY = self.laplacian.apply(np.concatenate([Y, f[None, :]], axis=0))
        W += self.scale_space * D2 * BY[:S]
        W -= (self.spec.tgrid.eta * self.q)[:, None] * f[None, :]
        z = np.empty(self.dim)
        z[: S * N] = W.reshape(-1)
        z[S * N:] = Y[S - 1] + self.scale_reg * D2[S - 1] * BY[S]
        return z

    def apply_precond_matrix(self, y: np.ndarray) -> np.ndarray:
        """P y: the system matrix with the top-right block column (-eta q_s I) zeroed
        (spectra.cpp:34-36). Used for backward-error checks."""
        y = np.asarray(y, dtype=np.float64)
        S, N = self.steps, self.N
        z = self.apply(y)
        z[: S * N] += ((self.spec.tgrid.eta * self.q)[:, None] * y[S * N:][None, :]).reshape(-1)
        return z


@dataclasses.dataclass
class RhsVector:
    z: np.ndarray


def build_rhs(A: SystemOperator, mu_eps: np.ndarray) -> RhsVector:
    """system.cpp:176-190: z^(s) = b_{s-1} D1^(s) o rho, z^(S+1) = mu_eps."""
    N = A.space_dim
    mu_eps = np.asarray(mu_eps, dtype=np.float64)
    if mu_eps.size != N:
        raise DimensionError("build_rhs: mu_eps must have length N(n)")
    S = A.steps
    z = np.empty(A.dim)
    z[: S * N] = (A.weights.b[:, None] * (A.diags.D1 * A.spec.rho[None, :])).reshape(-1)
    z[S * N:] = mu_eps
    return RhsVector(z)


def _lu_checked(blk: np.ndarray, time_index: int, what: str):
    """krylov.cpp:14-20 / system.cpp:214-219: min|U_ii| <= 1e-14 max|U_ii| => singular."""
    lu, piv = sla.lu_factor(blk, check_finite=False)
    diag = np.abs(np.diag(lu))
    dmax = diag.max()
    if dmax == 0.0 or diag.min() <= 1e-14 * dmax:
        raise SingularBlockError(f"{what}: singular block at time level {time_index}", time_index)
    return lu, piv


@dataclasses.dataclass
class ForwardSolution:
    states: List[np.ndarray]
    mu: np.ndarray


def forward_solve(A: SystemOperator, f_source: Optional[np.ndarray] = None,
                  P: Optional["BlockTriangularPreconditioner"] = None) -> ForwardSolution:
    """system.cpp:192-224: block forward substitution with dense LU per level.

    EXTENSION: with P given, each level's block G_s (identical to P's time blocks) is solved by
    P.solve_block — the substituted solve for 2D blocks whose dense LU is infeasible."""
    N, S = A.space_dim, A.steps
    e, b = A.weights.e, A.weights.b
    eta = A.spec.tgrid.eta
    f = A.spec.f_true if f_source is None else f_source
    Bd = A.laplacian.dense(N) if P is None else None
    if P is not None and P.inner == "pcg":
        P.pcg.dropped = False
    states: List[np.ndarray] = []
    for s in range(1, S + 1):
        d1 = A.diags.D1[s - 1]
        d2 = A.diags.D2[s - 1]
        rhs = b[s - 1] * (d1 * A.spec.rho) + eta * A.q[s - 1] * f
        for m in range(1, s):
            rhs = rhs - e[s - m] * (d1 * states[m - 1])
        if P is not None:
            states.append(P.solve_block(s, rhs, [states[s - 1 - k] for k in range(1, min(WARM_ORDER, s - 1) + 1)]))
            continue
        blk = A.scale_space * d2[:, None] * Bd
        blk[np.diag_indices(N)] += e[0] * d1
        lu = _lu_checked(blk, s, "forward_solve")
        states.append(sla.lu_solve(lu, rhs, check_finite=False))
    return ForwardSolution(states, states[-1])


def _splitmix64_at(seed: int, j: np.ndarray) -> np.ndarray:
    """system.cpp:231-236: SplitMix64 output j of the stream seeded at `seed` (uint64 wraparound)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (j.astype(np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _unit_open(z: np.ndarray) -> np.ndarray:
    # system.cpp:246-247: top 53 bits, centred into (0,1)
    return ((z >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def add_noise(mu: np.ndarray, eps: float, seed: int) -> np.ndarray:
    """system.cpp:240-251: mu_j + eps*(2u_j-1), u_j from SplitMix64 at index j (additive uniform)."""
    if eps < 0.0:
        raise ValueError("add_noise requires eps >= 0")
    mu = np.asarray(mu, dtype=np.float64)
    u = _unit_open(_splitmix64_at(seed, np.arange(mu.size, dtype=np.uint64)))
    return mu + eps * (2.0 * u - 1.0)


def gaussian_stream(n: int, seed: int) -> np.ndarray:
    """EXTENSION (BASELINE.json configs): i.i.d. N(0,1) from SplitMix64-at-index + Box-Muller.

    delta_{2p} = r cos(2 pi u2), delta_{2p+1} = r sin(2 pi u2), r = sqrt(-2 ln u1),
    u1 = U(stream index 2p), u2 = U(stream index 2p+1).
    """
    npair = (n + 1) // 2
    u1 = _unit_open(_splitmix64_at(seed, 2 * np.arange(npair, dtype=np.uint64)))
    u2 = _unit_open(_splitmix64_at(seed, 2 * np.arange(npair, dtype=np.uint64) + np.uint64(1)))
    r = np.sqrt(-2.0 * np.log(u1))
    out = np.empty(2 * npair)
    out[0::2] = r * np.cos(2.0 * math.pi * u2)
    out[1::2] = r * np.sin(2.0 * math.pi * u2)
    return out[:n]


def add_gaussian_noise(mu: np.ndarray, rel_eps: float, seed: int) -> np.ndarray:
    """EXTENSION: mu + rel_eps*||mu||*delta/||delta|| so ||mu_eps - mu||_2 = rel_eps ||mu||_2."""
    if rel_eps < 0.0:
        raise ValueError("add_gaussian_noise requires eps >= 0")
    mu = np.asarray(mu, dtype=np.float64)
    if rel_eps == 0.0:
        return mu.copy()
    delta = gaussian_stream(mu.size, seed)
    return mu + (rel_eps * np.linalg.norm(mu) / np.linalg.norm(delta)) * delta


def extract_reconstruction(y: np.ndarray, space_dim: int) -> np.ndarray:
    """system.cpp:253-257."""
    if y.size % space_dim != 0 or y.size < 2 * space_dim:
        raise DimensionError("extract_reconstruction: vector is not a stacked block vector")
    return y[-space_dim:].copy()


def relative_error(truth: np.ndarray, approx: np.ndarray) -> float:
    """system.cpp:259-263."""
    if truth.size != approx.size:
        raise DimensionError("relative_error: size mismatch")
    return float(np.linalg.norm(truth - approx) / np.linalg.norm(truth))


# --------------------------------------------------------------------------- dense assembly
SYSTEM_A, PRECONDITIONER_P, FORWARD_AHAT = "SystemA", "PreconditionerP", "ForwardAhat"


def assemble_dense_system(A: SystemOperator, kind: str = SYSTEM_A, cap: int = 4096) -> np.ndarray:
    """spectra.cpp:14-45 (verification oracle only)."""
    N, S = A.space_dim, A.steps
    dim = S * N if kind == FORWARD_AHAT else (S + 1) * N
    if dim > cap:
        raise ResourceLimitError(f"assemble_dense_system: dimension {dim} exceeds cap {cap}")
    Bd = A.laplacian.dense(cap)
    e = A.weights.e
    M = np.zeros((dim, dim))
    di = np.arange(N)
    for s in range(1, S + 1):
        d1 = A.diags.D1[s - 1]
        d2 = A.diags.D2[s - 1]
        r = (s - 1) * N
        M[r:r + N, r:r + N] = A.scale_space * d2[:, None] * Bd
        M[r + di, r + di] += e[0] * d1
        for m in range(1, s):
            M[r + di, (m - 1) * N + di] = e[s - m] * d1
        if kind == SYSTEM_A:
            M[r + di, S * N + di] = -A.spec.tgrid.eta * A.q[s - 1]
    if kind != FORWARD_AHAT:
        r = S * N
        M[r + di, (S - 1) * N + di] = 1.0
        M[r:r + N, r:r + N] = A.scale_reg * A.diags.D2[S - 1][:, None] * Bd
    return M


# --------------------------------------------------------------------------- preconditioner
class BlockTriangularPreconditioner:
    """krylov.cpp:24-70: S+1 dense diagonal blocks, PartialPivLU, block forward substitution.

    G_s = (eta/h^w) diag(D2^(s)) B + e_0 diag(D1^(s)),  G_f = (lambda/h^w) diag(D2^(S)) B.
    `cache=False` refactors each block on every apply (config 1's 68.8 GB of factors do not
    fit in host RAM here); the arithmetic is identical.
    """

    kDefaultBlockCap = 4096

    def __init__(self, A: SystemOperator, block_cap: int = kDefaultBlockCap, cache: bool = True,
                 inner: str = "auto", tol: float = 1e-14, maxit: int = 200):
        """inner="lu": the reference (dense PartialPivLU per block; ResourceLimitError above the cap).
        inner="pcg": EXTENSION, the substituted per-block solve of SURVEY 7.3 #1 (tau-preconditioned
        CG on the SPD form, identical to the device's).  inner="auto": "lu" unless the problem is 2D
        and N exceeds the cap, where the reference cannot run at all (config 2-4)."""
        self.A = A
        self.N = A.space_dim
        self.S = A.steps
        if inner == "auto":
            inner = "pcg" if (A.spec.sgrid.d == 2 and self.N > block_cap) else "lu"
        self.inner = inner
        if inner == "pcg":
            self.pcg = TauPCG(A, tol, maxit)
            return
        if self.N > block_cap:
            raise ResourceLimitError(
                f"BlockTriangularPreconditioner: block dimension {self.N} exceeds cap {block_cap}")
        self.Bd = A.laplacian.dense(block_cap)
        self.cache = cache
        self.factors = []
        # build and pivot-check every block (krylov.cpp:33-45)
        for s in range(1, self.S + 2):
            lu = _lu_checked(self.block(s), s, "precond_build")
            if cache:
                self.factors.append(lu)

    @property
    def dim(self) -> int:
        return (self.S + 1) * self.N

    def block(self, s: int) -> np.ndarray:
        A = self.A
        if s <= self.S:
            blk = A.scale_space * A.diags.D2[s - 1][:, None] * self.Bd
            blk[np.diag_indices(self.N)] += A.weights.e[0] * A.diags.D1[s - 1]
            return blk
        return A.scale_reg * A.diags.D2[self.S - 1][:, None] * self.Bd

    def _factor(self, s: int):
        if self.cache:
            return self.factors[s - 1]
        return _lu_checked(self.block(s), s, "precond_build")

    def solve_block(self, s: int, rhs: np.ndarray, prev: Optional[Sequence[np.ndarray]] = None) -> np.ndarray:
        """prev: the solutions of the preceding time levels, latest first (tau-PCG only: their
        constant / linear / quadratic extrapolation is the initial guess, as on the device)."""
        if self.inner == "pcg":
            x0 = None
            if prev and s <= self.S and self.pcg.warm and not self.pcg.dropped:
                # extrapolation through the previous levels (latest first), summed in j order as on the
                # device: x0 = sum_j w_j y_(s-j), w from TauPCG.warm_weights
                w = self.pcg.warm_weights(len(prev), s)
                x0 = np.zeros_like(prev[0])
                for j in range(1, len(w) + 1):
                    x0 = x0 + w[j - 1] * prev[j - 1]
            return self.pcg.solve(s, rhs, x0)
        return sla.lu_solve(self._factor(s), rhs, check_finite=False)

    def apply(self, z: np.ndarray) -> np.ndarray:
        """krylov.cpp:48-70."""
        z = np.asarray(z, dtype=np.float64)
        if z.size != self.dim:
            raise DimensionError(
                f"precond_apply: vector length {z.size} does not match preconditioner dimension {self.dim}")
        N, S = self.N, self.S
        e = self.A.weights.e
        y = np.empty(self.dim)
        Y = y[: S * N].reshape(S, N)
        if self.inner == "pcg":
            self.pcg.dropped = False
            self.pcg.rho = [math.inf] * 4
        for s in range(1, S + 1):
            rhs = z[(s - 1) * N: s * N].copy()
            if s > 1:
                acc = e[s - 1:0:-1] @ Y[: s - 1]  # sum_{m<s} e_{s-m} y^(m)
                rhs -= self.A.diags.D1[s - 1] * acc
            Y[s - 1] = self.solve_block(s, rhs, [Y[s - 1 - k] for k in range(1, min(LS_WINDOW, s - 1) + 1)])
        rhs = z[S * N:] - Y[S - 1]
        y[S * N:] = self.solve_block(S + 1, rhs)
        return y


WARM_ORDER = 6  # previous levels in the tau-PCG initial-guess extrapolation (the device's kWarmOrder)
LS_WINDOW = 10  # previous levels of the least-squares extrapolation (the device's kLsWindow)
FLOOR_THETA = 1.0  # stop at theta * u * ||M|| ||x||: the rounding floor of the residual (the device's kFloorTheta)
_U = 2.0 ** -53


def _hmean(delta: np.ndarray) -> float:
    """The tau preconditioner's shift: the harmonic mean of delta (0 if delta vanishes somewhere), summed in
    index order as on the device's host setup.  Where delta varies strongly (config 4: 80x) the arithmetic mean
    over-shifts the low frequencies, the only ones where delta matters against c g(theta)."""
    if delta.size == 0 or not np.all(delta > 0.0):
        return 0.0
    return float(delta.size / np.sum(1.0 / delta))


def _ls_weights(m: int, d: int):
    """Weights w_j of y_(s-j), j = 1..m: the value at 0 of the degree-d least-squares polynomial through
    the points (-j, y_(s-j)).  Exact rational arithmetic, rounded once (the device's kLsCoef literals)."""
    from fractions import Fraction
    V = [[Fraction(-(j + 1)) ** k for k in range(d + 1)] for j in range(m)]
    G = [[sum(V[j][a] * V[j][b] for j in range(m)) for b in range(d + 1)] for a in range(d + 1)]
    # solve G c = e0 by Gauss-Jordan in rationals; w_j = sum_k V[j][k] c_k
    n = d + 1
    aug = [G[i][:] + [Fraction(1 if i == 0 else 0)] for i in range(n)]
    for i in range(n):
        piv = next(r for r in range(i, n) if aug[r][i] != 0)
        aug[i], aug[piv] = aug[piv], aug[i]
        aug[i] = [v / aug[i][i] for v in aug[i]]
        for r in range(n):
            if r != i and aug[r][i] != 0:
                aug[r] = [a - aug[r][i] * b for a, b in zip(aug[r], aug[i])]
    c = [aug[i][n] for i in range(n)]
    return [float(sum(V[j][k] * c[k] for k in range(n))) for j in range(m)]


LS_COEF = _ls_weights(LS_WINDOW, WARM_ORDER - 1)


class TauPCG:
    """EXTENSION: exact-to-tolerance per-block solve for blocks too large to factor.

    G_s y = r with G_s = D2_s (c M0 + diag(delta_s)), c = eta/h^w, delta = e0 D1/D2 (time levels);
    G_f = cr D2_S B (f-block, delta = 0).  Solved as M y = r / D2 with M = c B + diag(delta) SPD, by
    CG preconditioned with the tau matrix  tau^{-1} = S diag(1/(c g(theta_j) + hmean(delta))) S (harmonic mean),
    S the orthonormal DST-I, g the symbol (sum_i 4 sin^2(theta_i/2))^{w/2} at theta_j = j pi/(n+1).
    x0 = 0 or the extrapolation through the previous levels (warm_weights); stop when
    ||r_k|| <= max(tol ||b||, u ||M|| ||x_k||) (2-norms; solve()) or after maxit steps.  The device
    (precond_iter.cu) runs the same recurrence in the same order of operations.
    """

    def __init__(self, A: SystemOperator, tol: float = 1e-14, maxit: int = 200):
        import scipy.fft as sf
        self.sf = sf
        self.A = A
        self.tol, self.maxit = tol, maxit
        self.n = list(A.spec.sgrid.n)
        th = [np.arange(1, ni + 1) * math.pi / (ni + 1) for ni in self.n]
        acc = 0.0
        for i, t in enumerate(th):
            shape = [1] * len(self.n)
            shape[i] = self.n[i]
            acc = acc + (4.0 * np.sin(t / 2.0) ** 2).reshape(shape)
        self.g = np.power(acc, A.spec.orders.omega / 2.0)
        self.iterations = []
        self.warm = True  # extrapolated initial guesses for the time levels (the device's FI_TAU_WARM=1)
        self.dropped = False  # set when a guess was worse than zero: no guesses for the rest of the apply
        # the latest guess of each kind (0 polynomial, 1 least squares): ||r|| / (u ||M|| ||x||)
        self.rho = [math.inf] * 4
        self.kind = 0
        self.theta = FLOOR_THETA  # 0: stop on tol ||b|| alone (the device's FI_TAU_FLOOR=0)
        self.lswin = LS_WINDOW  # 0: polynomial extrapolation on every level (the device's FI_TAU_LSWIN=0)
        S, N = A.steps, A.space_dim
        e0 = A.weights.e[0]
        for s in range(1, S + 1):
            d2 = A.diags.D2[s - 1]
            if np.all(d2 == 0.0):
                continue
            if np.any(d2 == 0.0) or np.any(A.diags.D1[s - 1] / d2 < 0.0):
                raise ValueError("TauPCG needs gamma2 != 0 and gamma1/gamma2 >= 0 per level")
        if np.any(A.diags.D2[S - 1] == 0.0):
            raise SingularBlockError(f"precond_build: singular block at time level {S + 1}", S + 1)

    def warm_weights(self, nprev: int, level: int = 0):
        """Weights of the previous nprev (<= LS_WINDOW) levels' solutions, latest first, in the initial
        guess of time level `level` (1-based).  Four kinds of guess compete:
          0  the polynomial through the last min(nprev, 6) levels, w_j = (-1)^(j+1) C(k, j)   ||w||_2 = 30.4
          1  the polynomial through the last 8 levels                                           ||w||_2 = 113
          2  the polynomial through the last 10 levels                                          ||w||_2 = 430
          3  the degree-5 least-squares polynomial through the last 10 levels                  ||w||_2 = 6.1
        A guess's residual is the extrapolation's truncation error (large near the solution's weak
        singularity at t = 0, falling like level^-order) plus the rounding floor u ||M|| ||x|| of the
        previous solutions' residuals amplified by ||w||_2: high orders win on the early levels, low
        noise on the late ones, and where the change happens depends on beta and the input.  So the kind
        is chosen by measurement: on the levels e, e+1, e+2, e+3 with e = 2^j or 3 2^(j-1) >= 16 each kind
        is tried once (kind = level - e); on every other level the kind whose latest guess was closest to
        the floor (rho, set in solve()) is used.  Until the first trial (level < 16) kind 0 is used."""
        self.kind = 0
        if self.lswin and nprev >= LS_WINDOW:
            hb = 1 << (level.bit_length() - 1)
            e = hb + hb // 2 if level >= hb + hb // 2 else hb
            if level >= 16 and level - e < 4:
                self.kind = level - e
            else:
                self.kind = min(range(4), key=lambda k: self.rho[k])  # ties: the lowest kind
        if self.kind == 3:
            return LS_COEF
        k = min(nprev, (WARM_ORDER, 8, 10)[self.kind])
        return [float((-1) ** (j + 1) * math.comb(k, j)) for j in range(1, k + 1)]

    def _tau_inv(self, r, lam):
        R = r.reshape(self.n)
        X = self.sf.dstn(R, type=1, norm="ortho")
        X /= lam
        return self.sf.idstn(X, type=1, norm="ortho").reshape(-1)

    def solve(self, s: int, rhs: np.ndarray, x0: Optional[np.ndarray] = None) -> np.ndarray:
        """x0 (time levels, EXTENSION identical to the device): an initial guess.  A pre-step sets
        x = x0, r = b - M x0; the level is done if r passes the stopping test, and a guess with
        ||r|| > ||b|| is dropped (x = 0, r = b) before the tau-preconditioned iteration starts.

        Stopping test: ||r|| <= max(tol ||b||, theta u ||M|| ||x||), ||M|| taken as the largest tau
        eigenvalue c max g + hmean(delta), u = 2^-53.  The second term is the rounding floor of a residual
        b - M x evaluated in double: below it the recursive r keeps falling while the true residual does
        not (measured on config 4: true residual 1.7e-13 ||b|| = 1.0 u ||M|| ||x|| at every level)."""
        A = self.A
        S = A.steps
        e0 = A.weights.e[0]
        if s <= S:
            d1, d2 = A.diags.D1[s - 1], A.diags.D2[s - 1]
            if np.all(d2 == 0.0):
                return rhs / (e0 * d1)
            c, delta = A.scale_space, e0 * d1 / d2
        else:
            d2 = A.diags.D2[S - 1]
            c, delta = A.scale_reg, np.zeros(A.space_dim)
        b = rhs / d2
        lam = c * self.g + _hmean(delta)
        normM = float(lam.max())
        floor = self.theta * _U * normM
        M = lambda v: c * A.laplacian.apply(v) + delta * v
        x = np.zeros_like(b)
        bn = np.linalg.norm(b)
        if bn == 0.0:
            self.iterations.append(0)
            return x
        r = b.copy()
        if s <= S and x0 is None:
            self.rho = [math.inf] * 4
        if x0 is not None and s <= S:
            x = x0.copy()
            r = b - M(x0)
            self.rho[self.kind] = float(np.linalg.norm(r)) / (_U * normM * float(np.linalg.norm(x)))
            if np.linalg.norm(r) <= max(self.tol * bn, floor * np.linalg.norm(x)):
                self.iterations.append(0)
                return x
            if float(r @ r) > float(b @ b):
                x = np.zeros_like(b)
                r = b.copy()
                self.dropped = True
        z = self._tau_inv(r, lam)
        p = z.copy()
        rz = float(r @ z)
        it = 0
        for it in range(1, self.maxit + 1):
            Ap = M(p)
            alpha = rz / float(p @ Ap)
            x += alpha * p
            r -= alpha * Ap
            if np.linalg.norm(r) <= max(self.tol * bn, floor * np.linalg.norm(x)):
                break
            z = self._tau_inv(r, lam)
            rz_new = float(r @ z)
            p = z + (rz_new / rz) * p
            rz = rz_new
        self.iterations.append(it)
        return x


# --------------------------------------------------------------------------- GMRES
@dataclasses.dataclass
class SolveReport:
    """krylov.hpp:17-24."""

    iterations: int = 0
    residual_history: List[float] = dataclasses.field(default_factory=list)
    converged: bool = False
    breakdown: bool = False
    wall_time_seconds: float = 0.0
    final_true_residual: float = 0.0


def gmres(apply_A, apply_M_inv, b: np.ndarray, tol: float = 1e-8, maxit: int = 0, restart: int = 0,
          x0: Optional[np.ndarray] = None):
    """krylov.cpp:72-209: left-preconditioned GMRES, MGS + one conditional reorthogonalisation,
    Givens-rotation least squares, convergence on the preconditioned relative residual.

    EXTENSION restart=m>0: GMRES(m).  Each cycle of at most m Arnoldi steps is the reference
    loop verbatim (history entry |g_{k+1}|/||M^-1 b|| per step, same breakdown tests); at the
    end of a cycle x is updated and, if no stop condition fired and iterations < maxit,
    r = M^-1(b - A x) is recomputed and the next cycle starts from it.  If that recomputed
    residual already satisfies ||r||/||M^-1 b|| <= tol the solve is declared converged
    without a new history entry.  `iterations` counts Arnoldi steps over all cycles and
    len(residual_history) == iterations + 1 always.  restart=0 is the reference's full GMRES.
    """
    t_start = time.perf_counter()
    if not (tol > 0.0):
        raise ValueError("gmres requires tol > 0")
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    maxit = maxit if maxit > 0 else n
    prec = (lambda v: apply_M_inv(v)) if apply_M_inv is not None else (lambda v: v)
    report = SolveReport()
    x = np.array(x0, dtype=np.float64) if x0 is not None else np.zeros(n)

    pb = prec(b)
    bnorm = float(np.linalg.norm(pb))
    if bnorm == 0.0:
        report.converged = True
        report.residual_history = [0.0]
        report.final_true_residual = 0.0
        report.wall_time_seconds = time.perf_counter() - t_start
        return np.zeros(n), report

    r0 = prec(b - apply_A(x)) if x0 is not None else pb
    beta = float(np.linalg.norm(r0))
    report.residual_history.append(beta / bnorm)
    if beta / bnorm <= tol:
        report.converged = True
        report.final_true_residual = float(np.linalg.norm(b - apply_A(x)) / np.linalg.norm(b))
        report.wall_time_seconds = time.perf_counter() - t_start
        return x, report

    cycle = restart if restart > 0 else maxit
    breakdown_tol = 1e-14 * bnorm
    iters = 0
    converged = breakdown = False
    while True:
        V = [r0 / beta]
        hcols: List[List[float]] = []
        g = [beta]
        cs: List[float] = []
        sn: List[float] = []
        kc = 0  # completed Arnoldi steps in this cycle
        stop = False
        for k in range(min(cycle, maxit - iters)):
            w = prec(apply_A(V[k]))
            pre_norm = float(np.linalg.norm(w))
            h = [0.0] * (k + 2)
            tmp = np.empty_like(w)  # w -= h V[i] without temporaries (same arithmetic)
            for i in range(k + 1):  # modified Gram-Schmidt (krylov.cpp:127-132)
                hik = float(V[i] @ w)
                h[i] += hik
                _sub_scaled(w, V[i], hik, tmp)
            if np.linalg.norm(w) < pre_norm * 0.70710678118654752:  # krylov.cpp:134-140
                for i in range(k + 1):
                    corr = float(V[i] @ w)
                    h[i] += corr
                    _sub_scaled(w, V[i], corr, tmp)
            del tmp
            hnext = float(np.linalg.norm(w))
            h[k + 1] = hnext
            if hnext > breakdown_tol:
                V.append(w / hnext)
            col_scale = max(abs(v) for v in h)
            for i in range(k):  # krylov.cpp:150-156
                t = cs[i] * h[i] + sn[i] * h[i + 1]
                h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1]
                h[i] = t
            denom = math.hypot(h[k], h[k + 1])
            if denom <= 1e-14 * col_scale or denom == 0.0:  # krylov.cpp:157-164
                breakdown = True
                stop = True
                break
            cs.append(h[k] / denom)
            sn.append(h[k + 1] / denom)
            h[k] = denom
            h.pop()
            hcols.append(h)
            g.append(-sn[-1] * g[-1])
            g[k] *= cs[-1]
            relres = abs(g[-1]) / bnorm
            report.residual_history.append(relres)
            iters += 1
            kc = k + 1
            if relres <= tol:
                converged = True
                stop = True
                break
            if hnext <= breakdown_tol:
                breakdown = True
                stop = True
                break
        if kc > 0:  # krylov.cpp:188-200
            yk = [0.0] * kc
            for i in range(kc - 1, -1, -1):
                acc = g[i]
                for j in range(i + 1, kc):
                    acc -= hcols[j][i] * yk[j]
                yk[i] = acc / hcols[i][i]
            for j in range(kc):
                x = x + yk[j] * V[j]
        if stop or iters >= maxit:
            break
        r0 = prec(b - apply_A(x))
        beta = float(np.linalg.norm(r0))
        if beta / bnorm <= tol or beta == 0.0:
            converged = True
            break

    report.iterations = iters
    report.converged = converged or (breakdown and report.residual_history[-1] <= tol)
    report.breakdown = breakdown and not report.converged
    report.final_true_residual = float(np.linalg.norm(b - apply_A(x)) / np.linalg.norm(b))
    report.wall_time_seconds = time.perf_counter() - t_start
    return x, report
