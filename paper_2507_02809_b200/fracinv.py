"""Reference-facing API of the B200 path, mirroring the fracinv C++ library.

Names, argument meaning and error behaviour follow /root/reference/proj/include/fracinv
(system.hpp, krylov.hpp, numerics.hpp, symbol.hpp, errors.hpp) so code written against the
reference reads the same:

    A = SystemOperator(spec)                         # system.hpp:72-104
    P = BlockTriangularPreconditioner(A)             # krylov.hpp:33-50
    mu = forward_solve(A).mu                         # system.hpp:107-119
    rhs = build_rhs(A, add_noise(mu, eps, seed))     # system.hpp:101, 121-125
    y, rep = gmres(A, P, rhs.z, GmresOptions(tol, maxit, restart))   # krylov.hpp:52-69

Every compute call goes through the C-ABI of libfracinv_b200.so (include/fracinv_b200.h):
the operator apply, the preconditioner setup/apply, the forward solve and GMRES run on the
GPU.  Host work here is problem assembly only (sampling the user's coefficient fields on the
grid, as system.cpp:104-119 does).  Vectors may be numpy arrays (host) or torch CUDA
tensors (device, zero-copy).
"""
from __future__ import annotations

import atexit
import ctypes
import dataclasses
import math
from typing import Callable, List, Optional, Sequence

import numpy as np

from ._lib import (FI_E_CONFIG, FI_E_CUDA, FI_E_DIM, FI_E_DOMAIN, FI_E_NOCONV, FI_E_RESOURCE, FI_E_SINGULAR, LINOP,
                   GmresOpts,
                   GmresReport, SystemDesc, c_double_p, last_error, lib)

# --------------------------------------------------------------------------- errors (errors.hpp:9-43)


class DimensionError(ValueError):
    pass


class ResourceLimitError(RuntimeError):
    pass


class SingularBlockError(RuntimeError):
    def __init__(self, what: str, time_index: int):
        super().__init__(what)
        self.time_index = time_index

    def __reduce__(self):
        return (SingularBlockError, (str(self), self.time_index))


class ConfigError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class NoConvergenceError(RuntimeError):
    """A tau-PCG block solve stopped at maxit above its tolerance (FI_E_NOCONV, EXTENSION)."""


_SHUTDOWN = [False]


@atexit.register
def _mark_shutdown():
    # handles are not released once the interpreter exits: the CUDA runtime may already be gone
    _SHUTDOWN[0] = True


def _check(rc: int):
    if rc == 0:
        return
    msg = last_error()
    if rc == FI_E_DIM:
        raise DimensionError(msg)
    if rc == FI_E_RESOURCE:
        raise ResourceLimitError(msg)
    if rc == FI_E_SINGULAR:
        raise SingularBlockError(msg, lib.fi_last_error_time_index())
    if rc == FI_E_DOMAIN:
        raise ValueError(msg)  # std::domain_error
    if rc == FI_E_CONFIG:
        raise ConfigError(msg)
    if rc == FI_E_NOCONV:
        raise NoConvergenceError(msg)
    raise CudaError(msg or f"fracinv_b200 error {rc}")


def _dp(a: np.ndarray):
    return a.ctypes.data_as(c_double_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# --------------------------------------------------------------------------- context
class Context:
    """One CUDA stream on one device (fi_ctx)."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        _check(lib.fi_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.device = device

    @property
    def stream(self) -> int:
        return lib.fi_ctx_stream(self.handle) or 0

    def synchronize(self):
        _check(lib.fi_ctx_synchronize(self.handle))

    @property
    def kernel_launches(self) -> int:
        return int(lib.fi_ctx_kernel_launches(self.handle))

    def after_torch(self):
        """Order this context's stream after the work torch has queued on its current stream (inputs a
        pending torch kernel still writes, outputs whose memory the caching allocator recycles)."""
        import torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        if getattr(self, "_ext", None) is None:
            self._ext = torch.cuda.ExternalStream(self.stream, device=torch.device("cuda", self.device))
        self._ext.wait_event(ev)

    def __del__(self, _shutdown=_SHUTDOWN, _lib=lib):
        if getattr(self, "handle", None) and not _shutdown[0]:
            _lib.fi_ctx_destroy(self.handle)
            self.handle = None


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# --------------------------------------------------------------------------- numerics
def gamma_fn(x: float) -> float:
    """numerics.hpp:33 (Lanczos, g=7)."""
    out = ctypes.c_double()
    _check(lib.fi_gamma(float(x), ctypes.byref(out)))
    return out.value


@dataclasses.dataclass
class FractionalOrders:
    """numerics.hpp:9-16."""

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
    """numerics.hpp:36."""
    b = np.empty(max(S, 1))
    e = np.empty(max(S, 1))
    _check(lib.fi_l1_weights(float(beta), int(S), _dp(b), _dp(e)))
    return L1Weights(b, e)


@dataclasses.dataclass
class TimeGrid:
    S: int
    T: float
    dt: float
    eta: float


def time_grid(beta: float, S: int, T: float) -> TimeGrid:
    """numerics.hpp:39."""
    dt, eta = ctypes.c_double(), ctypes.c_double()
    _check(lib.fi_time_grid(float(beta), int(S), float(T), ctypes.byref(dt), ctypes.byref(eta)))
    return TimeGrid(int(S), float(T), dt.value, eta.value)


class SpaceGrid:
    """symbol.hpp:13-31: common mesh width h=(hi-lo)/(n+1), nodes lo+j*h, last direction fastest."""

    def __init__(self, n: Sequence[int], lo: Sequence[float], hi: Sequence[float]):
        self.n = [int(v) for v in n]
        self.d = len(self.n)
        self.box_lo = [float(v) for v in lo]
        self.box_hi = [float(v) for v in hi]
        if self.d < 1:
            raise ValueError("SpaceGrid requires at least one direction")
        if len(self.box_lo) != self.d or len(self.box_hi) != self.d:
            raise DimensionError("SpaceGrid: box bounds must match the number of directions")
        if self.d > 2:
            raise ValueError("the B200 path supports d in {1, 2}")
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
        return int(np.prod(self.n))

    def node(self, direction: int, j: int) -> float:
        return self.box_lo[direction] + j * self.h

    def nodes(self) -> np.ndarray:
        axes = [self.box_lo[i] + np.arange(1, self.n[i] + 1, dtype=np.float64) * self.h for i in range(self.d)]
        mesh = np.meshgrid(*axes, indexing="ij")
        return np.stack([m.reshape(-1) for m in mesh], axis=1)


class SymbolCoefficients:
    """symbol.hpp:37-49."""

    def __init__(self, omega: float, n: Sequence[int], coeffs: np.ndarray):
        self.omega = omega
        self.n = [int(v) for v in n]
        self.d = len(self.n)
        self.coeffs = _f64(coeffs)

    def tensor_size(self) -> int:
        return int(np.prod([2 * v - 1 for v in self.n]))

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


def symbol_coeffs_1d(omega: float, n: int) -> SymbolCoefficients:
    """symbol.hpp:51-56."""
    out = np.empty(max(2 * n - 1, 1))
    _check(lib.fi_symbol_coeffs_1d(float(omega), int(n), _dp(out)))
    return SymbolCoefficients(omega, [n], out)


def symbol_coeffs_md(omega: float, n: Sequence[int], sample_cap: int = 1 << 26,
                     ctx: Optional["Context"] = None) -> SymbolCoefficients:
    """symbol.hpp:58-64.  ctx given (2D): the cosine sums run on that context's device, bit-for-bit
    the host result (fi_symbol_coeffs_md_dev)."""
    n = [int(v) for v in n]
    if any(v < 1 for v in n):
        raise ValueError("symbol_coeffs_md requires n_i >= 1")
    out = np.empty(int(np.prod([2 * v - 1 for v in n])))
    narr = (ctypes.c_int * len(n))(*n)
    if ctx is not None:
        _check(lib.fi_symbol_coeffs_md_dev(ctx.handle, float(omega), len(n), narr, int(sample_cap), _dp(out)))
    else:
        _check(lib.fi_symbol_coeffs_md(float(omega), len(n), narr, int(sample_cap), _dp(out)))
    return SymbolCoefficients(omega, n, out)


# --------------------------------------------------------------------------- problem assembly
@dataclasses.dataclass
class ProblemSpec:
    """system.hpp:26-38.  gamma1/gamma2: (nodes (N,d) array, t) -> (N,); q: t -> float."""

    orders: FractionalOrders
    sgrid: SpaceGrid
    tgrid: TimeGrid
    gamma1: Callable
    gamma2: Callable
    q: Callable
    rho: np.ndarray
    f_true: np.ndarray
    lam: float = 5e-3
    noise_eps: float = 0.0
    preset: str = "custom"


def make_problem(preset: str, beta: float, omega: float, n: Sequence[int], S: int, lam: float,
                 noise_eps: float) -> ProblemSpec:
    """system.hpp:41-49 (presets 'paper1d' and 'constant', Omega=(0,pi)^d, T=1)."""
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
    spec = ProblemSpec(FractionalOrders(beta, omega), grid, time_grid(beta, S, 1.0), g1, g2, q,
                       np.zeros(grid.total()), f(grid.nodes()), lam, noise_eps, preset)
    if not (lam > 0.0):
        raise ValueError("regularization parameter lambda must be positive")
    if noise_eps < 0.0:
        raise ValueError("noise level eps must be nonnegative")
    return spec


def make_custom_problem(orders: FractionalOrders, sgrid: SpaceGrid, S: int, T: float, gamma1, gamma2, q, rho,
                        f_true, lam: float, noise_eps: float) -> ProblemSpec:
    """system.hpp:51-55."""
    N = sgrid.total()
    rho, f_true = _f64(rho), _f64(f_true)
    if rho.size != N or f_true.size != N:
        raise DimensionError("make_custom_problem: rho/f_true must have length N(n)")
    if not (lam > 0.0):
        raise ValueError("regularization parameter lambda must be positive")
    if noise_eps < 0.0:
        raise ValueError("noise level eps must be nonnegative")
    return ProblemSpec(orders, sgrid, time_grid(orders.beta, S, T), gamma1, gamma2, q, rho, f_true, lam, noise_eps,
                       "custom")


@dataclasses.dataclass
class CoefficientDiagonals:
    D1: np.ndarray
    D2: np.ndarray


def sample_fields(spec: ProblemSpec) -> CoefficientDiagonals:
    """system.cpp:104-119: row s-1 holds gamma_k(x_j, t_s), t_s = s*dt."""
    N, S = spec.sgrid.total(), spec.tgrid.S
    X = spec.sgrid.nodes()
    D1, D2 = np.empty((S, N)), np.empty((S, N))
    for s in range(1, S + 1):
        t = s * spec.tgrid.dt
        D1[s - 1] = np.broadcast_to(np.asarray(spec.gamma1(X, t), dtype=np.float64), (N,))
        D2[s - 1] = np.broadcast_to(np.asarray(spec.gamma2(X, t), dtype=np.float64), (N,))
    return CoefficientDiagonals(D1, D2)


def _is_cuda_tensor(v) -> bool:
    return type(v).__module__.startswith("torch") and getattr(v, "is_cuda", False)


def _device_ptr(v, n: int) -> int:
    import torch
    if v.dtype != torch.float64 or not v.is_contiguous() or v.numel() != n:
        raise DimensionError(f"expected a contiguous float64 CUDA tensor of length {n}")
    return v.data_ptr()


class SystemOperator:
    """system.hpp:72-104: device-resident all-at-once operator; apply() runs kernel K1."""

    def __init__(self, spec: ProblemSpec, ctx: Optional[Context] = None, symbol: Optional[SymbolCoefficients] = None):
        self.ctx = ctx or default_context()
        self.spec = spec
        self.N = spec.sgrid.total()
        self.S = spec.tgrid.S
        self.diags = sample_fields(spec)
        self.weights = l1_weights(spec.orders.beta, self.S)
        if symbol is None:
            symbol = (symbol_coeffs_1d(spec.orders.omega, spec.sgrid.n[0]) if spec.sgrid.d == 1
                      else symbol_coeffs_md(spec.orders.omega, spec.sgrid.n, ctx=self.ctx))
        self.symbol = symbol
        self.q = np.array([float(spec.q(s * spec.tgrid.dt)) for s in range(1, self.S + 1)])
        if spec.rho.size != self.N or spec.f_true.size != self.N:
            raise DimensionError("SystemOperator: rho/f_true must have length N(n)")
        hw = math.pow(spec.sgrid.h, spec.orders.omega)
        self.scale_space = spec.tgrid.eta / hw
        self.scale_reg = spec.lam / hw
        self._keep = [_f64(symbol.coeffs), _f64(self.weights.e), _f64(self.weights.b), _f64(self.q),
                      _f64(self.diags.D1), _f64(self.diags.D2)]
        desc = SystemDesc()
        desc.d = spec.sgrid.d
        desc.n[0] = spec.sgrid.n[0]
        desc.n[1] = spec.sgrid.n[1] if spec.sgrid.d == 2 else 0
        desc.S = self.S
        desc.h = spec.sgrid.h
        desc.eta = spec.tgrid.eta
        desc.scale_space = self.scale_space
        desc.scale_reg = self.scale_reg
        desc.omega = spec.orders.omega
        desc.gen, desc.e, desc.b, desc.q, desc.D1, desc.D2 = [_dp(a) for a in self._keep]
        h = ctypes.c_void_p()
        _check(lib.fi_system_create(self.ctx.handle, ctypes.byref(desc), ctypes.byref(h)))
        self.handle = h
        self._keep = None

    APPLY_MODES = {"auto": 0, "dmma": 1, "fft": 2}

    def set_apply_mode(self, mode: str):
        """Realisation of the operator apply (also A inside gmres): "dmma" = K1, the dense FP64 DMMA
        contraction K U with K generated per tile; "fft" = K1f, the reference's circulant-embedded FFT
        Toeplitz products (toeplitz.cpp:68-114) as batched 2D transforms (2D grids with n_i + 1 a power
        of two); "auto" (default) = fft where supported — fi_system_set_apply_mode."""
        _check(lib.fi_system_set_apply_mode(self.handle, self.APPLY_MODES[mode]))

    @property
    def apply_mode(self) -> str:
        """The realisation in use: "dmma" or "fft"."""
        return {1: "dmma", 2: "fft"}[lib.fi_system_get_apply_mode(self.handle)]

    def set_split_apply(self, on: bool):
        """Arnoldi steps of gmres(self, P, ...) compute P^{-1} A v as v + P^{-1}((A - P) v) (default, one
        sweep per step) or as K1 then P^{-1} (the reference's order) — fi_system_set_split_apply."""
        _check(lib.fi_system_set_split_apply(self.handle, 1 if on else 0))

    # reference accessors
    def space_dim(self) -> int:
        return self.N

    def steps(self) -> int:
        return self.S

    def dim(self) -> int:
        return (self.S + 1) * self.N

    def q_values(self) -> np.ndarray:
        return self.q

    def diagonals(self) -> CoefficientDiagonals:
        return self.diags

    def apply(self, y):
        """z = A y (system.cpp:144-174). numpy in -> numpy out; CUDA tensor in -> CUDA tensor out."""
        n = self.dim()
        if _is_cuda_tensor(y):
            import torch
            yp = _device_ptr(y, n)
            z = torch.empty_like(y)
            self.ctx.after_torch()
            _check(lib.fi_system_apply(self.handle, yp, z.data_ptr()))
            self.ctx.synchronize()
            return z
        y = _f64(y)
        if y.size != n:
            raise DimensionError(f"SystemOperator::apply: vector length {y.size} does not match operator dimension {n}")
        z = np.empty(n)
        _check(lib.fi_system_apply_host(self.handle, _dp(y), _dp(z)))
        return z

    __call__ = apply

    def __del__(self, _shutdown=_SHUTDOWN, _lib=lib):
        if getattr(self, "handle", None) and not _shutdown[0]:
            _lib.fi_system_destroy(self.handle)
            self.handle = None


class BlockTriangularPreconditioner:
    """krylov.hpp:33-50: per-level inverses built on the GPU; apply() runs kernel K2."""

    kDefaultBlockCap = 4096

    def __init__(self, A: SystemOperator, block_cap: int = kDefaultBlockCap, inner: str = "auto",
                 tol: float = 1e-14, maxit: int = 200):
        """inner="lu" (dense per-block solve, the reference; N > block_cap -> ResourceLimitError),
        "pcg" (EXTENSION: tau-preconditioned CG per block), or "auto" (dense up to
        the cap, tau-PCG above it for 2D — configs 2-4, which the reference cannot run)."""
        self.A = A
        mode = {"auto": -1, "lu": 0, "pcg": 1}[inner]
        if block_cap <= 0 and mode != 1:
            # krylov.cpp:27-29: N > block_cap throws (the C-ABI reads block_cap <= 0 as the default)
            raise ResourceLimitError(f"BlockTriangularPreconditioner: block dimension {A.N} exceeds cap {block_cap}")
        h = ctypes.c_void_p()
        _check(lib.fi_precond_create_ex(A.handle, int(block_cap), mode, float(tol), int(maxit), ctypes.byref(h)))
        self.handle = h

    @property
    def inner(self) -> str:
        return "pcg" if lib.fi_precond_inner(self.handle) == 1 else "lu"

    @property
    def form(self) -> str:
        """Storage of the block inverses: "tiles" (packed FP64/FP32), "hodlr" or "pcg" (none)."""
        return {0: "tiles", 1: "pcg", 2: "hodlr"}[lib.fi_precond_form(self.handle)]

    def dim(self) -> int:
        return self.A.dim()

    def device_bytes(self) -> int:
        return int(lib.fi_precond_bytes(self.handle))

    def build_check(self) -> dict:
        """The build's a-posteriori check of HODLR-compressed inverses (fi_precond_build_check)."""
        out = (ctypes.c_double * 2)()
        _check(lib.fi_precond_build_check(self.handle, out))
        return {"forward": out[0], "backward": out[1]}

    def stats(self, reset: bool = False) -> dict:
        """tau-PCG inner-solve counters since the last reset (fi_precond_stats; zeros for dense blocks)."""
        out = (ctypes.c_longlong * 4)()
        _check(lib.fi_precond_stats(self.handle, out, 1 if reset else 0))
        return {"cg_steps": int(out[0]), "nonconverged_blocks": int(out[1]), "max_steps_per_block": int(out[2]),
                "applies": int(out[3])}

    def set_refine(self, refine: bool):
        """Refinement sweep off (default: one FP64 sweep over the polished inverses, forward parity
        with LU solves) or on (an extra sweep; LU-grade residual as well)."""
        _check(lib.fi_precond_set_refine(self.handle, 1 if refine else 0))

    def apply(self, z):
        """y = P^{-1} z by forward block substitution (krylov.cpp:48-70)."""
        n = self.dim()
        if _is_cuda_tensor(z):
            import torch
            zp = _device_ptr(z, n)
            y = torch.empty_like(z)
            self.A.ctx.after_torch()
            _check(lib.fi_precond_apply(self.handle, zp, y.data_ptr()))
            self.A.ctx.synchronize()
            return y
        z = _f64(z)
        if z.size != n:
            raise DimensionError(f"precond_apply: vector length {z.size} does not match preconditioner dimension {n}")
        y = np.empty(n)
        _check(lib.fi_precond_apply_host(self.handle, _dp(z), _dp(y)))
        return y

    __call__ = apply

    def __del__(self, _shutdown=_SHUTDOWN, _lib=lib):
        if getattr(self, "handle", None) and not _shutdown[0]:
            _lib.fi_precond_destroy(self.handle)
            self.handle = None


@dataclasses.dataclass
class RhsVector:
    z: np.ndarray


def build_rhs(A: SystemOperator, mu_eps) -> RhsVector:
    """system.cpp:176-190."""
    mu_eps = _f64(mu_eps)
    if mu_eps.size != A.N:
        raise DimensionError("build_rhs: mu_eps must have length N(n)")
    z = np.empty(A.dim())
    _check(lib.fi_build_rhs(A.handle, _dp(_f64(A.spec.rho)), _dp(mu_eps), _dp(z)))
    return RhsVector(z)


@dataclasses.dataclass
class ForwardSolution:
    states: List[np.ndarray]
    mu: np.ndarray


def forward_solve(A: SystemOperator, P: Optional[BlockTriangularPreconditioner] = None) -> ForwardSolution:
    """system.cpp:192-224 on the device, through P's time-level inverses (built if P is None)."""
    states = np.empty((A.S, A.N))
    mu = np.empty(A.N)
    _check(lib.fi_forward_solve(A.handle, P.handle if P is not None else None, _dp(_f64(A.spec.rho)),
                                _dp(_f64(A.spec.f_true)), _dp(states), _dp(mu)))
    return ForwardSolution([states[s] for s in range(A.S)], mu)


def add_noise(mu, eps: float, seed: int) -> np.ndarray:
    """system.cpp:240-251 (additive uniform, SplitMix64 at index j)."""
    mu = _f64(mu)
    out = np.empty_like(mu)
    _check(lib.fi_add_noise(_dp(mu), mu.size, float(eps), int(seed), _dp(out)))
    return out


def add_gaussian_noise(mu, rel_eps: float, seed: int) -> np.ndarray:
    """EXTENSION (BASELINE.json): i.i.d. Gaussian noise scaled to rel_eps * ||mu||_2."""
    mu = _f64(mu)
    out = np.empty_like(mu)
    _check(lib.fi_add_gaussian_noise(_dp(mu), mu.size, float(rel_eps), int(seed), _dp(out)))
    return out


def extract_reconstruction(y, space_dim: int) -> np.ndarray:
    """system.cpp:253-257."""
    y = np.asarray(y)
    if y.size % space_dim != 0 or y.size < 2 * space_dim:
        raise DimensionError("extract_reconstruction: vector is not a stacked block vector")
    return y[-space_dim:].copy()


def relative_error(truth, approx) -> float:
    """system.cpp:259-263."""
    truth, approx = np.asarray(truth), np.asarray(approx)
    if truth.size != approx.size:
        raise DimensionError("relative_error: size mismatch")
    return float(np.linalg.norm(truth - approx) / np.linalg.norm(truth))


# --------------------------------------------------------------------------- GMRES
@dataclasses.dataclass
class GmresOptions:
    """krylov.hpp:54-57 + restart (EXTENSION; 0 = full GMRES, the reference)."""

    tol: float = 1e-8
    maxit: int = 0
    restart: int = 0


@dataclasses.dataclass
class SolveReport:
    """krylov.hpp:17-24."""

    iterations: int = 0
    residual_history: List[float] = dataclasses.field(default_factory=list)
    converged: bool = False
    breakdown: bool = False
    wall_time_seconds: float = 0.0
    final_true_residual: float = 0.0
    inner_nonconverged: int = 0  # EXTENSION: tau-PCG block solves that stopped at maxit above tol


def _report(rep: GmresReport, hist: np.ndarray) -> SolveReport:
    if rep.inner_nonconverged:
        import warnings
        warnings.warn(f"gmres: {rep.inner_nonconverged} tau-PCG block solve(s) stopped at maxit above tol; "
                      "the preconditioner was not applied exactly", RuntimeWarning, stacklevel=3)
    return SolveReport(rep.iterations, [float(v) for v in hist[: rep.history_len]], bool(rep.converged),
                       bool(rep.breakdown), rep.wall_time_seconds, rep.final_true_residual, rep.inner_nonconverged)


class _CAI:
    """Minimal __cuda_array_interface__ view of a device pointer (for LinearOp callbacks)."""

    def __init__(self, ptr: int, n: int, readonly: bool):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, readonly), "version": 2}


def _as_tensor(ptr: int, n: int):
    import torch
    return torch.as_tensor(_CAI(ptr, n, False), device="cuda")


def gmres(apply_A, apply_M_inv, b, opts: Optional[GmresOptions] = None, x0=None, **kw):
    """krylov.hpp:59-69: left-preconditioned GMRES, all iteration state on the device.

    apply_A / apply_M_inv: a SystemOperator / BlockTriangularPreconditioner (device path,
    fi_gmres), or generic callables y = op(x) on torch CUDA tensors (LinearOp, fi_gmres_op).
    apply_M_inv None = no preconditioning.  b (and x0): numpy (host) or torch CUDA tensors.
    """
    opts = opts or GmresOptions(**kw)
    o = GmresOpts(float(opts.tol), int(opts.maxit), int(opts.restart))
    rep = GmresReport()
    if isinstance(apply_A, SystemOperator) and (apply_M_inv is None or
                                                isinstance(apply_M_inv, BlockTriangularPreconditioner)):
        A = apply_A
        n = A.dim()
        cap = (opts.maxit if opts.maxit > 0 else min(n, 1 << 20)) + 1
        hist = np.zeros(cap)
        Ph = apply_M_inv.handle if apply_M_inv is not None else None
        if _is_cuda_tensor(b):
            import torch
            bp = _device_ptr(b, n)
            x0p = _device_ptr(x0, n) if x0 is not None else None
            x = torch.empty_like(b)
            A.ctx.after_torch()
            _check(lib.fi_gmres(A.handle, Ph, bp, x0p, x.data_ptr(), ctypes.byref(o), ctypes.byref(rep), _dp(hist),
                                cap))
            return x, _report(rep, hist)
        b = _f64(b)
        if b.size != n:
            raise DimensionError("gmres: right-hand side length does not match the operator")
        x = np.empty(n)
        x0a = _f64(x0) if x0 is not None else None
        _check(lib.fi_gmres_host(A.handle, Ph, _dp(b), _dp(x0a) if x0a is not None else None, _dp(x),
                                 ctypes.byref(o), ctypes.byref(rep), _dp(hist), cap))
        return x, _report(rep, hist)

    # generic LinearOp path
    import torch
    ctx = default_context()
    host = not _is_cuda_tensor(b)
    bt = torch.as_tensor(_f64(b)).cuda() if host else b.contiguous()
    n = bt.numel()
    x0t = None
    if x0 is not None:
        x0t = torch.as_tensor(_f64(x0)).cuda() if not _is_cuda_tensor(x0) else x0.contiguous()
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream)
    errors = []

    def wrap(op):
        def cb(user, xp, yp):
            try:
                with torch.cuda.stream(stream):
                    xt = _as_tensor(xp, n)
                    yt = _as_tensor(yp, n)
                    yt.copy_(op(xt))
                return 0
            except Exception as ex:  # surfaced after the call
                errors.append(ex)
                return 1
        return LINOP(cb)

    cbA = wrap(apply_A)
    cbM = wrap(apply_M_inv) if apply_M_inv is not None else ctypes.cast(None, LINOP)
    x = torch.empty_like(bt)
    cap = (opts.maxit if opts.maxit > 0 else n) + 1
    hist = np.zeros(cap)
    rc = lib.fi_gmres_op(ctx.handle, n, cbA, None, cbM, None, bt.data_ptr(),
                         x0t.data_ptr() if x0t is not None else None, x.data_ptr(), ctypes.byref(o),
                         ctypes.byref(rep), _dp(hist), cap)
    if errors:
        raise errors[0]
    _check(rc)
    return (x.cpu().numpy() if host else x), _report(rep, hist)
