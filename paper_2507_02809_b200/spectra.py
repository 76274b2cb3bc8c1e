"""Spectra of the all-at-once system on the GPU (verification, Table 1 / Fig. 1).

Mirrors spectra.hpp / spectra.cpp:14-90:

* `assemble_dense_system(A, kind, cap)` — the dense block matrix, assembled by a CUDA kernel from the
  operator's own data (`fi_assemble_dense`), bit-for-bit the reference realisation;
* `eigenvalues_dense`, `eigenvalues_preconditioned`, `condition_number_2`,
  `condition_number_preconditioned`, `spectral_summary` — the same quantities, computed on the
  device by torch.linalg (cuSOLVER / MAGMA library routines: this is a verification path, not the
  solve path).

Errors follow the reference: ResourceLimitError above the dense cap, DimensionError for mismatched
sizes, EigensolverError if the eigensolver fails.
"""
from __future__ import annotations

import dataclasses
from typing import List

import numpy as np

from . import fracinv as F

SYSTEM_A, PRECONDITIONER_P, FORWARD_AHAT = "SystemA", "PreconditionerP", "ForwardAhat"
_KIND = {SYSTEM_A: 0, PRECONDITIONER_P: 1, FORWARD_AHAT: 2}


class EigensolverError(RuntimeError):
    """errors.hpp: EigensolverError."""


def _torch():
    import torch
    return torch


def assemble_dense_system(A: F.SystemOperator, kind: str = SYSTEM_A, cap: int = 4096):
    """spectra.cpp:14-45 on the device: a (dim, dim) float64 CUDA tensor (row-major)."""
    torch = _torch()
    if kind not in _KIND:
        raise ValueError(f"unknown dense kind '{kind}'")
    N, S = A.space_dim(), A.steps()
    dim = S * N if kind == FORWARD_AHAT else (S + 1) * N
    if dim > cap:
        raise F.ResourceLimitError(f"assemble_dense_system: dimension {dim} exceeds cap {cap}")
    M = torch.empty((dim, dim), dtype=torch.float64, device=f"cuda:{A.ctx.device}")
    torch.cuda.synchronize()
    F._check(F.lib.fi_assemble_dense(A.handle, _KIND[kind], int(cap), M.data_ptr()))
    A.ctx.synchronize()
    return M


def _as_cuda(M):
    torch = _torch()
    if isinstance(M, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(M, dtype=np.float64)).cuda()
    return M


def eigenvalues_dense(M) -> np.ndarray:
    """spectra.cpp:47-53: all eigenvalues (complex)."""
    torch = _torch()
    try:
        ev = torch.linalg.eigvals(_as_cuda(M))
    except RuntimeError as ex:  # the library's non-convergence
        raise EigensolverError(f"dense eigensolver did not converge: {ex}")
    return ev.cpu().numpy()


def eigenvalues_preconditioned(P, A) -> np.ndarray:
    """spectra.cpp:55-61: eigenvalues of P^{-1} A (LU solve)."""
    torch = _torch()
    P, A = _as_cuda(P), _as_cuda(A)
    if P.shape != A.shape:
        raise F.DimensionError("eigenvalues_preconditioned: P and A sizes differ")
    return eigenvalues_dense(torch.linalg.solve(P, A))


def condition_number_2(M) -> float:
    """spectra.cpp:63-70: sigma_max / sigma_min; infinity for a singular matrix."""
    torch = _torch()
    sv = torch.linalg.svdvals(_as_cuda(M))
    smin = float(sv[-1])
    return float("inf") if smin == 0.0 else float(sv[0]) / smin


def condition_number_preconditioned(P, A) -> float:
    """spectra.cpp:72-77."""
    torch = _torch()
    P, A = _as_cuda(P), _as_cuda(A)
    if P.shape != A.shape:
        raise F.DimensionError("condition_number_preconditioned: P and A sizes differ")
    return condition_number_2(torch.linalg.solve(P, A))


@dataclasses.dataclass
class SpectralSummary:
    """spectra.hpp: eigenvalues, 2-norm condition number, cluster statistics around 1."""

    eigenvalues: List[complex]
    cond_2: float
    cluster_count: int
    outlier_count: int


def spectral_summary(M, cluster_tol: float = 1e-6) -> SpectralSummary:
    """spectra.cpp:79-90."""
    ev = eigenvalues_dense(M)
    near = np.abs(ev - 1.0) <= cluster_tol
    return SpectralSummary([complex(v) for v in ev], condition_number_2(M), int(near.sum()), int((~near).sum()))
