"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol declared
in include/fracinv_b200.h, its host setup numerics match the oracle / golden tables, and
device entry points fail loudly (status code + message) when no CUDA device is present."""
import ctypes
import math
import os
from collections import defaultdict

import numpy as np
import pytest

from helpers import load_csv
from oracle import fracinv_oracle as O
from paper_2507_02809_b200 import _lib
from paper_2507_02809_b200 import fracinv as F

lib = _lib.lib


def test_library_exports_every_declared_symbol():
    declared = _lib.declared_symbols()
    assert len(declared) >= 30
    raw = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared if not hasattr(raw, s)]
    assert not missing, missing
    # and the binding covers them all
    assert set(declared) <= set(_lib._SIGS), set(declared) - set(_lib._SIGS)


def test_gamma_and_l1_and_time_grid_match_oracle():
    for x, expected in load_csv("gamma_reference.csv"):
        assert abs(F.gamma_fn(x) - expected) <= 1e-13 * expected
        assert F.gamma_fn(x) == O.gamma_fn(x)
    with pytest.raises(ValueError):
        F.gamma_fn(0.0)
    for beta in (0.1, 0.5, 0.9):
        w, wo = F.l1_weights(beta, 512), O.l1_weights(beta, 512)
        assert np.array_equal(w.b, wo.b) and np.array_equal(w.e, wo.e)
        g, go = F.time_grid(beta, 64, 1.0), O.time_grid(beta, 64, 1.0)
        assert g.eta == go.eta and g.dt == go.dt
    with pytest.raises(ValueError):
        F.l1_weights(1.0, 4)
    with pytest.raises(ValueError):
        F.time_grid(0.5, 0, 1.0)


def test_symbol_coefficients_match_golden_and_oracle():
    table = defaultdict(list)
    for omega, l, a in load_csv("symbol_coeffs_reference.csv"):
        table[omega].append(a)
    for omega, a in table.items():
        a = np.array(a)
        sym = F.symbol_coeffs_1d(omega, a.size)
        got = sym.coeffs[a.size - 1:]
        tol = np.where(np.arange(a.size) < 256, 5e-13, 2e-12)
        assert np.all(np.abs(got - a) <= tol * np.abs(a))
        assert np.array_equal(sym.coeffs, O.symbol_coeffs_1d(omega, a.size).coeffs)
    # multilevel rectangle rule: same quadrature as the reference, different summation order
    for n in ([16], [4, 4], [5, 2], [12, 9]):
        f, o = F.symbol_coeffs_md(1.9, n), O.symbol_coeffs_md(1.9, n)
        assert np.max(np.abs(f.coeffs - o.coeffs)) <= 5e-14 * np.max(np.abs(o.coeffs))
    with pytest.raises(F.ResourceLimitError):
        F.symbol_coeffs_md(1.5, [5000, 5000])


def test_noise_generators_match_oracle():
    mu = np.sin(np.linspace(0, 3, 777))
    assert np.array_equal(F.add_noise(mu, 0.01, 5), O.add_noise(mu, 0.01, 5))
    g, go = F.add_gaussian_noise(mu, 0.01, 1000), O.add_gaussian_noise(mu, 0.01, 1000)
    assert np.max(np.abs(g - go)) <= 1e-15 * np.max(np.abs(mu)) * 10
    assert abs(np.linalg.norm(g - mu) - 0.01 * np.linalg.norm(mu)) <= 1e-14 * np.linalg.norm(mu)


def test_space_grid_and_presets_mirror_reference():
    g = F.SpaceGrid([2, 3], [0.0, 0.0], [1.0, 4.0 / 3.0])
    assert np.allclose(g.nodes(), O.SpaceGrid([2, 3], [0.0, 0.0], [1.0, 4.0 / 3.0]).nodes(), rtol=0, atol=0)
    with pytest.raises(ValueError):
        F.SpaceGrid([4, 4], [0.0, 0.0], [1.0, 2.0])
    with pytest.raises(F.ConfigError):
        F.make_problem("nope", 0.5, 1.5, [8], 4, 1e-2, 0.0)
    spec, speco = F.make_problem("paper1d", 0.5, 1.5, [15], 4, 5e-3, 0.01), O.make_problem(
        "paper1d", 0.5, 1.5, [15], 4, 5e-3, 0.01)
    d, do = F.sample_fields(spec), O.sample_fields(speco)
    assert np.array_equal(d.D1, do.D1) and np.array_equal(d.D2, do.D2)


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="GPU present: the no-device path is not reachable")
def test_device_calls_fail_loudly_without_gpu():
    with pytest.raises(F.CudaError):
        F.Context(0)
    h = ctypes.c_void_p()
    rc = lib.fi_ctx_create(0, ctypes.byref(h))
    assert rc == _lib.FI_E_CUDA and _lib.last_error()
