"""Generating tensor of the 2D fractional Laplacian on the device:
fi_symbol_coeffs_md_dev must be bit-for-bit the host restatement (symbol.cpp:112-191), which the
CPU tests pin against the reference's own symmetry and quadrature checks."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
F = pytest.importorskip("paper_2507_02809_b200.fracinv")


@pytest.mark.parametrize("omega,n", [(1.5, [4, 3]), (1.9, [6, 5]), (1.1, [16, 16]), (1.2, [127, 127]),
                                     (1.5, [255, 255]), (1.9, [300, 10]), (2.0, [1, 7])])
def test_device_symbol_is_bitwise_host(omega, n):
    host = F.symbol_coeffs_md(omega, n)
    dev = F.symbol_coeffs_md(omega, n, ctx=F.default_context())
    assert dev.coeffs.shape == host.coeffs.shape
    assert np.array_equal(dev.coeffs.view(np.uint64), host.coeffs.view(np.uint64))


def test_device_symbol_errors():
    ctx = F.default_context()
    with pytest.raises(F.ResourceLimitError):
        F.symbol_coeffs_md(1.5, [255, 255], sample_cap=1 << 19, ctx=ctx)
    with pytest.raises(ValueError):
        F.symbol_coeffs_md(2.5, [8, 8], ctx=ctx)
