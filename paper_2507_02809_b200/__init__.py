"""B200-native preconditioned GMRES for the all-at-once system of arXiv 2507.02809.

The compute path is libfracinv_b200.so (hand-written sm_100a CUDA behind the C-ABI in
include/fracinv_b200.h); `fracinv` mirrors the reference library's API on top of it.

The library is loaded on first use of the API (`from paper_2507_02809_b200 import fracinv`, or any
attribute of the package such as `paper_2507_02809_b200.SystemOperator`), and that load fails loudly
when the .so is missing.  Importing a pure-Python submodule (`paper_2507_02809_b200.configs`) does
not map the library, so the CPU reference arm of bench.py never loads the product.
"""
import importlib

__all__ = ["fracinv", "solve", "spectra", "configs"]


def __getattr__(name):
    if name in ("fracinv", "solve", "spectra", "configs", "_lib"):
        return importlib.import_module(f".{name}", __name__)
    fr = importlib.import_module(".fracinv", __name__)
    try:
        return getattr(fr, name)
    except AttributeError:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}") from None
