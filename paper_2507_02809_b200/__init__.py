"""B200-native preconditioned GMRES for the all-at-once system of arXiv 2507.02809.

The compute path is libfracinv_b200.so (hand-written sm_100a CUDA behind the C-ABI in
include/fracinv_b200.h); `fracinv` mirrors the reference library's API on top of it.
"""
from . import fracinv  # noqa: F401  (loads the shared library; fails loudly if it is missing)
from .fracinv import *  # noqa: F401,F403
