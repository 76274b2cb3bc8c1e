"""ctypes binding of the C-ABI declared in include/fracinv_b200.h.

The shared library is the product; there is no Python or CPU fallback.  Importing this
module fails loudly when libfracinv_b200.so is missing.
"""
import ctypes
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FI_LIB_PATH") or os.path.join(PKG, "libfracinv_b200.so")  # FI_LIB_PATH: A/B builds
HEADER = os.path.join(os.path.dirname(PKG), "include", "fracinv_b200.h")

FI_OK, FI_E_DIM, FI_E_RESOURCE, FI_E_SINGULAR, FI_E_DOMAIN, FI_E_CUDA, FI_E_NOCONV, FI_E_CONFIG = range(8)

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int_p = ctypes.POINTER(ctypes.c_int)
c_void_p = ctypes.c_void_p


class SystemDesc(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int),
        ("n", ctypes.c_int * 2),
        ("S", ctypes.c_int),
        ("h", ctypes.c_double),
        ("eta", ctypes.c_double),
        ("scale_space", ctypes.c_double),
        ("scale_reg", ctypes.c_double),
        ("gen", c_double_p),
        ("e", c_double_p),
        ("b", c_double_p),
        ("q", c_double_p),
        ("D1", c_double_p),
        ("D2", c_double_p),
        ("omega", ctypes.c_double),
    ]


class GmresOpts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("maxit", ctypes.c_int), ("restart", ctypes.c_int)]


class GmresReport(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int),
        ("converged", ctypes.c_int),
        ("breakdown", ctypes.c_int),
        ("wall_time_seconds", ctypes.c_double),
        ("final_true_residual", ctypes.c_double),
        ("history_len", ctypes.c_int),
        ("inner_nonconverged", ctypes.c_int),
    ]


LINOP = ctypes.CFUNCTYPE(ctypes.c_int, c_void_p, c_void_p, c_void_p)

_SIGS = {
    "fi_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(c_void_p)]),
    "fi_ctx_destroy": (None, [c_void_p]),
    "fi_ctx_stream": (c_void_p, [c_void_p]),
    "fi_ctx_synchronize": (ctypes.c_int, [c_void_p]),
    "fi_last_error": (ctypes.c_char_p, []),
    "fi_last_error_time_index": (ctypes.c_int, []),
    "fi_ctx_kernel_launches": (ctypes.c_longlong, [c_void_p]),
    "fi_gamma": (ctypes.c_int, [ctypes.c_double, c_double_p]),
    "fi_l1_weights": (ctypes.c_int, [ctypes.c_double, ctypes.c_int, c_double_p, c_double_p]),
    "fi_time_grid": (ctypes.c_int, [ctypes.c_double, ctypes.c_int, ctypes.c_double, c_double_p, c_double_p]),
    "fi_symbol_coeffs_1d": (ctypes.c_int, [ctypes.c_double, ctypes.c_int, c_double_p]),
    "fi_symbol_coeffs_md": (ctypes.c_int, [ctypes.c_double, ctypes.c_int, c_int_p, ctypes.c_longlong, c_double_p]),
    "fi_mgs_round_timed": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "fi_mgs_step_timed": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]),
    "fi_assemble_dense": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p]),
    "fi_system_set_split_apply": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "fi_system_set_apply_mode": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "fi_system_get_apply_mode": (ctypes.c_int, [ctypes.c_void_p]),
    "fi_symbol_coeffs_md_dev": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int, c_int_p, ctypes.c_longlong,
                                               c_double_p]),
    "fi_add_gaussian_noise": (ctypes.c_int,
                              [c_double_p, ctypes.c_longlong, ctypes.c_double, ctypes.c_ulonglong, c_double_p]),
    "fi_add_noise": (ctypes.c_int, [c_double_p, ctypes.c_longlong, ctypes.c_double, ctypes.c_ulonglong, c_double_p]),
    "fi_system_create": (ctypes.c_int, [c_void_p, ctypes.POINTER(SystemDesc), ctypes.POINTER(c_void_p)]),
    "fi_system_destroy": (None, [c_void_p]),
    "fi_system_dim": (ctypes.c_longlong, [c_void_p]),
    "fi_system_space_dim": (ctypes.c_longlong, [c_void_p]),
    "fi_system_apply": (ctypes.c_int, [c_void_p, c_void_p, c_void_p]),
    "fi_system_apply_host": (ctypes.c_int, [c_void_p, c_double_p, c_double_p]),
    "fi_system_apply_timed": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, ctypes.c_int, c_double_p]),
    "fi_precond_create": (ctypes.c_int, [c_void_p, ctypes.c_longlong, ctypes.POINTER(c_void_p)]),
    "fi_precond_destroy": (None, [c_void_p]),
    "fi_precond_apply": (ctypes.c_int, [c_void_p, c_void_p, c_void_p]),
    "fi_precond_apply_host": (ctypes.c_int, [c_void_p, c_double_p, c_double_p]),
    "fi_precond_apply_timed": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, ctypes.c_int, c_double_p]),
    "fi_precond_bytes": (ctypes.c_longlong, [c_void_p]),
    "fi_precond_stats": (ctypes.c_int, [c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]),
    "fi_precond_build_check": (ctypes.c_int, [c_void_p, ctypes.POINTER(ctypes.c_double)]),
    "fi_precond_set_refine": (ctypes.c_int, [c_void_p, ctypes.c_int]),
    "fi_precond_create_ex": (ctypes.c_int, [c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                             ctypes.POINTER(c_void_p)]),
    "fi_precond_inner": (ctypes.c_int, [c_void_p]),
    "fi_precond_form": (ctypes.c_int, [c_void_p]),
    "fi_build_rhs": (ctypes.c_int, [c_void_p, c_double_p, c_double_p, c_double_p]),
    "fi_forward_solve": (ctypes.c_int, [c_void_p, c_void_p, c_double_p, c_double_p, c_double_p, c_double_p]),
    "fi_gmres": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, ctypes.POINTER(GmresOpts),
                                ctypes.POINTER(GmresReport), c_double_p, ctypes.c_int]),
    "fi_gmres_host": (ctypes.c_int, [c_void_p, c_void_p, c_double_p, c_double_p, c_double_p,
                                     ctypes.POINTER(GmresOpts), ctypes.POINTER(GmresReport), c_double_p,
                                     ctypes.c_int]),
    "fi_gmres_op": (ctypes.c_int, [c_void_p, ctypes.c_longlong, LINOP, c_void_p, LINOP, c_void_p, c_void_p,
                                   c_void_p, c_void_p, ctypes.POINTER(GmresOpts), ctypes.POINTER(GmresReport),
                                   c_double_p, ctypes.c_int]),
}


def declared_symbols():
    """Every `fi_*` function declared in include/fracinv_b200.h."""
    text = open(HEADER).read()
    decl = re.compile(r"^(?:int|void|long long|const char\s*\*|void\s*\*)\s*\*?\s*(fi_[a-z0-9_]+)\s*\(", re.M)
    return sorted(set(decl.findall(text)))


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        if os.environ.get("FI_LIB_PATH") and not hasattr(lib, name):
            continue  # an A/B build of an older ABI
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()


def last_error():
    msg = lib.fi_last_error()
    return msg.decode() if msg else ""
