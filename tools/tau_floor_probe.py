"""Where does the tau-PCG block solve's residual stop falling?  (oracle only, CPU)

Runs the oracle's preconditioner substitution on the first nlev time levels of a BASELINE 2D config with the
previous stopping rule (recursive ||r|| <= 1e-14 ||b||) and prints, every 32 levels, the residual of the
extrapolated guess and of the final solution re-evaluated in 80-bit arithmetic (numpy longdouble through
scipy.fft) next to u ||M|| ||x|| / ||b||, the rounding floor the device and the oracle now stop at (DESIGN 4,
K5 stopping rule).   usage: python tools/tau_floor_probe.py [cfg=4] [nlev=320]"""
import math
import os
import sys

os.environ.setdefault("FI_ORACLE_WORKERS", "4")
import numpy as np
import scipy.fft as sf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import fracinv_oracle as O  # noqa: E402
from paper_2507_02809_b200.configs import baseline_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nlev = int(sys.argv[2]) if len(sys.argv) > 2 else 320
A = O.SystemOperator(baseline_problem(O, cfg))
pcg = O.BlockTriangularPreconditioner(A, inner="pcg").pcg
N, T = A.N, A.laplacian
g = np.load(os.path.join(ROOT, "tests", "golden", f"oracle_config{cfg}.npz"))["f"]
g = g / np.linalg.norm(g)
eta, e = A.spec.tgrid.eta, A.weights.e
n = T.grid.n
# the embedded generating tensor in long double (its float64 entries are exactly representable)
col = np.zeros(T.embed, dtype=np.longdouble)
src, dst = [], []
for ni in n:
    k = np.arange(2 * ni)
    dst.append(k[k != ni])
    src.append(np.where(k < ni, k, k - 2 * ni)[k != ni] + ni - 1)
col[np.ix_(*dst)] = T.sym.tensor().astype(np.longdouble)[np.ix_(*src)]
spec = sf.rfftn(col)


def B_ld(v):
    y = sf.irfftn(sf.rfftn(v.astype(np.longdouble).reshape(n), s=T.embed) * spec, s=T.embed)
    return y[tuple(slice(0, ni) for ni in n)].reshape(-1)


Y = np.zeros((nlev, N))
for s in range(1, nlev + 1):
    rhs = -eta * A.q[s - 1] * g  # the split Arnoldi step's input: -eta q_s f_v
    if s > 1:
        rhs = rhs - A.diags.D1[s - 1] * (e[s - 1:0:-1] @ Y[:s - 1])
    d1, d2 = A.diags.D1[s - 1], A.diags.D2[s - 1]
    c, delta = A.scale_space, e[0] * d1 / d2
    b = rhs / d2
    lam = c * pcg.g + O._hmean(delta)
    M = lambda v: c * T.apply(v) + delta * v
    true_res = lambda v: float(np.linalg.norm(b.astype(np.longdouble) - (np.longdouble(c) * B_ld(v) + delta * v.astype(np.longdouble))))
    bn = np.linalg.norm(b)
    k = min(O.WARM_ORDER, s - 1)
    x, r = np.zeros(N), b.copy()
    if k:
        x = sum(float((-1) ** (j + 1) * math.comb(k, j)) * Y[s - 1 - j] for j in range(1, k + 1))
        r = b - M(x)
    show = s % 32 == 0
    if show:
        print(f"level {s}: guess ||r||/||b|| {np.linalg.norm(r) / bn:.2e} (80-bit {true_res(x) / bn:.2e})", end="  ")
    z = pcg._tau_inv(r, lam)
    p, rz, it = z.copy(), float(r @ z), 0
    for it in range(1, 201):
        Ap = M(p)
        alpha = rz / float(p @ Ap)
        x = x + alpha * p
        r = r - alpha * Ap
        if np.linalg.norm(r) <= 1e-14 * bn:
            break
        z = pcg._tau_inv(r, lam)
        rzn = float(r @ z)
        p, rz = z + (rzn / rz) * p, rzn
    Y[s - 1] = x
    if show:
        print(f"{it} CG steps: recursive {np.linalg.norm(r) / bn:.1e}, true (80-bit) {true_res(x) / bn:.2e}, "
              f"u||M||||x||/||b|| {2.0 ** -53 * lam.max() * np.linalg.norm(x) / bn:.2e}", flush=True)
