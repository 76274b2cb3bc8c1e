"""The reference-style C++ program (tests/cpp/test_facade.cpp) over the C++ façade and C-ABI:
BASELINE config 0 end to end against the CPU oracle, plus the reference's error contract."""
import json
import os
import subprocess
import warnings

import numpy as np
import pytest

from oracle import fracinv_oracle as O
from paper_2507_02809_b200.configs import baseline_problem

pytestmark = pytest.mark.gpu
warnings.filterwarnings("ignore", module="scipy")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "test_facade")


def test_cpp_facade_config0(tmp_path):
    if not os.path.exists(EXE):
        subprocess.run(["bash", os.path.join(ROOT, "tests", "cpp", "build.sh")], check=True)
    out = tmp_path / "f.bin"
    res = subprocess.run([EXE, str(out)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    rep = json.loads(res.stdout.strip().splitlines()[-1])
    f = np.fromfile(out, dtype=np.float64)
    Ao = O.SystemOperator(baseline_problem(O, 0))
    Po = O.BlockTriangularPreconditioner(Ao)
    z = O.build_rhs(Ao, O.add_gaussian_noise(O.forward_solve(Ao).mu, 0.01, 1000)).z
    xo, repo = O.gmres(Ao.apply, Po.apply, z, tol=1e-10, restart=50)
    assert rep["converged"] and abs(rep["iterations"] - repo.iterations) <= 1
    assert rep["history_len"] == rep["iterations"] + 1
    assert np.linalg.norm(f - xo[-255:]) / np.linalg.norm(xo[-255:]) <= 1e-8
    assert rep["singular_index"] == 3 and rep["dimension_error"]
    assert rep["tau_inner"] == 1 and rep["tau_vs_dense"] <= 1e-12  # substituted 2D block solve
    # the operator's realisations through the facade: K1f by default on the 2D grid, equal to K1; 1D refuses FFT
    assert rep["fft_default"] and rep["fft_vs_dmma"] <= 1e-13 and rep["fft_refused_1d"]
