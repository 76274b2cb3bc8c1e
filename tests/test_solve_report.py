"""The `fracinv solve` report (paper_2507_02809_b200/solve.py): config
parsing and echo (experiment.cpp:25-120), `%.17g` formatting (experiment.cpp:15-20), CLI exit
codes (tools/main.cpp:150-168) on CPU; on the GPU the reference's own solve test case
(test_experiment.cpp:188-219) and parity of the whole pipeline with the oracle's."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2507_02809_b200 import solve as SV

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_config_from_json_keys_and_defaults():
    cfg = SV.config_from_json({})
    assert (cfg.preset, cfg.beta, cfg.omega, cfg.n, cfg.S, cfg.lam, cfg.eps, cfg.seed) == \
        ("paper1d", 0.1, 1.9, [16], [16], 5e-3, 0.01, 1)
    assert cfg.use_precond and cfg.tol == 1e-8 and cfg.maxit == 0 and cfg.dense_cap == 4096
    cfg = SV.config_from_json({"n": [32, 16], "S": 8, "lambda": [1e-3, 1e-2], "eps": 0.0, "seed": [5, 6],
                               "precond": "block_tri", "tol": 1e-10, "maxit": 7, "orders": [[0.5, 1.5]]})
    assert cfg.n == [32, 16] and cfg.S == [8] and cfg.lam == 1e-3 and cfg.lambda_sweep == [1e-3, 1e-2]
    assert cfg.seed == 5 and cfg.seeds == [5, 6] and cfg.use_precond and cfg.orders == [(0.5, 1.5)]
    assert not SV.config_from_json({"precond": "none"}).use_precond


@pytest.mark.parametrize("bad", [{"bogus": 1}, {"precond": "ilu"}, {"tol": 0.0}, {"workers": 0}, {"n": []},
                                 {"n": [1.5]}, {"lambda": []}, {"orders": [[0.5]]}])
def test_config_from_json_rejects(bad):
    with pytest.raises(SV.ConfigError):
        SV.config_from_json(bad)


def test_config_to_json_echo():
    cfg = SV.config_from_json({"beta": 0.5, "omega": 1.5, "S": [32, 64], "precond": "none"})
    j = SV.config_to_json(cfg)
    assert set(j) == {"preset", "beta", "omega", "n", "S", "lambda", "eps", "seed", "precond", "tol", "maxit"}
    assert j["S"] == 32 and j["precond"] == "none" and j["beta"] == 0.5


def test_format_double():
    assert SV.format_double(-0.0) == "0"
    assert SV.format_double(0.1) == "0.10000000000000001"
    assert SV.format_double(1.0) == "1"
    assert float(SV.format_double(np.pi)) == np.pi


def _cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2507_02809_b200.solve", *args], capture_output=True,
                          text=True, cwd=cwd or ROOT, timeout=600)


@pytest.mark.parametrize("args", [["--omega", "2.5"], ["--config", "/nonexistent.json"], ["--bogus-flag"]])
def test_cli_usage_errors_exit_2(args):
    r = _cli(*args)
    assert r.returncode == 2, r.stderr


def test_cli_config_error_exit_2(tmp_path):
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"unknown_key": 1}))
    r = _cli("--config", str(p))
    assert r.returncode == 2 and "config error" in r.stderr


@pytest.mark.gpu
def test_run_solve_reference_case():
    """test_experiment.cpp:188-219 verbatim: paper1d, (0.1, 1.9), n = S = 16."""
    cfg = SV.ExperimentConfig(preset="paper1d", beta=0.1, omega=1.9, n=[16], S=[16], lam=5e-3, eps=0.01, seed=1)
    out = SV.run_solve(cfg)
    assert out.converged
    it = out.report["iterations"]
    assert 6 <= it <= 10  # reference count is 8
    assert out.report["converged"] is True
    assert out.report["final_true_residual"] < 1e-4
    assert out.report["recon_error"] < 0.2
    assert "residual_history" in out.report and "wall_time_seconds" in out.report
    assert out.report["config"]["preset"] == "paper1d"
    lines = out.recon_csv.strip().split("\n")
    assert len(lines) == 17 and lines[0] == "x,f_true,f_recon"
    row = lines[1].split(",")
    assert len(row) == 3
    x = float(row[0])
    assert float(row[1]) == pytest.approx(x * np.sin(x), rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("precond", [True, False])
def test_run_solve_matches_oracle_pipeline(precond):
    """The device pipeline (forward solve, noise, rhs, GMRES) against the oracle's on the same
    inputs: identical iteration count, history and reconstruction to 1e-10."""
    from oracle import fracinv_oracle as O
    cfg = SV.ExperimentConfig(beta=0.5, omega=1.5, n=[32], S=[16], use_precond=precond)
    out = SV.run_solve(cfg)
    Ao = O.SystemOperator(O.make_problem("paper1d", 0.5, 1.5, [32], 16, 5e-3, 0.01))
    mu = O.forward_solve(Ao).mu
    z = O.build_rhs(Ao, O.add_noise(mu, 0.01, 1)).z
    Po = O.BlockTriangularPreconditioner(Ao) if precond else None
    x, rep = O.gmres(Ao.apply, Po.apply if Po else None, z, tol=1e-8, maxit=0)
    f = x[-Ao.space_dim:]
    assert out.report["iterations"] == rep.iterations
    assert np.allclose(out.report["residual_history"], rep.residual_history, rtol=1e-6, atol=1e-14)
    fr = np.array([float(l.split(",")[2]) for l in out.recon_csv.strip().split("\n")[1:]])
    assert np.linalg.norm(fr - f) / np.linalg.norm(f) <= 1e-10


@pytest.mark.gpu
def test_cli_solve_writes_report_and_csv(tmp_path):
    out = tmp_path / "recon.csv"
    r = _cli("--beta", "0.5", "--omega", "1.5", "--n", "16", "--S", "16", "--out", str(out))
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["converged"] and rep["config"]["beta"] == 0.5
    assert out.read_text().startswith("x,f_true,f_recon\n")
    # non-convergence: exit code 4 (tools/main.cpp:141-145)
    r = _cli("--n", "16", "--S", "16", "--maxit", "1", "--precond", "none")
    assert r.returncode == 4


@pytest.mark.gpu
def test_baseline_config0_report():
    g = np.load(os.path.join(ROOT, "tests", "golden", "oracle_config0.npz"))
    out = SV.run_baseline_solve(0)
    assert out.converged and abs(out.report["iterations"] - int(g["iterations"])) <= 1
    assert out.report["recon_error"] == pytest.approx(float(g["recon_error"]), rel=1e-6)
    assert out.recon_csv.split("\n")[0] == "x,f_true,f_recon"
