"""`fracinv solve` on the GPU: one inverse-problem solve and its report.

Mirrors the reference's solve command end to end:

* `ExperimentConfig`, `config_from_json`, `config_to_json`  — experiment.hpp:23-50,
  experiment.cpp:25-120 (same keys, same validation, unknown keys rejected with ConfigError);
* `solve_pipeline` — experiment.cpp:236-259: forward solve of f*, additive noise, right-hand
  side, GMRES (preconditioned and/or not), reconstruction error;
* `run_solve` — experiment.cpp:292-328: the report (keys iterations, converged,
  residual_history, final_true_residual, recon_error, wall_time_seconds, config) and the
  reconstruction CSV (`x,f_true,f_recon` or `x1,x2,f_true,f_recon`, every value `%.17g`);
* `main` — tools/main.cpp:116-170: the report printed as JSON (indent 2), the CSV written to
  `--out`, exit codes 0 (ok), 2 (usage / config / domain / resource), 3 (numerical), 4 (not
  converged).

Every numerical step runs through the device path (`fracinv.SystemOperator`,
`BlockTriangularPreconditioner`, `gmres`); this module is host-side orchestration only.

Extension: `--baseline-config i` solves BASELINE.json config i instead of a preset problem
(GMRES(50), seeded Gaussian noise; see configs.py), with the same report and CSV.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import sys
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import fracinv as F

ConfigError = F.ConfigError

_KEYS = ("preset", "beta", "omega", "orders", "n", "S", "lambda", "eps", "seed", "precond", "tol", "maxit", "mode",
         "out", "workers", "dense_cap")


@dataclasses.dataclass
class ExperimentConfig:
    """experiment.hpp:23-43 (defaults identical)."""

    preset: str = "paper1d"
    beta: float = 0.1
    omega: float = 1.9
    orders: List[Tuple[float, float]] = dataclasses.field(default_factory=list)
    n: List[int] = dataclasses.field(default_factory=lambda: [16])
    S: List[int] = dataclasses.field(default_factory=lambda: [16])
    lam: float = 5e-3
    lambda_sweep: List[float] = dataclasses.field(default_factory=list)
    eps: float = 0.01
    eps_sweep: List[float] = dataclasses.field(default_factory=list)
    seed: int = 1
    seeds: List[int] = dataclasses.field(default_factory=list)
    use_precond: bool = True
    tol: float = 1e-8
    maxit: int = 0  # 0 selects the matrix dimension
    mode: str = ""
    out: str = ""
    workers: int = 1
    dense_cap: int = F.BlockTriangularPreconditioner.kDefaultBlockCap


def format_double(v: float) -> str:
    """experiment.cpp:15-20: `%.17g`, -0 canonicalised to 0."""
    if v == 0.0:
        v = 0.0
    return "%.17g" % v


def _as_list(j: dict, key: str, typ):
    v = j[key]
    vals = v if isinstance(v, list) else [v]
    out = []
    for x in vals:
        if typ is int:
            if isinstance(x, bool) or not isinstance(x, (int, float)) or float(x) != int(x):
                raise ConfigError(f"'{key}' must be an integer or a list of integers")
            out.append(int(x))
        else:
            if isinstance(x, bool) or not isinstance(x, (int, float)):
                raise ConfigError(f"'{key}' must be a number or a list of numbers")
            out.append(float(x))
    return out


def config_from_json(j: dict) -> ExperimentConfig:
    """experiment.cpp:25-104: every recognised key, unknown keys rejected (ConfigError)."""
    if not isinstance(j, dict):
        raise ConfigError("config must be a JSON object")
    cfg = ExperimentConfig()
    for key, value in j.items():
        if key not in _KEYS:
            raise ConfigError(f"unknown config key '{key}'")
        if key == "preset":
            cfg.preset = str(value)
        elif key == "beta":
            cfg.beta = float(value)
        elif key == "omega":
            cfg.omega = float(value)
        elif key == "orders":
            if not isinstance(value, list) or not all(isinstance(p, list) and len(p) == 2 for p in value):
                raise ConfigError("'orders' must be a list of [beta, omega] pairs")
            cfg.orders = [(float(p[0]), float(p[1])) for p in value]
        elif key == "n":
            cfg.n = _as_list(j, key, int)
        elif key == "S":
            cfg.S = _as_list(j, key, int)
        elif key == "lambda":
            cfg.lambda_sweep = _as_list(j, key, float)
            if not cfg.lambda_sweep:
                raise ConfigError("'lambda' list must be non-empty")
            cfg.lam = cfg.lambda_sweep[0]
        elif key == "eps":
            cfg.eps_sweep = _as_list(j, key, float)
            if not cfg.eps_sweep:
                raise ConfigError("'eps' list must be non-empty")
            cfg.eps = cfg.eps_sweep[0]
        elif key == "seed":
            cfg.seeds = _as_list(j, key, int)
            if not cfg.seeds:
                raise ConfigError("'seed' list must be non-empty")
            cfg.seed = cfg.seeds[0]
        elif key == "precond":
            s = str(value)
            if s == "none":
                cfg.use_precond = False
            elif s in ("block-tri", "block_tri"):
                cfg.use_precond = True
            else:
                raise ConfigError(f"unknown precond '{s}' (expected 'none' or 'block-tri')")
        elif key == "tol":
            cfg.tol = float(value)
        elif key == "maxit":
            cfg.maxit = int(value)
        elif key == "mode":
            cfg.mode = str(value)
        elif key == "out":
            cfg.out = str(value)
        elif key == "workers":
            cfg.workers = int(value)
        elif key == "dense_cap":
            cfg.dense_cap = int(value)
    if not cfg.n:
        raise ConfigError("'n' must be non-empty")
    if not cfg.S:
        raise ConfigError("'S' must be non-empty")
    if not cfg.tol > 0.0:
        raise ConfigError("'tol' must be positive")
    if cfg.workers < 1:
        raise ConfigError("'workers' must be at least 1")
    return cfg


def config_to_json(cfg: ExperimentConfig) -> dict:
    """experiment.cpp:106-120: the effective single-run configuration echoed in a solve report."""
    return {"preset": cfg.preset, "beta": cfg.beta, "omega": cfg.omega, "n": list(cfg.n), "S": cfg.S[0],
            "lambda": cfg.lam, "eps": cfg.eps, "seed": cfg.seed, "precond": "block-tri" if cfg.use_precond else "none",
            "tol": cfg.tol, "maxit": cfg.maxit}


@dataclasses.dataclass
class PipelineResult:
    """experiment.cpp:226-234."""

    prec: F.SolveReport = dataclasses.field(default_factory=F.SolveReport)
    unprec: F.SolveReport = dataclasses.field(default_factory=F.SolveReport)
    recon_error: float = 0.0
    f_recon: Optional[np.ndarray] = None
    ran_unprec: bool = False
    ran_prec: bool = False


def solve_pipeline(op: F.SystemOperator, P: Optional[F.BlockTriangularPreconditioner], run_unprec: bool, eps: float,
                   seed: int, tol: float, maxit: int, *, restart: int = 0, gaussian: bool = False) -> PipelineResult:
    """experiment.cpp:236-259: manufacture data, add noise, solve, reconstruct.

    restart / gaussian: EXTENSIONS for the BASELINE configurations (GMRES(m); Gaussian noise of
    relative L2 level eps instead of the reference's additive uniform noise)."""
    mu = F.forward_solve(op, P).mu
    mu_eps = F.add_gaussian_noise(mu, eps, seed) if gaussian else F.add_noise(mu, eps, seed)
    rhs = F.build_rhs(op, mu_eps)
    out = PipelineResult()
    y = None
    opts = F.GmresOptions(tol=tol, maxit=maxit, restart=restart)
    if P is not None:
        y, out.prec = F.gmres(op, P, rhs.z, opts)
        out.ran_prec = True
    if run_unprec or P is None:
        yu, out.unprec = F.gmres(op, None, rhs.z, opts)
        out.ran_unprec = True
        if P is None:
            y = yu
    out.f_recon = F.extract_reconstruction(y, op.space_dim())
    out.recon_error = F.relative_error(op.spec.f_true, out.f_recon)
    return out


@dataclasses.dataclass
class SolveOutcome:
    """experiment.hpp (SolveOutcome): convergence flag, JSON report, reconstruction CSV."""

    converged: bool
    report: dict
    recon_csv: str


def _outcome(op: F.SystemOperator, res: PipelineResult, rep: F.SolveReport, config: dict) -> SolveOutcome:
    report = {
        "iterations": rep.iterations,
        "converged": rep.converged,
        "residual_history": list(rep.residual_history),
        "final_true_residual": rep.final_true_residual,
        "recon_error": res.recon_error,
        "wall_time_seconds": rep.wall_time_seconds,
        "config": config,
    }
    nodes = op.spec.sgrid.nodes()
    d = nodes.shape[1]
    head = "x,f_true,f_recon\n" if d == 1 else "".join(f"x{i + 1}," for i in range(d)) + "f_true,f_recon\n"
    rows = [head]
    f_true = np.asarray(op.spec.f_true)
    for j in range(nodes.shape[0]):
        rows.append("".join(format_double(float(c)) + "," for c in nodes[j]) + format_double(float(f_true[j])) + ","
                    + format_double(float(res.f_recon[j])) + "\n")
    return SolveOutcome(rep.converged, report, "".join(rows))


def run_solve(cfg: ExperimentConfig) -> SolveOutcome:
    """experiment.cpp:292-328."""
    op = F.SystemOperator(F.make_problem(cfg.preset, cfg.beta, cfg.omega, cfg.n, cfg.S[0], cfg.lam, cfg.eps))
    P = F.BlockTriangularPreconditioner(op, cfg.dense_cap) if cfg.use_precond else None
    res = solve_pipeline(op, P, not cfg.use_precond, cfg.eps, cfg.seed, cfg.tol, cfg.maxit)
    rep = res.prec if cfg.use_precond else res.unprec
    return _outcome(op, res, rep, config_to_json(cfg))


def run_baseline_solve(cfg_index: int, use_precond: bool = True, maxit: int = 0) -> SolveOutcome:
    """EXTENSION: BASELINE.json config `cfg_index` (GMRES(50), seeded Gaussian noise) with the
    same report and CSV as run_solve."""
    from .configs import NAMES, NOISE, RESTART, SEED_BASE, TOL, baseline_problem
    op = F.SystemOperator(baseline_problem(F, cfg_index))
    P = F.BlockTriangularPreconditioner(op) if use_precond else None
    seed = SEED_BASE + cfg_index
    res = solve_pipeline(op, P, not use_precond, NOISE[cfg_index], seed, TOL[cfg_index], maxit, restart=RESTART,
                         gaussian=True)
    rep = res.prec if use_precond else res.unprec
    config = {"baseline_config": cfg_index, "workload": NAMES[cfg_index], "n": list(op.spec.sgrid.n),
              "S": op.steps(), "eps": NOISE[cfg_index], "noise": "gaussian", "seed": seed,
              "precond": "block-tri" if use_precond else "none", "tol": TOL[cfg_index], "maxit": maxit,
              "restart": RESTART}
    return _outcome(op, res, rep, config)


def _parse_list(s: str, typ):
    return [typ(v) for v in s.replace(",", " ").split()]


def main(argv: Optional[Sequence[str]] = None) -> int:
    """tools/main.cpp:116-170 (solve subcommand): flags override the --config file's fields."""
    ap = argparse.ArgumentParser(prog="python -m paper_2507_02809_b200.solve",
                                 description="run one inverse-problem solve on the GPU and report")
    ap.add_argument("--config", default="", help="JSON config file; flags override its fields")
    ap.add_argument("--beta", type=float)
    ap.add_argument("--omega", type=float)
    ap.add_argument("--n", help="grid size per direction (comma separated)")
    ap.add_argument("--S", type=int)
    ap.add_argument("--lambda", dest="lam", type=float)
    ap.add_argument("--eps", type=float)
    ap.add_argument("--seed", type=int)
    ap.add_argument("--preset")
    ap.add_argument("--precond", choices=["none", "block-tri", "block_tri"])
    ap.add_argument("--tol", type=float)
    ap.add_argument("--maxit", type=int)
    ap.add_argument("--out")
    ap.add_argument("--dense-cap", dest="dense_cap", type=int)
    ap.add_argument("--baseline-config", type=int, choices=[0, 1, 2, 3, 4],
                    help="EXTENSION: solve BASELINE.json config i (GMRES(50), Gaussian noise)")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    try:
        if args.baseline_config is not None:
            outcome = run_baseline_solve(args.baseline_config, args.precond != "none", args.maxit or 0)
            out_path = args.out or ""
        else:
            j = {}
            if args.config:
                try:
                    with open(args.config) as fh:
                        j = json.load(fh)
                except OSError:
                    raise ConfigError(f"cannot open config file '{args.config}'")
                except json.JSONDecodeError as ex:
                    raise ConfigError(f"malformed config JSON: {ex}")
            for key, val in (("beta", args.beta), ("omega", args.omega), ("S", args.S), ("lambda", args.lam),
                             ("eps", args.eps), ("seed", args.seed), ("preset", args.preset),
                             ("precond", args.precond), ("tol", args.tol), ("maxit", args.maxit), ("out", args.out),
                             ("dense_cap", args.dense_cap)):
                if val is not None:
                    j[key] = val
            if args.n is not None:
                j["n"] = _parse_list(args.n, int)
            cfg = config_from_json(j)
            if not (cfg.omega > 1.0 and cfg.omega <= 2.0):
                raise ConfigError(f"omega must lie in (1,2] for the fractional Laplacian symbol, got {cfg.omega}")
            outcome = run_solve(cfg)
            out_path = cfg.out
        print(json.dumps(outcome.report, indent=2))
        if out_path:
            with open(out_path, "w") as fh:
                fh.write(outcome.recon_csv)
        if not outcome.converged:
            print("gmres did not reach the requested tolerance", file=sys.stderr)
            return 4
    except ConfigError as ex:
        print(f"config error: {ex}", file=sys.stderr)
        return 2
    except F.DimensionError as ex:  # std::domain_error family in the reference
        print(f"invalid parameter: {ex}", file=sys.stderr)
        return 2
    except ValueError as ex:
        print(f"invalid parameter: {ex}", file=sys.stderr)
        return 2
    except F.ResourceLimitError as ex:
        print(f"resource limit: {ex} (see --dense-cap)", file=sys.stderr)
        return 2
    except F.SingularBlockError as ex:
        print(f"numerical failure: {ex}", file=sys.stderr)
        return 3
    except Exception as ex:  # noqa: BLE001 (the reference maps every other exception to 3)
        print(f"error: {ex}", file=sys.stderr)
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
