"""Batch front door with the solve on the GPU (the reference's `pnrte run`,
cli.py:133-171: problem -> assemble -> CGNR -> unstagger -> artifacts).

    python -m paper_1807_00410_b200.run run --problem cfg2 --order 3 --out out/

Artifacts: field.pnfld (PNFLD1), profile.csv (fluence along +x through the
centre), solve.log (residual history).  Exit status follows cli.py:27-30:
0 converged, 2 bad configuration, 3 not converged or vacuum at admission,
4 internal error.

Problems: `pointsource` (homogeneous medium with a unit emitter,
problems.py:130-156) and the BASELINE configurations `cfg1`..`cfg5`
(configs.py).  Methods: `pn` (matrix-free P_N stencil) and `cda` (collapsed
diffusion: explicit device CSR from general.py, field order 0).
"""

from __future__ import annotations

import argparse
import math
import os
import sys
from dataclasses import dataclass, replace

import numpy as np

from . import fields as fio
from .problems import ProblemSpec, SingularRiskError, floor_sigma_t, phase_fields, validate_for_solve
from .program import InvalidOrderError, PlacementError, build_tables, q_name

EXIT_OK, EXIT_CONFIG, EXIT_NOCONV, EXIT_INTERNAL = 0, 2, 3, 4
PROBLEMS = ("pointsource", "cfg1", "cfg2", "cfg3", "cfg4", "cfg5")
SQRT_4PI = math.sqrt(4.0 * math.pi)


class ConfigError(Exception):
    """A run option with a bad name or value (exit status 2)."""


def _flag(text):
    word = str(text).strip().lower()
    if word in ("1", "true", "yes", "on"):
        return True
    if word in ("0", "false", "no", "off"):
        return False
    raise ValueError(f"not a boolean: {text!r}")


# option name -> (parser, default, admissible-value check or None)
OPTIONS = {
    "problem": (str, "pointsource", lambda v: v in PROBLEMS),
    "method": (str, "pn", lambda v: v in ("pn", "cda")),
    "order": (int, 1, None),
    "res": (int, 0, lambda v: v >= 0),                   # 0: the problem's default
    "floor": (float, -1.0, None),                        # <= 0: the problem's default
    "tol": (float, 1e-8, lambda v: v > 0),
    "max_iter": (int, 50000, lambda v: v >= 1),
    "out": (str, "out", None),
    "seed": (int, 0, None),
    "jacobi": (_flag, False, None),
    "mode": (str, "fast", lambda v: v in ("fast", "faithful")),
    "bc": (str, "", lambda v: v in ("", "dirichlet", "neumann")),   # '': the problem's
    "device": (int, 0, lambda v: v >= 0),
}


@dataclass(frozen=True)
class RunConfig:
    problem: str = "pointsource"
    method: str = "pn"
    order: int = 1
    res: int = 0
    floor: float = -1.0
    tol: float = 1e-8
    max_iter: int = 50000
    out: str = "out"
    seed: int = 0
    jacobi: bool = False
    mode: str = "fast"
    bc: str = ""
    device: int = 0


def config_from_mapping(mapping):
    """RunConfig from string (or typed) values; keys may use '-' or '_'."""
    values = {}
    for raw_key, raw in mapping.items():
        key = str(raw_key).replace("-", "_")
        if key not in OPTIONS:
            raise ConfigError(f"unknown option {raw_key!r}")
        parse, _, ok = OPTIONS[key]
        try:
            val = parse(raw)
        except (TypeError, ValueError) as exc:
            raise ConfigError(f"option {raw_key!r}: {exc}") from None
        if ok is not None and not ok(val):
            raise ConfigError(f"option {raw_key!r}: value {raw!r} not allowed")
        values[key] = val
    cfg = RunConfig(**values)
    if cfg.method == "pn" and cfg.order < 1:
        raise ConfigError(f"order must be >= 1 for the P_N method, got {cfg.order}")
    return cfg


def make_pointsource(res=80, sigma_t=8.0, albedo=0.9, extent=2.0, g=0.0, max_band=8):
    """Homogeneous medium, unit isotropic emitter in the centre voxel with the
    power-preserving amplitude 1/(h^3 sqrt(4 pi)) (problems.py:130-156)."""
    if res < 8:
        raise ValueError("resolution too small for the point source problem")
    n = int(res)
    h = extent / n
    shape = (n,) * 3
    emission = np.zeros(shape)
    emission[(n // 2,) * 3] = 1.0 / (h ** 3 * SQRT_4PI)
    flds = {"sigma_t": np.full(shape, float(sigma_t)), "sigma_s": np.full(shape, float(albedo * sigma_t)),
            q_name(0, 0): emission, **phase_fields(g, max_band)}
    return ProblemSpec(dim=3, origin=(-extent / 2.0,) * 3, extent=(extent,) * 3, res=shape, fields=flds,
                       bc="dirichlet", sigma_t_floor=min(sigma_t, 1.0), name="pointsource")


def build_problem(cfg):
    """The ProblemSpec a run solves: generator, sigma_t floor, boundary."""
    from .configs import make_config
    if cfg.problem == "pointsource":
        spec, tau = make_pointsource(cfg.res or 80, max_band=max(8, cfg.order)), None
    else:
        kw = {"seed": cfg.seed, **({"n": cfg.res} if cfg.res else {})}
        made = make_config(int(cfg.problem[len("cfg"):]), **kw)
        spec, tau = made.spec, made.floor
    if cfg.floor > 0:
        tau = cfg.floor
    spec = floor_sigma_t(spec, tau) if tau else spec
    return replace(spec, bc=cfg.bc) if cfg.bc else spec


def center_profile(spec, coll):
    """(r, fluence) along +x through the centre line (cli.py:119-130): from
    the emitter voxel for the point source, across the domain otherwise."""
    fluence = SQRT_4PI * coll[..., 0]
    centre = tuple(r // 2 for r in spec.res)
    if spec.name == "pointsource":
        values = fluence[centre[0]:, centre[1], centre[2]]
        return np.arange(values.shape[0]) * spec.h, values
    values = fluence[:, centre[1], centre[2]]
    return spec.centers(0) - spec.origin[0], values


def _solve(cfg, spec, log):
    """Device assembly + CGNR + unstagger; returns (rows, collocated, order, report)."""
    from .solver import PnContext, assemble_general
    if cfg.method == "cda":
        from .general import build_cda_program
        op, rhs = assemble_general(build_cda_program(spec.dim), spec, device=cfg.device)
        grid_ctx, order, what = op, 0, "CDA: explicit device CSR, field-dependent couplings"
    else:
        grid_ctx = PnContext(build_tables(cfg.order, dim=spec.dim), spec.res, spec.h, device=cfg.device)
        grid_ctx.set_fields(spec)
        order = cfg.order
        if spec.bc == "neumann":
            op, rhs = grid_ctx.assemble_csr("neumann")
            what = f"P{cfg.order}, Neumann: explicit device CSR"
        else:
            op, rhs = grid_ctx, None
            what = f"matrix-free P{cfg.order} stencil"
    log(f"assembled {op.R_local} rows on cuda:{cfg.device} ({what})")
    x, report = op.solve(tol=cfg.tol, max_iter=cfg.max_iter, jacobi=cfg.jacobi, mode=cfg.mode, b=rhs)
    return op.R_local, grid_ctx.unstagger(x).cpu().numpy(), order, report


def _artifacts(cfg, spec, rows, coll, order, report, log):
    log(f"solve: {report.iterations} iterations, converged={report.converged}, "
        f"normal={report.normal_residual:.3e}, primal={report.primal_residual:.3e}, wall={report.wall_time:.2f}s")
    os.makedirs(cfg.out, exist_ok=True)
    fio.write_field(os.path.join(cfg.out, "field.pnfld"), coll, order)
    fio.write_profile(os.path.join(cfg.out, "profile.csv"), zip(*center_profile(spec, coll)))
    summary = {"rows": rows, "method": cfg.method, "mode": cfg.mode, "bc": spec.bc,
               "iterations": report.iterations, "converged": report.converged,
               "normal_residual": repr(report.normal_residual), "primal_residual": repr(report.primal_residual),
               "wall_time": repr(report.wall_time)}
    history = [f"{k} {n!r} {p!r}" for k, (n, p) in
               enumerate(zip(report.normal_history, report.primal_history), start=1)]
    with open(os.path.join(cfg.out, "solve.log"), "w") as fh:
        fh.write("\n".join([f"{k} {v}" for k, v in summary.items()] + ["# iter normal primal"] + history) + "\n")


def run(cfg, log=print):
    spec = build_problem(cfg)
    validate_for_solve(spec)
    rows, coll, order, report = _solve(cfg, spec, log)
    _artifacts(cfg, spec, rows, coll, order, report, log)
    return report


# exception class -> (exit status, message prefix), checked in order
_FAILURES = ((ConfigError, EXIT_CONFIG, "config error"), (InvalidOrderError, EXIT_CONFIG, "config error"),
             (SingularRiskError, EXIT_NOCONV, "singular system"), (PlacementError, EXIT_INTERNAL, "internal error"),
             (ValueError, EXIT_CONFIG, "config error"), (OSError, EXIT_CONFIG, "config error"))


def _status(exc):
    for cls, code, prefix in _FAILURES:
        if isinstance(exc, cls):
            print(f"{prefix}: {exc}", file=sys.stderr)
            return code
    raise exc


def _parser():
    ap = argparse.ArgumentParser(prog="pnrte-b200", description="B200 P_N solve: run a problem, write artifacts")
    commands = ap.add_subparsers(dest="command", required=True)
    p = commands.add_parser("run")
    p.add_argument("--spec", help="key=value configuration file")
    for name, (parse, _, _) in OPTIONS.items():
        flag = "--" + name.replace("_", "-")
        if parse is _flag:
            p.add_argument(flag, dest=name, action="store_const", const="true")
        else:
            p.add_argument(flag, dest=name)
    return ap


def main(argv=None):
    try:
        args = _parser().parse_args(argv)
    except SystemExit as exc:
        return EXIT_CONFIG if exc.code not in (0, None) else EXIT_OK
    try:
        settings = fio.read_config(args.spec) if args.spec else {}
        settings.update({k: v for k, v in vars(args).items() if k in OPTIONS and v is not None})
        cfg = config_from_mapping(settings)
        report = run(cfg)
    except Exception as exc:   # mapped to the reference's exit statuses
        return _status(exc)
    if not report.converged:
        print("solver did not converge", file=sys.stderr)
        return EXIT_NOCONV
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
