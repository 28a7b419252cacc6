"""Device-integrated batch run (the reference's `pnrte run`, cli.py:133-171).

    python -m paper_1807_00410_b200.run run --problem cfg2 --order 3 --out out/

Same pipeline and artifacts as the reference CLI, with the solve on the GPU:
build the stencil tables -> assemble on the device -> CGNR -> unstagger ->
field.pnfld (PNFLD1), profile.csv (fluence along +x through the centre),
solve.log (residual history).  Exit codes as cli.py:27-30: 0 ok, 2 config
error, 3 non-convergence or singular system (vacuum) at admission, 4
internal error.

Problems: `pointsource` (homogeneous medium, unit point emitter,
problems.py:130-156 restated) and the BASELINE configurations `cfg1`..`cfg5`
(configs.py).  Methods: `pn` (matrix-free P_N stencil) and `cda` (collapsed
diffusion, field-dependent couplings: explicit device CSR from
general.py, field order 0 as cli.py:156).  The 2-D checkerboard is not a
`run` problem here.
"""

from __future__ import annotations

import argparse
import math
import os
import sys
from dataclasses import dataclass, fields as dc_fields, replace

import numpy as np

from . import fields as fio
from .problems import ProblemSpec, SingularRiskError, floor_sigma_t, phase_fields, validate_for_solve
from .program import InvalidOrderError, PlacementError, build_tables, q_name

EXIT_OK, EXIT_CONFIG, EXIT_NOCONV, EXIT_INTERNAL = 0, 2, 3, 4
PROBLEMS = ("pointsource", "cfg1", "cfg2", "cfg3", "cfg4", "cfg5")
SQRT_4PI = math.sqrt(4.0 * math.pi)


class ConfigError(Exception):
    pass


@dataclass
class RunConfig:
    problem: str = "pointsource"
    method: str = "pn"            # pn | cda
    order: int = 1
    res: int = 0                  # 0 = problem default
    floor: float = -1.0           # < 0 = problem default
    tol: float = 1e-8
    max_iter: int = 50000
    out: str = "out"
    seed: int = 0
    jacobi: bool = False
    mode: str = "fast"            # fast | faithful
    bc: str = ""                  # '' = problem default | dirichlet | neumann (cli.py:46,105-107)
    device: int = 0

    def validated(self):
        if self.problem not in PROBLEMS:
            raise ConfigError(f"unknown problem {self.problem!r}")
        if self.method not in ("pn", "cda"):
            raise ConfigError(f"unknown method {self.method!r}")
        if self.method == "pn" and self.order < 1:
            raise ConfigError(f"order must be >= 1, got {self.order}")
        if self.tol <= 0:
            raise ConfigError("tol must be positive")
        if self.max_iter < 1:
            raise ConfigError("max-iter must be >= 1")
        if self.mode not in ("fast", "faithful"):
            raise ConfigError(f"unknown mode {self.mode!r}")
        if self.bc and self.bc not in ("dirichlet", "neumann"):
            raise ConfigError(f"unknown bc {self.bc!r}")
        return self


_BOOLS = {"true": True, "false": False, "1": True, "0": False}


def config_from_mapping(mapping):
    cfg = RunConfig()
    known = {f.name for f in dc_fields(RunConfig)}
    for key, val in mapping.items():
        name = key.replace("-", "_")
        if name not in known:
            raise ConfigError(f"unknown config key {key!r}")
        cur = getattr(cfg, name)
        if isinstance(cur, bool):
            if str(val).lower() not in _BOOLS:
                raise ConfigError(f"bad boolean for {key!r}: {val!r}")
            setattr(cfg, name, _BOOLS[str(val).lower()])
        elif isinstance(cur, int):
            setattr(cfg, name, int(val))
        elif isinstance(cur, float):
            setattr(cfg, name, float(val))
        else:
            setattr(cfg, name, str(val))
    return cfg.validated()


def make_pointsource(res=80, sigma_t=8.0, albedo=0.9, extent=2.0, g=0.0, max_band=8):
    """Homogeneous medium with a unit isotropic emitter in the centre voxel,
    power-preserving 1/(h^3 sqrt(4 pi)) (problems.py:130-156)."""
    if res < 8:
        raise ValueError("resolution too small for the point source problem")
    n = int(res)
    h = extent / n
    shape = (n, n, n)
    q00 = np.zeros(shape)
    c = n // 2
    q00[c, c, c] = 1.0 / (h ** 3 * SQRT_4PI)
    f = {"sigma_t": np.full(shape, float(sigma_t)), "sigma_s": np.full(shape, float(albedo * sigma_t)),
         q_name(0, 0): q00}
    f.update(phase_fields(g, max_band))
    half = extent / 2.0
    return ProblemSpec(dim=3, origin=(-half,) * 3, extent=(extent,) * 3, res=shape, fields=f, bc="dirichlet",
                       sigma_t_floor=min(sigma_t, 1.0), name="pointsource")


def build_problem(cfg):
    from .configs import make_config
    if cfg.problem == "pointsource":
        spec, floor = make_pointsource(cfg.res or 80, max_band=max(8, cfg.order)), None
    else:
        idx = int(cfg.problem[3:])
        kw = {"seed": cfg.seed}
        if cfg.res:
            kw["n"] = cfg.res
        c = make_config(idx, **kw)
        spec, floor = c.spec, c.floor
    tau = cfg.floor if cfg.floor > 0 else floor
    if tau:
        spec = floor_sigma_t(spec, tau)
    if cfg.bc:
        spec = replace(spec, bc=cfg.bc)
    return spec


def center_profile(spec, coll):
    """Fluence sqrt(4 pi) L00 along +x through the centre (cli.py:119-130)."""
    flu = SQRT_4PI * coll[..., 0]
    if spec.name == "pointsource":
        src = tuple(r // 2 for r in spec.res)
        line = flu[(slice(src[0], None),) + src[1:]]
        r = np.arange(line.shape[0]) * spec.h
    else:
        mid = tuple(r // 2 for r in spec.res)
        line = flu[(slice(None),) + mid[1:]]
        r = spec.centers(0) - spec.origin[0]
    return r, line


def run(cfg, log=print):
    from .solver import PnContext
    spec = build_problem(cfg)
    validate_for_solve(spec)
    if cfg.method == "cda":
        return _run_cda(cfg, spec, log)
    tables = build_tables(cfg.order)
    os.makedirs(cfg.out, exist_ok=True)
    ctx = PnContext(tables, spec.res, spec.h, device=cfg.device)
    ctx.set_fields(spec)
    R = ctx.R_local
    if spec.bc == "neumann":
        op, b = ctx.assemble_csr("neumann")
        log(f"assembled {R} rows on cuda:{cfg.device} (P{cfg.order}, Neumann: explicit device CSR)")
    else:
        op, b = ctx, None
        log(f"assembled {R} rows on cuda:{cfg.device} (matrix-free P{cfg.order} stencil)")
    x, report = op.solve(tol=cfg.tol, max_iter=cfg.max_iter, jacobi=cfg.jacobi, mode=cfg.mode, b=b)
    coll = ctx.unstagger(x).cpu().numpy()
    _write(cfg, spec, R, coll, cfg.order, report, log)
    return report


def _run_cda(cfg, spec, log):
    from .general import build_cda_program
    from .solver import assemble_general
    os.makedirs(cfg.out, exist_ok=True)
    csr, q = assemble_general(build_cda_program(spec.dim), spec, device=cfg.device)
    R = csr.R_local
    log(f"assembled {R} rows on cuda:{cfg.device} (CDA: explicit device CSR, field-dependent couplings)")
    x, report = csr.solve(tol=cfg.tol, max_iter=cfg.max_iter, jacobi=cfg.jacobi, mode=cfg.mode, b=q)
    coll = csr.unstagger(x).cpu().numpy()
    _write(cfg, spec, R, coll, 0, report, log)
    return report


def _write(cfg, spec, R, coll, order, report, log):
    log(f"solve: {report.iterations} iterations, converged={report.converged}, "
        f"normal={report.normal_residual:.3e}, primal={report.primal_residual:.3e}, "
        f"wall={report.wall_time:.2f}s")
    fio.write_field(os.path.join(cfg.out, "field.pnfld"), coll, order)
    r, line = center_profile(spec, coll)
    fio.write_profile(os.path.join(cfg.out, "profile.csv"), zip(r, line))
    with open(os.path.join(cfg.out, "solve.log"), "w") as fh:
        fh.write(f"rows {R}\nmethod {cfg.method}\nmode {cfg.mode}\nbc {spec.bc}\n")
        fh.write(f"iterations {report.iterations}\nconverged {report.converged}\n")
        fh.write(f"normal_residual {report.normal_residual!r}\nprimal_residual {report.primal_residual!r}\n")
        fh.write(f"wall_time {report.wall_time!r}\n# iter normal primal\n")
        for i, (nr, pr) in enumerate(zip(report.normal_history, report.primal_history), 1):
            fh.write(f"{i} {nr!r} {pr!r}\n")
    return report


def main(argv=None):
    parser = argparse.ArgumentParser(prog="pnrte-b200", description="B200 P_N solve: run a problem, export artifacts")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("run")
    p.add_argument("--spec", help="key=value config file")
    for f in dc_fields(RunConfig):
        if f.type in ("bool", bool):
            p.add_argument("--" + f.name.replace("_", "-"), dest=f.name, action="store_true", default=None)
        else:
            p.add_argument("--" + f.name.replace("_", "-"), dest=f.name, default=None)
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return EXIT_CONFIG if exc.code not in (0, None) else 0
    try:
        mapping = fio.read_config(args.spec) if args.spec else {}
        for f in dc_fields(RunConfig):
            v = getattr(args, f.name, None)
            if v is not None:
                mapping[f.name] = v
        cfg = config_from_mapping(mapping)
    except (ConfigError, ValueError, OSError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    try:
        report = run(cfg)
    except (InvalidOrderError, ConfigError, ValueError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except SingularRiskError as exc:
        print(f"singular system: {exc}", file=sys.stderr)
        return EXIT_NOCONV
    except PlacementError as exc:
        print(f"internal error: {exc}", file=sys.stderr)
        return EXIT_INTERNAL
    if not report.converged:
        print("solver did not converge", file=sys.stderr)
        return EXIT_NOCONV
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
