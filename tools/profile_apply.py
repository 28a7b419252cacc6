"""Run a few fast operator applies of a config (for ncu / nsys-less profiling)."""
import argparse, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_1807_00410_b200.configs import make_config
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--what", type=int, default=0)
a = ap.parse_args()
cfg = make_config(a.config, **({"n": a.n} if a.n else {}))
c = PnContext(build_tables(cfg.N), cfg.spec.res, cfg.spec.h)
c.set_fields(cfg.spec)
c.bench(a.what, 3)
ms = c.bench(a.what, a.reps)
print(f"cfg{a.config} n={cfg.spec.res} what={a.what}: {ms:.3f} ms per launch-group, {c.R_local/ms/1e6:.1f} Gunk/s")
