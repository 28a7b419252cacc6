"""Time the fast CG vector kernels and the fused iteration on a config (bench modes 1, 4, 5)."""
import argparse, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_1807_00410_b200.configs import make_config
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
cfg = make_config(a.config)
c = PnContext(build_tables(cfg.N), cfg.spec.res, cfg.spec.h)
c.set_fields(cfg.spec)
gb = c.R_local * 8 / 1e9
for what, passes, name in ((4, 3, "r update"), (5, 5, "x/p update"), (1, None, "CG iteration")):
    c.bench(what, 3)
    ms = c.bench(what, a.reps)
    extra = f", {passes * gb / ms * 1e3:.0f} GB/s over {passes} passes" if passes else ""
    print(f"cfg{a.config} {name}: {ms:.3f} ms{extra}", flush=True)
