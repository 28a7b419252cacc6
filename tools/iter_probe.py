"""Per-iteration cost of the real fast solve (graph batches, fixed iteration
count) against the bench's bare iteration loop, on a config."""
import argparse, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--iters", type=int, default=100)
a = ap.parse_args()
cfg = make_config(a.config)
spec = solve_spec(cfg)
c = PnContext(build_tables(cfg.N), spec.res, spec.h)
c.set_fields(spec)
c.bench(1, 3)
print(f"cfg{a.config} bench iteration: {c.bench(1, 20):.3f} ms", flush=True)
for ce in (0, 4, 16, 64):
    c.solve(tol=1e-300, max_iter=8, check_every=ce)
    ts = []
    for n in (a.iters // 2, a.iters):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        c.solve(tol=1e-300, max_iter=n, check_every=ce)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(f"cfg{a.config} solve check_every={ce}: {1e3 * (ts[1] - ts[0]) / (a.iters - a.iters // 2):.3f} ms/iteration "
          f"(fixed overhead {1e3 * (2 * ts[0] - ts[1]):.1f} ms)", flush=True)
