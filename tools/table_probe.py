"""Operator apply of the table kernel (grids with nx % 32 != 0) against the
segmented kernel, and the paper's point-source solves (80^3, P1 / P5)."""
import json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.run import make_pointsource
from paper_1807_00410_b200.solver import PnContext
for N, n in ((1, 80), (5, 80), (5, 96)):
    spec = make_pointsource(n)
    c = PnContext(build_tables(N), spec.res, spec.h)
    c.set_fields(spec)
    c.bench(0, 3)
    ms = c.bench(0, 20)
    c.solve(tol=1e-10, max_iter=5)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rep = c.solve(tol=1e-10, max_iter=200000)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"N": N, "n": n, "apply_ms": ms, "gunk_s": c.R_local / (ms / 1e3) / 1e9, "solve_s": dt,
                      "iterations": rep.iterations, "ms_per_iteration": 1e3 * dt / max(1, rep.iterations)}),
          flush=True)
    del c
