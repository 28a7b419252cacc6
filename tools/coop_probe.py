"""One-launch small solve (launch_cg_small) vs the graph-replayed launch chain:
ms per iteration of fixed-iteration fast solves over grid sizes and orders,
and config-1/2 time to residual 1e-6 on both paths (PNRTE_SMALL_MAX)."""
import json, os, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1] / "tests"))
from cases import rand_spec


def timed(ctx, **kw):
    ctx.solve(**dict(kw, max_iter=5))
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        x, rep = ctx.solve(**kw)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        best = t if best is None else min(best, t)
    return best, rep


for N, n in [(1, 8), (1, 16), (1, 24), (1, 32), (1, 40), (1, 48), (1, 64), (3, 8), (3, 12), (3, 16), (3, 20), (3, 24), (3, 32),
             (5, 8), (5, 12), (5, 16), (5, 24), (7, 8), (7, 12), (7, 16)]:
    spec = rand_spec(N, (n, n, n), 1)
    row = {"N": N, "n": n, "R": n ** 3 * (N + 1) ** 2}
    for name, lim in (("small", str(1 << 40)), ("chain", "0")):
        os.environ["PNRTE_SMALL_MAX"] = lim
        c = PnContext(build_tables(N), spec.res, spec.h)
        c.set_fields(spec)
        t, rep = timed(c, tol=1e-300, max_iter=300)
        row[name + "_us_per_it"] = 1e6 * t / rep.iterations
        del c
    print(json.dumps(row), flush=True)

for idx in (1, 2):
    cfg = make_config(idx)
    spec = solve_spec(cfg)
    row = {"config": idx}
    for name, lim in (("small", str(1 << 40)), ("chain", "0")):
        os.environ["PNRTE_SMALL_MAX"] = lim
        c = PnContext(build_tables(cfg.N), spec.res, spec.h)
        c.set_fields(spec)
        t, rep = timed(c, tol=cfg.tol, max_iter=cfg.max_iter)
        row[name] = {"seconds": t, "iterations": rep.iterations, "converged": rep.converged,
                     "normal_residual": rep.normal_residual}
        del c
    print(json.dumps(row), flush=True)

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench
for name, lim in (("small", str(1 << 40)), ("chain", "0"), ("default", None)):
    if lim is None:
        os.environ.pop("PNRTE_SMALL_MAX", None)
    else:
        os.environ["PNRTE_SMALL_MAX"] = lim
    print(json.dumps({"paper_workloads": name, **bench.paper_workloads(0)}), flush=True)
