"""Time-to-residual (fast mode, device-resident inputs) for configs 1-4."""
import argparse, json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,4")
ap.add_argument("--max-iter", type=int, default=20000)
ap.add_argument("--jacobi", action="store_true", help="the reference's jacobi=True option (solver.py:189)")
a = ap.parse_args()
for idx in [int(v) for v in a.configs.split(",")]:
    cfg = make_config(idx)
    spec = solve_spec(cfg)
    c = PnContext(build_tables(cfg.N), spec.res, spec.h)
    t0 = time.perf_counter(); c.set_fields(spec); torch.cuda.synchronize(); t_setup = time.perf_counter() - t0
    c.solve(tol=cfg.tol, max_iter=5, jacobi=a.jacobi)   # warm-up as in bench.py: module loading, graph capture
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = c.solve(tol=cfg.tol, max_iter=min(cfg.max_iter, a.max_iter), jacobi=a.jacobi)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(json.dumps({"config": idx, "N": cfg.N, "res": spec.res, "floor": cfg.floor, "tol": cfg.tol, "jacobi": a.jacobi,
                      "iterations": rep.iterations, "converged": rep.converged,
                      "normal_residual": rep.normal_residual, "primal_residual": rep.primal_residual,
                      "seconds": t, "ms_per_iteration": 1e3 * t / max(rep.iterations, 1), "setup_s": t_setup}), flush=True)
    del c, x
    torch.cuda.empty_cache()
