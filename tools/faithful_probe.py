"""Cost of the faithful (reference-arithmetic) solve at full size: ms per
iteration of a fixed-iteration config-3 (or --config) solve under several
OpenBLAS emulations (threads, kernel: 0 SkylakeX, 1 Haswell)."""
import argparse, json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
cfg = make_config(a.config, **({"n": a.n} if a.n else {}))
spec = solve_spec(cfg)
c = PnContext(build_tables(cfg.N), spec.res, spec.h)
c.set_fields(spec)
for T, k in ((8, 0), (8, 1), (1, 1), (1, 0)):
    c.solve(tol=1e-30, max_iter=2, mode="faithful", blas_threads=T, blas_kernel=k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = c.solve(tol=1e-30, max_iter=a.iters, mode="faithful", blas_threads=T, blas_kernel=k)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"config": a.config, "res": list(spec.res), "blas_threads": T, "blas_kernel": k,
                      "iterations": rep.iterations, "ms_per_iteration": round(1e3 * dt / rep.iterations, 3)}), flush=True)
