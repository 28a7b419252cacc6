"""Time to residual 1e-6 against the graph batch length (iterations between
host polls of the device stop flag), configs 1-3."""
import json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
for idx in (1, 2, 3):
    cfg = make_config(idx)
    spec = solve_spec(cfg)
    c = PnContext(build_tables(cfg.N), spec.res, spec.h)
    c.set_fields(spec)
    for ce in (0, 4, 8, 16, 32, 64):
        c.solve(tol=cfg.tol, max_iter=5, check_every=ce)
        best = None
        for rep_ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, rep = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, check_every=ce)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        print(json.dumps({"config": idx, "check_every": ce, "iterations": rep.iterations, "best_of_3_s": best}), flush=True)
    del c
    torch.cuda.empty_cache()
