"""Per-kernel and per-iteration cost on the small (L2-sized) configurations:
apply, apply + fused reductions, r update, x/p update, the stream-launched
iteration and the graph-replayed solve (ms per iteration)."""
import argparse, json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3")
ap.add_argument("--iters", type=int, default=200)
a = ap.parse_args()
names = {0: "apply", 2: "apply+red", 4: "r_update", 5: "xp_update", 1: "iteration(stream)"}
for idx in [int(v) for v in a.configs.split(",")]:
    cfg = make_config(idx)
    spec = solve_spec(cfg)
    c = PnContext(build_tables(cfg.N), spec.res, spec.h)
    c.set_fields(spec)
    out = {"config": idx}
    for w, n in names.items():
        c.bench(w, 5)
        out[n + "_us"] = 1e3 * c.bench(w, 100)
    c.solve(tol=1e-300, max_iter=8)
    ts = []
    for n in (a.iters // 2, a.iters):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        c.solve(tol=1e-300, max_iter=n)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    out["solve_us_per_it"] = 1e6 * (ts[1] - ts[0]) / (a.iters - a.iters // 2)
    out["solve_fixed_ms"] = 1e3 * (2 * ts[0] - ts[1])
    print(json.dumps(out), flush=True)
    del c
    torch.cuda.empty_cache()
