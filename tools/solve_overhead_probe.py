"""Fixed (per-solve) overhead of PnContext.solve on config 1: wall time of
solves with 0 / 1 / 16 iterations and a cProfile of the Python side."""
import cProfile, pstats, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
cfg = make_config(1)
spec = solve_spec(cfg)
c = PnContext(build_tables(cfg.N), spec.res, spec.h)
c.set_fields(spec)
for n in (0, 1, 16, 0, 1, 16):
    c.solve(tol=1e-300, max_iter=max(n, 1))
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        x, rep = c.solve(tol=1e-300, max_iter=n)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"max_iter={n}: median {1e3 * ts[10]:.3f} ms, min {1e3 * ts[0]:.3f} ms, C wall {1e3 * rep.wall_time:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    c.solve(tol=1e-300, max_iter=16)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(15)
