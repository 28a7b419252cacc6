"""Config 5 (P5, 512^3, 4.83e9 unknowns, 8 GPUs only) on one GPU: the per-rank
work of one interior z-slab at world = 8 / 4 / 2 (its halos are not
exchanged; the apply and iteration traffic are those of one rank), plus the
weak-scaling companion at k = 1 (256^3 P5, same generator) solved for the
fixed 200 iterations of BASELINE.json."""
import json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config, config3
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext

t0 = time.perf_counter()
cfg = make_config(5)
print(f"cfg5 generated in {time.perf_counter() - t0:.1f}s", file=sys.stderr, flush=True)
t = build_tables(cfg.N)
nx, ny, nz = cfg.spec.res
U = (cfg.N + 1) ** 2
R = nx * ny * nz * U
for world in (8, 4, 2):
    nzl = nz // world
    rank = world // 2
    c = PnContext(t, cfg.spec.res, cfg.spec.h, z0=rank * nzl, nz_local=nzl, rank=rank, world=world)
    c.set_fields(cfg.spec)
    c.bench(0, 3)
    ms = c.bench(0, 20)
    c.bench(1, 2)
    it = c.bench(1, 10)
    nvox_l = nx * ny * nzl
    gbs = 8 * nvox_l * (2 * U + 2) / (ms / 1e3) / 1e9
    print(json.dumps({"config": 5, "world": world, "nz_local": nzl, "apply_ms_per_rank": ms,
                      "achieved_gbs_per_rank": gbs, "cg_iter_ms_per_rank": it,
                      "est_job_gunk_s_apply": R / (ms / 1e3) / 1e9,
                      "est_200_iterations_s": 200 * it / 1e3}), flush=True)
    del c
    torch.cuda.empty_cache()
del cfg

# weak-scaling companion, k = 1: 256^3 P5 on one GPU, fixed 200 iterations
w = config3(n=256, base_period=64)
c = PnContext(build_tables(w.N), w.spec.res, w.spec.h)
c.set_fields(w.spec)
c.bench(0, 3)
ms = c.bench(0, 20)
c.solve(tol=1e-300, max_iter=5)
torch.cuda.synchronize()
t0 = time.perf_counter()
x, rep = c.solve(tol=1e-300, max_iter=200)
torch.cuda.synchronize()
ts = time.perf_counter() - t0
Rw = 256 ** 3 * U
print(json.dumps({"config": "5-weak k=1 (256^3 P5)", "apply_ms": ms, "gunk_s_apply": Rw / (ms / 1e3) / 1e9,
                  "solve_200_iterations_s": ts, "iterations": rep.iterations,
                  "gunk_s_2_applies_per_iteration": 2 * Rw * rep.iterations / ts / 1e9}), flush=True)
