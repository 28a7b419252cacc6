"""Per-rank apply time of config 4 at world = 1, 2, 4, 8: one interior z-slab
context on this GPU (its halos are not exchanged; the work and memory traffic
are those of one rank).  Estimates strong-scaling compute efficiency."""
import json, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_1807_00410_b200.configs import make_config
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
cfg = make_config(4)
t = build_tables(cfg.N)
R = 256 ** 3 * 64
base = None
for world in (1, 2, 4, 8):
    nzl = 256 // world
    rank = world // 2
    c = PnContext(t, cfg.spec.res, cfg.spec.h, z0=rank * nzl, nz_local=nzl, rank=rank, world=world)
    c.set_fields(cfg.spec)
    c.bench(0, 3)
    ms = c.bench(0, 20)
    it = c.bench(1, 5) if world > 1 else c.bench(1, 5)
    base = base or ms
    print(json.dumps({"world": world, "nz_local": nzl, "apply_ms_per_rank": ms, "cg_iter_ms_per_rank": it,
                      "est_job_gunk_s": R / (ms / 1e3) / 1e9, "compute_efficiency": base / (world * ms)}), flush=True)
    del c
