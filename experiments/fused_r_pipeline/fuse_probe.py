"""A/B of the fused residual update + A^T apply (k_seg_fr, PNRTE_SEG_FUSE_R=1)
against the launch chain: bit-identity of fixed-iteration fast solves (solution
and both histories) on small grids with the bulk path forced, then a config's
CG iteration time, a sustained fixed-iteration solve and its hashes.

    python experiments/fused_r_pipeline/fuse_probe.py  (with the patch applied) [--config 4] [--n 0] [--iters 300] [--skip-check]
"""
import argparse
import hashlib
import json
import os
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from cases import rand_spec  # noqa: E402
from paper_1807_00410_b200.configs import make_config, solve_spec  # noqa: E402
from paper_1807_00410_b200.program import build_tables  # noqa: E402
from paper_1807_00410_b200.solver import PnContext  # noqa: E402


def ctx(N, spec, fuse):
    os.environ["PNRTE_SEG_FUSE_R"] = str(fuse)
    c = PnContext(build_tables(N), spec.res, spec.h)
    c.set_fields(spec)
    os.environ.pop("PNRTE_SEG_FUSE_R")
    return c


def digest(x, rep):
    h = hashlib.sha256()
    h.update(x.cpu().numpy().tobytes())
    h.update(np.array(rep.normal_history).tobytes())
    h.update(np.array(rep.primal_history).tobytes())
    return h.hexdigest()[:16]


def check():
    os.environ["PNRTE_SEG_BULK"] = "1"
    os.environ["PNRTE_SMALL_MAX"] = "0"
    ok = True
    for N, res in ((1, (64, 9, 6)), (2, (96, 7, 5)), (3, (64, 9, 6)), (4, (32, 10, 7)), (6, (32, 6, 9)), (7, (64, 9, 6)),
                   (7, (40, 11, 5)), (3, (80, 13, 4)), (7, (128, 37, 20)), (7, (64, 70, 9)), (4, (96, 130, 5))):
        spec = rand_spec(N, res, 40 + N)
        d = []
        for fuse in (0, 1):
            c = ctx(N, spec, fuse)
            h = []
            for jac in (False, True):
                xs, rep = c.solve(tol=1e-30, max_iter=40, jacobi=jac)
                h.append(digest(xs, rep))
            xs, rep = c.solve(tol=1e-7, max_iter=4000)
            h.append(digest(xs, rep) + f":{rep.iterations}")
            d.append(h)
            del c
        print(json.dumps({"check": f"P{N} {res}", "chain": d[0], "fused": d[1], "same": d[0] == d[1]}), flush=True)
        ok = ok and d[0] == d[1]
    os.environ.pop("PNRTE_SEG_BULK")
    os.environ.pop("PNRTE_SMALL_MAX")
    return ok


def timing(cfg_id, n, iters):
    cfg = make_config(cfg_id, **({"n": n} if n else {}))
    spec = solve_spec(cfg)
    for fuse, D in [(0, 0)] + [(1, int(d)) for d in os.environ.get("FUSE_DS", "6").split(",")]:
        if D:
            os.environ["PNRTE_SEG_FUSE_D"] = str(D)
        c = ctx(cfg.N, spec, fuse)
        out = {"config": cfg_id, "res": list(spec.res), "fused": fuse, "D": D}
        c.bench(1, 3)
        out["cg_iteration_ms_bench"] = round(c.bench(1, 30), 4)
        c.solve(tol=1e-30, max_iter=5)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = c.solve(tol=1e-30, max_iter=iters)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out["solve_ms_per_iteration"] = round(1e3 * dt / rep.iterations, 4)
        out["iterations"] = rep.iterations
        out["digest"] = digest(x, rep)
        print(json.dumps(out), flush=True)
        del c, x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--iters", type=int, default=300)
    ap.add_argument("--skip-check", action="store_true")
    a = ap.parse_args()
    if not a.skip_check and not check():
        print(json.dumps({"error": "fused kernel differs from the launch chain"}))
        sys.exit(1)
    timing(a.config, a.n, a.iters)
