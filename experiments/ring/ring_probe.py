"""A/B of the k_seg grid against the persistent ring kernel (PNRTE_SEG_RING=1)
in one library build: bit-identity of applies and fixed-iteration fast solves on
small grids (bulk path forced), then config-4 (or --config) apply timings on
dense / zero operands, burst and sustained with NVML clocks, and the CG iteration.

    python experiments/ring/ring_probe.py  (with the patch applied) [--config 4] [--n 256] [--skip-check]
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
sys.path.insert(0, str(ROOT / "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from cases import probe_vector, rand_spec  # noqa: E402
from paper_1807_00410_b200.configs import make_config  # noqa: E402
from paper_1807_00410_b200.program import build_tables  # noqa: E402
from paper_1807_00410_b200.solver import PnContext  # noqa: E402
from power_probe import Nvml  # noqa: E402


def ctx(N, spec, ring):
    os.environ["PNRTE_SEG_RING"] = str(ring)
    c = PnContext(build_tables(N), spec.res, spec.h)
    c.set_fields(spec)
    os.environ.pop("PNRTE_SEG_RING")
    return c


def check():
    os.environ["PNRTE_SEG_BULK"] = "1"
    os.environ["PNRTE_SMALL_MAX"] = "0"
    ok = True
    for N, res in ((1, (64, 9, 6)), (2, (96, 7, 5)), (3, (64, 9, 6)), (4, (32, 10, 7)), (5, (64, 9, 6)), (6, (32, 6, 9)),
                   (7, (64, 9, 6)), (7, (40, 11, 5)), (5, (80, 13, 4)), (7, (128, 37, 20))):
        spec = rand_spec(N, res, 40 + N)
        d = []
        for ring in (0, 1):
            c = ctx(N, spec, ring)
            x = probe_vector(c.R_local)
            h = hashlib.sha256()
            for tr in (0, 1):
                h.update(c.apply(x, tr).cpu().numpy().tobytes())
            for jac in (False, True):
                xs, rep = c.solve(tol=1e-30, max_iter=25, jacobi=jac)
                h.update(xs.cpu().numpy().tobytes() + np.array(rep.normal_history).tobytes())
            d.append(h.hexdigest()[:16])
            del c
        print(json.dumps({"check": f"P{N} {res}", "grid": d[0], "ring": d[1], "same": d[0] == d[1]}), flush=True)
        ok = ok and d[0] == d[1]
    os.environ.pop("PNRTE_SEG_BULK")
    os.environ.pop("PNRTE_SMALL_MAX")
    return ok


def timing(cfg_id, n, rings):
    cfg = make_config(cfg_id, **({"n": n} if n else {}))
    for ring in rings:
        c = ctx(cfg.N, cfg.spec, ring)
        R = c.R_local
        out = {"config": cfg_id, "res": list(cfg.spec.res), "ring": ring}
        c.bench(0, 5)
        with Nvml() as mon:
            for label, what, reps in (("zero_burst", 6, 40), ("dense_burst", 7, 40), ("dense_sustained", 7, 600)):
                c.bench(what, 0)
                time.sleep(1.0)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ms = c.bench(0, reps)
                t1 = time.perf_counter()
                out[label] = {"ms": round(ms, 4), "gunk_s": round(R / ms / 1e6, 1), **mon.window(t0, t1)}
            c.bench(7, 0)
            time.sleep(1.0)
            c.bench(1, 3)
            out["cg_iteration_ms"] = c.bench(1, 40)
        print(json.dumps(out), flush=True)
        del c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--skip-check", action="store_true")
    ap.add_argument("--rings", default="0,1")
    a = ap.parse_args()
    if not a.skip_check and not check():
        print(json.dumps({"error": "ring kernel differs from the grid kernel"}))
        sys.exit(1)
    timing(a.config, a.n, [int(r) for r in a.rings.split(",")])
