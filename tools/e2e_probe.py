"""Where the end-to-end drop-in call spends its time (config 4, 50 fixed
iterations): context creation, field upload + assembly, solve, unstagger,
D2H of the collocated grid, teardown -- each stage timed after a device sync.

    python tools/e2e_probe.py [--iters 50]
"""
import argparse
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1807_00410_b200.configs import make_config  # noqa: E402
from paper_1807_00410_b200.program import build_tables  # noqa: E402
from paper_1807_00410_b200.solver import PnContext  # noqa: E402

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from bench import pinned_spec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = make_config(4)
    spec, keep = pinned_spec(cfg.spec)
    nx, ny, nz = spec.res
    U = (cfg.N + 1) ** 2
    out = torch.empty((nx, ny, nz, U), dtype=torch.float64, pin_memory=True)
    t = build_tables(cfg.N)
    for rep in range(a.reps):
        st = {}

        def mark(name, t0):
            torch.cuda.synchronize()
            st[name] = time.perf_counter() - t0
            return time.perf_counter()

        t0 = time.perf_counter()
        c = PnContext(t, spec.res, spec.h)
        t0 = mark("create", t0)
        c.set_fields(spec)
        t0 = mark("set_fields", t0)
        x, r = c.solve(tol=1e-300, max_iter=a.iters)
        t0 = mark("solve", t0)
        coll = c.unstagger(x)
        t0 = mark("unstagger", t0)
        out.copy_(coll)
        t0 = mark("d2h", t0)
        del coll, x
        del c
        t0 = mark("destroy", t0)
        torch.cuda.empty_cache()
        t0 = mark("empty_cache", t0)
        st["total"] = sum(st.values())
        st["rep"] = rep
        st["solve_wall_reported"] = r.wall_time
        print(json.dumps(st), flush=True)


if __name__ == "__main__":
    main()
