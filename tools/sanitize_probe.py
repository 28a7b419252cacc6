"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
the segmented operator on both staging paths (bulk TMA + mbarrier, cp.async)
with and without fused reductions, the cooperative one-launch solve
(k_cg_small), the graph-replayed chain, and the faithful table operator.

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from cases import probe_vector, rand_spec  # noqa: E402
from paper_1807_00410_b200.program import build_tables  # noqa: E402
from paper_1807_00410_b200.solver import PnContext  # noqa: E402


def run(N, res, bulk):
    os.environ["PNRTE_SEG_BULK"] = bulk
    spec = rand_spec(N, res, 5 + N)
    c = PnContext(build_tables(N), res, spec.h)
    c.set_fields(spec)
    x = probe_vector(c.R_local)
    ys = [c.apply(x, tr, "fast") for tr in (0, 1)]
    c.bench(2, 2)                                              # fused ww / zz reductions
    os.environ["PNRTE_SMALL_MAX"] = "0"
    _, r1 = c.solve(tol=1e-300, max_iter=6, jacobi=True)      # graph-replayed chain (Jacobi)
    os.environ.pop("PNRTE_SMALL_MAX")
    _, r2 = c.solve(tol=1e-300, max_iter=6)                   # one-launch cooperative solve when small
    yf = c.apply(x, 0, "faithful")
    torch.cuda.synchronize()
    print(f"N={N} res={res} bulk={bulk}: |Ax|={float(ys[0].norm()):.6e} |A^Tx|={float(ys[1].norm()):.6e} "
          f"it={r1.iterations},{r2.iterations} faithful={float(yf.norm()):.6e}", flush=True)


if __name__ == "__main__":
    for N in (1, 3, 7):
        for bulk in ("1", "0"):
            run(N, (64, 9, 5), bulk)
    print("sanitize probe done")
