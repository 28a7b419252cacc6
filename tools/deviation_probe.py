"""Distance of the fast solve from the reference-arithmetic (faithful) solve at
tol 1e-6, per config: iterations of both, relative L2 of the field difference,
and the same for an alternative dot order (the reference's own sensitivity).

    python tools/deviation_probe.py [--cases 1,2,3n32,4n32,3]
"""
import argparse, json, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="1,2,3n32,4n32,3n64,4n64,3")
a = ap.parse_args()


def rel(x, y):
    return float(torch.linalg.vector_norm(x - y) / torch.linalg.vector_norm(y))


for case in a.cases.split(","):
    idx, _, n = case.partition("n")
    cfg = make_config(int(idx), **({"n": int(n)} if n else {}))
    spec = solve_spec(cfg)
    c = PnContext(build_tables(cfg.N), spec.res, spec.h)
    c.set_fields(spec)
    xs, rs = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="faithful", blas_threads=8, blas_kernel=0)
    xf, rf = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="fast")
    out = {"case": case, "res": list(spec.res), "N": cfg.N, "faithful_iterations": rs.iterations,
           "fast_iterations": rf.iterations, "fast_vs_faithful": rel(xf, xs)}
    for T, k in ((8, 2), (64, 0)):
        xa, ra = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="faithful", blas_threads=T, blas_kernel=k)
        out[f"delta_T{T}_k{k}"] = [ra.iterations, rel(xa, xs)]
        del xa
    print(json.dumps(out), flush=True)
    del c, xs, xf
    torch.cuda.empty_cache()
