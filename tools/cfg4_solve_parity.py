"""Solve-level parity at full-size config 4 (P7 256^3, tau = 1, tol 1e-6), a
one-off too long for the test suite (~35 min per faithful solve): the device's
faithful mode -- the reference's arithmetic, bit-identical to the reference /
oracle wherever they can run, including this config's assembly and products --
stands in for the reference, which cannot assemble this system in host memory.

  faithful SkylakeX x 8   -> iterations, sha256 of x and of both histories
  faithful pairwise x 8   -> delta = the trajectory's sensitivity to the dot order
  fast                    -> iterations (+-1), field distance (<= max(1e-8, 4 delta)),
                             residual histories (first 10 entries within 1e-6)

    python tools/cfg4_solve_parity.py [--config 4] [--n 0] [--out gpurun_out/r02_cfg4_solve_parity.json]
"""
import argparse, hashlib, json, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--out", default="gpurun_out/r02_cfg4_solve_parity.json")
ap.add_argument("--skip-delta", action="store_true")
ap.add_argument("--skip-fast", action="store_true")
ap.add_argument("--alts", default="8:2", help="comma list of threads:kernel dot orders for the delta probes")
a = ap.parse_args()


def sha(t):
    h = hashlib.sha256()
    flat = t.reshape(-1)
    step = 1 << 27
    for o in range(0, flat.numel(), step):
        h.update(flat[o:o + step].cpu().numpy().tobytes())
    return h.hexdigest()


def rel(x, y):
    return float(torch.linalg.vector_norm(x - y) / torch.linalg.vector_norm(y))


cfg = make_config(a.config, **({"n": a.n} if a.n else {}))
spec = solve_spec(cfg)
c = PnContext(build_tables(cfg.N), spec.res, spec.h)
c.set_fields(spec)
out = {"config": a.config, "res": list(spec.res), "N": cfg.N, "tol": cfg.tol, "sigma_t_floor": cfg.floor}


def dump():
    pathlib.Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    pathlib.Path(a.out).write_text(json.dumps(out))
    print(json.dumps({k: v for k, v in out.items() if not k.endswith("history")}), flush=True)


xf = rf = None
if not a.skip_fast:
    t0 = time.perf_counter()
    xf, rf = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="fast")
    torch.cuda.synchronize()
    out["fast"] = {"iterations": rf.iterations, "converged": rf.converged, "normal_residual": rf.normal_residual,
                   "seconds": time.perf_counter() - t0, "x_sha256": sha(xf)}
    dump()
t0 = time.perf_counter()
xs, rs = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="faithful", blas_threads=8, blas_kernel=0)
torch.cuda.synchronize()
out["faithful_skx8"] = {"iterations": rs.iterations, "converged": rs.converged, "normal_residual": rs.normal_residual,
                        "seconds": time.perf_counter() - t0, "x_sha256": sha(xs),
                        "normal_history_sha256": hashlib.sha256(np.array(rs.normal_history).tobytes()).hexdigest(),
                        "primal_history_sha256": hashlib.sha256(np.array(rs.primal_history).tobytes()).hexdigest()}
if xf is not None:
    nf, ns = np.array(rf.normal_history), np.array(rs.normal_history)
    k = min(len(nf), len(ns))
    out["fast_vs_faithful"] = {"iteration_difference": rf.iterations - rs.iterations, "field_rel_l2": rel(xf, xs),
                               "normal_history_first10_max_rel": float(np.max(np.abs(nf[:10] / ns[:10] - 1))),
                               "normal_history_max_rel": float(np.max(np.abs(nf[:k] / ns[:k] - 1)))}
out["faithful_normal_history"] = rs.normal_history
dump()
del xf
if not a.skip_delta:
    deltas = {}
    for spec_ in a.alts.split(","):
        T, kn = (int(v) for v in spec_.split(":"))
        t0 = time.perf_counter()
        xa, ra = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="faithful", blas_threads=T, blas_kernel=kn)
        torch.cuda.synchronize()
        name = {0: "skylakex", 1: "haswell", 2: "pairwise"}[kn] + f"_x{T}"
        deltas[name] = rel(xa, xs)
        out["faithful_" + name] = {"iterations": ra.iterations, "seconds": time.perf_counter() - t0,
                                   "delta_field_rel_l2": deltas[name]}
        del xa
        dump()
    if "fast_vs_faithful" in out:
        d = max(deltas.values())
        out["verdict"] = {"iterations_within_1": abs(out["fast_vs_faithful"]["iteration_difference"]) <= 1,
                          "delta_max": d, "field_bound": max(1e-8, 4 * d),
                          "field_within_bound": out["fast_vs_faithful"]["field_rel_l2"] <= max(1e-8, 4 * d)}
        dump()
