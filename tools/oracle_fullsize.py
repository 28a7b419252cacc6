"""Full-size oracle pins for configs 3 and 4 (run here, on the CPU container;
the GPU box only reads the committed tests/golden/fullsize.json).

    python tools/oracle_fullsize.py [cfg4] [cfg3]

The C oracle (oracle/pn_oracle.c) is the reference's solve path restated op
for op and pinned bit for bit to the live reference (tests/test_oracle.py);
at these sizes the reference itself does not fit in host RAM (SURVEY.md
s8a row a5: config 3+ out of RAM), so the oracle stands in for it.

  cfg4  P7 256^3: sha256 of the assembled diagonal and RHS
        (solver.py:96-186), of A x and A^T x for the probe vector
        x = default_rng(99).normal(size=R) (tests/cases.probe_vector)
  cfg3  P5 128^3 with the sigma_t floor tau = 1 (configs.solve_spec): the
        whole CGNR solve to 1e-6 (solver.py:189-257) under the OpenBLAS
        configuration of the committed fixtures (8 threads, SkylakeX):
        iteration count, sha256 of x, both residual histories
"""

import hashlib
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle.oracle import StencilOracle  # noqa: E402
from paper_1807_00410_b200.configs import make_config, solve_spec  # noqa: E402
from paper_1807_00410_b200.program import build_tables  # noqa: E402

OUT = ROOT / "tests" / "golden" / "fullsize.json"


def sha(a):
    h = hashlib.sha256()
    a = np.ascontiguousarray(a)
    mv = memoryview(a.reshape(-1).view(np.uint8))
    step = 1 << 28
    for o in range(0, len(mv), step):
        h.update(mv[o:o + step])
    return h.hexdigest()


def load():
    return json.loads(OUT.read_text()) if OUT.exists() else {}


def save(d):
    OUT.write_text(json.dumps(d, indent=1))


def cfg4():
    cfg = make_config(4)
    t0 = time.time()
    o = StencilOracle(build_tables(cfg.N), cfg.spec)
    out = {"N": cfg.N, "res": list(cfg.spec.res), "setup_s": time.time() - t0,
           "diag_sha256": sha(o.diag), "rhs_sha256": sha(o.rhs),
           "rhs_nonzeros": int(np.count_nonzero(o.rhs)), "diag_sum": float(np.sum(o.diag))}
    print("cfg4 setup", out, flush=True)
    x = np.random.default_rng(99).normal(size=o.R)
    for tr in (0, 1):
        t0 = time.time()
        y = o.apply(x, transpose=bool(tr))
        out[f"A{'t' if tr else ''}x_sha256"] = sha(y)
        out[f"A{'t' if tr else ''}x_norm"] = float(np.linalg.norm(y))
        print("cfg4 apply", tr, time.time() - t0, flush=True)
        del y
    d = load()
    d["cfg4"] = out
    save(d)


def cfg3():
    cfg = make_config(3)
    spec = solve_spec(cfg)
    o = StencilOracle(build_tables(cfg.N), spec)
    t0 = time.time()
    x, rep = o.cgnr(tol=cfg.tol, max_iter=cfg.max_iter, blas_threads=8, blas_kernel=0)
    out = {"N": cfg.N, "res": list(spec.res), "tol": cfg.tol, "sigma_t_floor": cfg.floor,
           "blas": {"threads": 8, "architecture": "SkylakeX"},
           "iterations": rep["iterations"], "converged": rep["converged"],
           "normal_residual": rep["normal_residual"], "primal_residual": rep["primal_residual"],
           "x_sha256": sha(x), "x_norm": float(np.linalg.norm(x)),
           "diag_sha256": sha(o.diag), "rhs_sha256": sha(o.rhs),
           "normal_history": rep["normal_history"], "primal_history": rep["primal_history"],
           "solve_s": time.time() - t0}
    print("cfg3", rep["iterations"], out["x_sha256"][:16], out["solve_s"], flush=True)
    d = load()
    d["cfg3"] = out
    save(d)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg4", "cfg3"]
    for w in which:
        globals()[w]()
