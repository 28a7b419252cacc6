"""A/B check of two builds of the library (PNRTE_LIB): fast-mode solve of a
config (and a small loopback slab group) -> sha256 of the solution and the
residual histories, for bit-identity of a change that must not alter results."""
import hashlib, json, os, pathlib, sys
os.environ["PNRTE_SMALL_MAX"] = "0"   # the launch chain (plane sums + scalar steps)
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
out = {}
for idx, it in ((1, 400), (2, 300)):
    cfg = make_config(idx)
    spec = solve_spec(cfg)
    c = PnContext(build_tables(cfg.N), spec.res, spec.h)
    c.set_fields(spec)
    for jac in (False, True):
        x, rep = c.solve(tol=1e-7, max_iter=it, jacobi=jac)
        h = hashlib.sha256(x.cpu().numpy().tobytes() + np.array(rep.normal_history).tobytes()
                           + np.array(rep.primal_history).tobytes()).hexdigest()
        out[f"cfg{idx}_jac{int(jac)}"] = [rep.iterations, h[:16]]
print(json.dumps(out))
