"""Quick GPU probe: parity of every device entry point against the C oracle."""
import sys, time, pathlib
import numpy as np
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.problems import ProblemSpec, phase_fields
from paper_1807_00410_b200.program import q_name
from paper_1807_00410_b200.solver import PnContext
from paper_1807_00410_b200.configs import make_config
from oracle.oracle import StencilOracle

def rand_spec(N, res, seed):
    rng = np.random.default_rng(seed)
    st = rng.uniform(0.5, 20, res); ss = st * rng.uniform(0, 0.99, res)
    f = {"sigma_t": st, "sigma_s": ss}; f.update(phase_fields(0.6, N))
    for l in range(N + 1):
        for m in range(-l, l + 1):
            if rng.random() < 0.5: f[q_name(l, m)] = rng.normal(size=res)
    return ProblemSpec(dim=3, origin=(0, 0, 0), extent=tuple(r * 0.125 for r in res), res=res, fields=f)

def rel(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

ok = True
for N, res in [(1, (5, 6, 7)), (3, (4, 5, 6)), (7, (3, 4, 5)), (1, (32, 8, 6)), (3, (64, 9, 5)), (5, (32, 16, 4)), (7, (32, 8, 3))]:
    sp = rand_spec(N, res, N * 7 + res[0])
    t = build_tables(N); o = StencilOracle(t, sp)
    c = PnContext(t, res, sp.h); c.set_fields(sp)
    d, r = c.diag_rhs(); d = d.cpu().numpy(); r = r.cpu().numpy()
    x = np.random.default_rng(1).normal(size=o.R)
    line = [f"N={N} res={res}", f"diag {d.tobytes()==o.diag.tobytes()}", f"rhs {r.tobytes()==o.rhs.tobytes()}"]
    for tr in (0, 1):
        yf = c.apply(x, tr, "faithful").cpu().numpy(); yo = o.apply(x, bool(tr))
        ys = c.apply(x, tr, "fast").cpu().numpy()
        line.append(f"T{tr} faithful {yf.tobytes()==yo.tobytes()} fast {rel(ys, yo):.2e}")
    jd = c.jacobi_diag().cpu().numpy(); line.append(f"jac {jd.tobytes()==o.jacobi_diag().tobytes()}")
    for jac in (False, True):
        xf, rf = c.solve(tol=1e-9, max_iter=400, jacobi=jac, mode="faithful", blas_threads=8, blas_kernel=0)
        xo, ro = o.cgnr(tol=1e-9, max_iter=400, jacobi=jac, blas_threads=8, blas_kernel=0)
        xs, rs = c.solve(tol=1e-9, max_iter=400, jacobi=jac, mode="fast")
        line.append(f"solve jac={jac} it {rf.iterations}/{ro['iterations']}/{rs.iterations} bit {xf.cpu().numpy().tobytes()==xo.tobytes()} fast {rel(xs.cpu().numpy(), xo):.1e}")
    u = c.unstagger(x).cpu().numpy(); line.append(f"unstag {u.tobytes()==o.unstagger(x).tobytes()}")
    print(" | ".join(line), flush=True)

for idx in (1, 2):
    cfg = make_config(idx); t = build_tables(cfg.N)
    c = PnContext(t, cfg.spec.res, cfg.spec.h); c.set_fields(cfg.spec)
    t0 = time.time(); xf, rf = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="faithful", blas_threads=8, blas_kernel=0); t1 = time.time() - t0
    t0 = time.time(); xs, rs = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="fast"); t2 = time.time() - t0
    import hashlib
    print(f"cfg{idx}: faithful it={rf.iterations} sha={hashlib.sha256(xf.cpu().numpy().tobytes()).hexdigest()[:16]} {t1:.2f}s | fast it={rs.iterations} rel={rel(xs.cpu().numpy(), xf.cpu().numpy()):.2e} {t2:.3f}s", flush=True)
    for what in (0, 1):
        ms = c.bench(what, 50); ms = c.bench(what, 200)
        R = c.R_local
        print(f"   bench what={what}: {ms*1e3:.1f} us -> {R/ms/1e6 * (2 if what else 1):.1f} Gunk/s", flush=True)
