"""Throughput of the widened rows on one GPU: device CSR
assembly + CSR operator (Neumann and Dirichlet config 2), general (CDA)
programs, and the post-processing kernels.  CSR apply roofline bytes:
12 B per stored entry (value + int32 column) + 8 B per row pointer + 16 B per
row (read x once, write y)."""
import json, pathlib, sys, time
from dataclasses import replace
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch
from paper_1807_00410_b200.configs import make_config
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext, assemble_general, fluence, reconstruct_radiance, unknown_order
from paper_1807_00410_b200.general import build_cda_program
from cases import rand_spec

PEAK = json.loads((pathlib.Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (pathlib.Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6650.0


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def csr_apply_line(name, csr, reps=50):
    n = csr.R_local
    nnz = csr.csr_export().nnz if n < 50_000_000 else None
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    ms_a = timed(lambda: csr.apply(x), reps)
    ms_t = timed(lambda: csr.apply(x, transpose=True), reps)
    b = 12 * nnz + 8 * (n + 1) + 16 * n
    return {"case": name, "rows": n, "nnz": nnz, "apply_ms": ms_a, "apply_T_ms": ms_t,
            "gunk_s": n / (ms_a / 1e3) / 1e9, "achieved_gbs": b / (ms_a / 1e3) / 1e9,
            "frac": b / (ms_a / 1e3) / 1e9 / PEAK}


out = []
# config 2 (P3 64^3): matrix-free vs device CSR (Dirichlet), Neumann CSR
cfg = make_config(2)
t = build_tables(cfg.N)
ctx = PnContext(t, cfg.spec.res, cfg.spec.h)
ctx.set_fields(cfg.spec)
ctx.bench(0, 5)
ms_mf = ctx.bench(0, 100)
line = {"case": "cfg2 matrix-free apply", "apply_ms": ms_mf, "gunk_s": ctx.R_local / (ms_mf / 1e3) / 1e9}
out.append(line)
print(json.dumps(line), flush=True)
for bc in ("dirichlet", "neumann"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    csr, q = ctx.assemble_csr(bc)
    torch.cuda.synchronize()
    t_asm = time.perf_counter() - t0
    line = csr_apply_line(f"cfg2 {bc} device CSR", csr)
    line["assemble_csr_s"] = t_asm
    csr.solve(tol=1e-6, max_iter=5, b=q)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = csr.solve(tol=1e-6, max_iter=20000, b=q)
    torch.cuda.synchronize()
    line.update({"solve_1e-6_s": time.perf_counter() - t0, "iterations": rep.iterations,
                 "converged": rep.converged})
    out.append(line)
    print(json.dumps(line), flush=True)
    del csr, q, x

# general (CDA) program, 3-D, 64^3 random heterogeneous medium
prog = build_cda_program(3)
spec = rand_spec(1, (64, 64, 64), 7)
for bc in ("dirichlet", "neumann"):
    sp = replace(spec, bc=bc)
    assemble_general(prog, sp)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    csr, q = assemble_general(prog, sp)
    torch.cuda.synchronize()
    t_asm = time.perf_counter() - t0
    line = csr_apply_line(f"CDA 3-D 64^3 {bc}", csr)
    line["assemble_general_s"] = t_asm
    csr.solve(tol=1e-6, max_iter=5, b=q)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = csr.solve(tol=1e-300, max_iter=200, b=q)
    torch.cuda.synchronize()
    line.update({"solve_200_iterations_s": time.perf_counter() - t0})
    out.append(line)
    print(json.dumps(line), flush=True)
    del csr, q, x

# post-processing on the config-2 solution
x, rep = ctx.solve(tol=1e-6, max_iter=20000)
coll = ctx.unstagger(x).reshape(*cfg.spec.res, t.U)
fl_ms = timed(lambda: fluence(coll), 20)
rng = np.random.default_rng(0)
lo = np.asarray(cfg.spec.origin)
hi = lo + np.asarray(cfg.spec.extent)
P, D = 65536, 128
pts = rng.uniform(lo, hi, size=(P, 3))
dirs = rng.normal(size=(D, 3))
dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
unk = unknown_order(t)
rr_ms = timed(lambda: reconstruct_radiance(coll, unk, cfg.spec, pts, dirs), 5)
line = {"case": "post-processing, cfg2 solution (P3 64^3)", "fluence_ms": fl_ms,
        "radiance_points": P, "radiance_directions": D, "radiance_ms": rr_ms,
        "radiance_pairs_per_s": P * D / (rr_ms / 1e3)}
out.append(line)
print(json.dumps(line), flush=True)
