"""Regenerate tests/golden/ from the LIVE reference (run in the container that
has /root/reference; the GPU box only reads the committed fixtures).

    PYTHONPATH=/root/reference/pkg/src python tools/make_goldens.py

Writes
  tables_N{1..7}.json  flattened StencilPrograms of compile_program(build_pn(N,3))
  cases.npz            per small case: reference CSR A, Q, A@x, A.T@x, colsum(A o A),
                       CGNR (plain + Jacobi) x / histories / counts, unstagger(x)
  neumann.npz/.json    bc="neumann" cases: reference CSR A, Q, A@x, A.T@x, colsum(A o A),
                       CGNR x / histories (python tools/make_goldens.py --neumann-only)
  cda.npz/.json        CDA programs (build_cda, 2-D and 3-D, both boundary conditions): reference
                       CSR A, Q, CGNR x / histories, unstagger (python tools/make_goldens.py --cda-only)
  configs.json         reference solves of configs 1 and 2: iteration count, sha256
                       of the solution bits, histories, residuals; input hashes
  perfcfg.json         reference solves of the config-3 and config-4 generators at 32^3
                       (sigma_t floor tau = 1, tol 1e-6): iteration count, sha256 of x,
                       Q, A, A@probe, A.T@probe, histories, residuals
                       (python tools/make_goldens.py --perfcfg-only)
The numpy/OpenBLAS configuration used is recorded (blas threads and kernel):
faithful-mode GPU runs must emulate that configuration to be bit-identical.
"""

import hashlib
import json
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

from pnrte.equations import build_pn  # noqa: E402
from pnrte.solver import assemble, solve_normal_cg, unstagger  # noqa: E402
from pnrte.stencil import compile_program  # noqa: E402
from threadpoolctl import threadpool_info  # noqa: E402

from cases import (CASES, CASES_2D, CASES_CDA, NEUMANN_CASES, case_inputs, cda_inputs, probe_vector,  # noqa: E402
                   rand_spec)
from paper_1807_00410_b200.problems import make_checkerboard  # noqa: E402
from paper_1807_00410_b200.configs import make_config  # noqa: E402
from paper_1807_00410_b200.program import tables_from_program, to_json  # noqa: E402

GOLD = ROOT / "tests" / "golden"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def blas():
    for info in threadpool_info():
        if info.get("internal_api") == "openblas":
            return {"threads": int(info["num_threads"]), "architecture": info.get("architecture"),
                    "version": info.get("version")}
    return {}


def neumann():
    arrs = {}
    meta = {"blas": blas(), "cases": {}}
    for name in NEUMANN_CASES:
        _, spec = case_inputs(name)
        prog = compile_program(build_pn(int(name.split("_")[1][1:]), spec.dim))
        sysm = assemble(prog, spec)
        A = sysm.A
        x = probe_vector(A.shape[0])
        arrs[f"{name}/indptr"] = A.indptr.astype(np.int64)
        arrs[f"{name}/indices"] = A.indices.astype(np.int32)
        arrs[f"{name}/data"] = A.data
        arrs[f"{name}/Q"] = sysm.Q
        arrs[f"{name}/Ax"] = A @ x
        arrs[f"{name}/Atx"] = A.T @ x
        arrs[f"{name}/jac"] = np.asarray(A.multiply(A).sum(axis=0)).ravel()
        xs, rep = solve_normal_cg(sysm, tol=1e-9, max_iter=300)
        arrs[f"{name}/cg0/x"] = xs
        arrs[f"{name}/cg0/nh"] = np.array(rep.normal_history)
        arrs[f"{name}/cg0/ph"] = np.array(rep.primal_history)
        meta["cases"][name] = {"cg0": {"iterations": rep.iterations, "converged": rep.converged,
                                       "normal_residual": rep.normal_residual,
                                       "primal_residual": rep.primal_residual}}
        print(name, meta["cases"][name], flush=True)
    np.savez_compressed(GOLD / "neumann.npz", **arrs)
    (GOLD / "neumann.json").write_text(json.dumps(meta, indent=1))


def cda():
    from pnrte.equations import build_cda
    arrs = {}
    meta = {"blas": blas(), "cases": {}}
    for name, dim, *_ in CASES_CDA:
        _, spec = cda_inputs(name)
        prog = compile_program(build_cda(dim))
        sysm = assemble(prog, spec)
        A = sysm.A
        x = probe_vector(A.shape[0])
        arrs[f"{name}/indptr"] = A.indptr.astype(np.int64)
        arrs[f"{name}/indices"] = A.indices.astype(np.int32)
        arrs[f"{name}/data"] = A.data
        arrs[f"{name}/Q"] = sysm.Q
        arrs[f"{name}/Ax"] = A @ x
        arrs[f"{name}/Atx"] = A.T @ x
        xs, rep = solve_normal_cg(sysm, tol=1e-10, max_iter=500)
        arrs[f"{name}/cg0/x"] = xs
        arrs[f"{name}/cg0/nh"] = np.array(rep.normal_history)
        arrs[f"{name}/cg0/ph"] = np.array(rep.primal_history)
        arrs[f"{name}/unstagger"] = unstagger(xs, prog, spec.res)
        meta["cases"][name] = {"cg0": {"iterations": rep.iterations, "converged": rep.converged,
                                       "normal_residual": rep.normal_residual}}
        print(name, meta["cases"][name], flush=True)
    np.savez_compressed(GOLD / "cda.npz", **arrs)
    (GOLD / "cda.json").write_text(json.dumps(meta, indent=1))


def perfcfg():
    """Reduced-size stand-ins of the performance configs, solved by the live
    reference exactly as configs.solve_spec sets them up (floor tau = 1)."""
    from paper_1807_00410_b200.configs import solve_spec
    out = {"blas": blas()}
    for idx, n in ((3, 32), (4, 32)):
        cfg = make_config(idx, n=n)
        spec = solve_spec(cfg)
        prog = compile_program(build_pn(cfg.N, 3))
        sysm = assemble(prog, spec)
        A = sysm.A
        x = probe_vector(A.shape[0])
        xs, rep = solve_normal_cg(sysm, tol=cfg.tol, max_iter=cfg.max_iter)
        out[f"cfg{idx}_n{n}"] = {
            "N": cfg.N, "res": list(spec.res), "tol": cfg.tol, "sigma_t_floor": cfg.floor,
            "iterations": rep.iterations, "converged": rep.converged,
            "normal_residual": rep.normal_residual, "primal_residual": rep.primal_residual,
            "x_sha256": sha(xs), "x_norm": float(np.linalg.norm(xs)), "Q_sha256": sha(sysm.Q),
            "A_data_sha256": sha(A.data), "A_indices_sha256": sha(A.indices.astype(np.int32)),
            "Ax_sha256": sha(A @ x), "Atx_sha256": sha(A.T.tocsr() @ x),
            "unstagger_sha256": sha(unstagger(xs, prog, spec.res)),
            "normal_history": rep.normal_history, "primal_history": rep.primal_history,
        }
        print(f"cfg{idx}_n{n}", rep.iterations, sha(xs)[:16], flush=True)
    (GOLD / "perfcfg.json").write_text(json.dumps(out, indent=1))


def main():
    if "--perfcfg-only" in sys.argv:
        perfcfg()
        return
    if "--neumann-only" in sys.argv:
        neumann()
        return
    if "--cda-only" in sys.argv:
        cda()
        return
    if "--tables-2d-only" in sys.argv:   # 2-D tables up to P5 (the paper's checkerboard runs)
        for N in (1, 2, 3, 4, 5):
            t = tables_from_program(compile_program(build_pn(N, 2)))
            (GOLD / f"tables_N{N}_2d.json").write_text(json.dumps(to_json(t), separators=(",", ":")))
        return
    neumann()
    cda()
    GOLD.mkdir(parents=True, exist_ok=True)
    for N in range(1, 8):
        t = tables_from_program(compile_program(build_pn(N, 3)))
        (GOLD / f"tables_N{N}.json").write_text(json.dumps(to_json(t), separators=(",", ":")))
    for N in (1, 2, 3, 4, 5):
        t = tables_from_program(compile_program(build_pn(N, 2)))
        (GOLD / f"tables_N{N}_2d.json").write_text(json.dumps(to_json(t), separators=(",", ":")))
    arrs = {}
    meta = {"blas": blas(), "cases": {}}
    todo = [(name, N, res, rand_spec(N, res, seed), 3) for name, N, res, seed in CASES]
    todo += [(name, N, (n, n), make_checkerboard(n), 2) for name, N, n in CASES_2D]
    for name, N, res, spec, dim in todo:
        prog = compile_program(build_pn(N, dim))
        sysm = assemble(prog, spec)
        A = sysm.A
        x = probe_vector(A.shape[0])
        arrs[f"{name}/indptr"] = A.indptr.astype(np.int64)
        arrs[f"{name}/indices"] = A.indices.astype(np.int32)
        arrs[f"{name}/data"] = A.data
        arrs[f"{name}/Q"] = sysm.Q
        arrs[f"{name}/Ax"] = A @ x
        arrs[f"{name}/Atx"] = A.T.tocsr() @ x
        arrs[f"{name}/jac"] = np.asarray(A.multiply(A).sum(axis=0)).ravel()
        m = {}
        for jac in (False, True):
            xs, rep = solve_normal_cg(sysm, tol=1e-9, max_iter=400, jacobi=jac)
            k = f"{name}/cg{int(jac)}"
            arrs[k + "/x"] = xs
            arrs[k + "/nh"] = np.array(rep.normal_history)
            arrs[k + "/ph"] = np.array(rep.primal_history)
            m[f"cg{int(jac)}"] = {"iterations": rep.iterations, "converged": rep.converged,
                                  "normal_residual": rep.normal_residual, "primal_residual": rep.primal_residual}
            if not jac:
                arrs[f"{name}/unstagger"] = unstagger(xs, prog, res)
        meta["cases"][name] = m
        print(name, m, flush=True)
    np.savez_compressed(GOLD / "cases.npz", **arrs)
    (GOLD / "cases.json").write_text(json.dumps(meta, indent=1))
    cfgs = {"blas": blas()}
    for idx in (1, 2):
        cfg = make_config(idx)
        sysm = assemble(compile_program(build_pn(cfg.N, 3)), cfg.spec)
        xs, rep = solve_normal_cg(sysm, tol=cfg.tol, max_iter=cfg.max_iter)
        cfgs[f"cfg{idx}"] = {
            "N": cfg.N, "res": list(cfg.spec.res), "tol": cfg.tol,
            "iterations": rep.iterations, "converged": rep.converged,
            "normal_residual": rep.normal_residual, "primal_residual": rep.primal_residual,
            "x_sha256": sha(xs), "Q_sha256": sha(sysm.Q), "A_data_sha256": sha(sysm.A.data),
            "x_norm": float(np.linalg.norm(xs)), "x_head": xs[:8].tolist(),
            "normal_history": rep.normal_history, "primal_history": rep.primal_history,
            "fields_sha256": {k: sha(np.asarray(v)) for k, v in sorted(cfg.spec.fields.items())},
        }
        print(f"cfg{idx}", rep.iterations, cfgs[f"cfg{idx}"]["x_sha256"][:16], flush=True)
    for idx, n in ((3, 32), (4, 32)):
        cfg = make_config(idx, n=n)
        cfgs[f"cfg{idx}_n{n}_fields_sha256"] = {k: sha(np.asarray(v)) for k, v in sorted(cfg.spec.fields.items())}
    (GOLD / "configs.json").write_text(json.dumps(cfgs, indent=1))


if __name__ == "__main__":
    main()
