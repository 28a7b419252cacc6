"""Neumann boundaries (bc="neumann", solver.py:133-135,146-147) on the device:
pn_assemble_csr builds the reference's coo->csr system on the GPU (clipped
writes, summed duplicates, unpinned RHS) and the CSR operator solves it.
Checked against the reference fixtures (tests/golden/neumann.npz) and the
oracle (or_csr_bc)."""

from dataclasses import replace

import numpy as np
import pytest

from cases import NEUMANN_CASES, case_inputs, probe_vector, rand_spec
from oracle.oracle import StencilOracle
from paper_1807_00410_b200.program import build_tables

pytestmark = pytest.mark.gpu

FIX_BLAS = (8, 0)


@pytest.fixture(scope="module")
def systems():
    from paper_1807_00410_b200.solver import assemble
    out = {}
    for name in NEUMANN_CASES:
        tables, spec = case_inputs(name)
        out[name] = assemble(tables, spec)
    return out


@pytest.mark.parametrize("case", NEUMANN_CASES)
def test_neumann_assembly_bit_exact(case, systems, golden):
    s, g = systems[case], golden["neumann"]
    A = s.A.to_scipy()
    assert np.array_equal(A.indptr, g[f"{case}/indptr"])
    assert np.array_equal(A.indices, g[f"{case}/indices"])
    assert A.data.tobytes() == g[f"{case}/data"].tobytes()
    assert s.Q.tobytes() == g[f"{case}/Q"].tobytes()
    At = s.A.T.to_scipy()
    assert (At != A.T.tocsr()).nnz == 0


@pytest.mark.parametrize("case", NEUMANN_CASES)
def test_neumann_products(case, systems, golden):
    s, g = systems[case], golden["neumann"]
    x = probe_vector(s.A.shape[0])
    assert s.A.matvec(x, mode="faithful").tobytes() == g[f"{case}/Ax"].tobytes()
    assert s.A.T.matvec(x, mode="faithful").tobytes() == g[f"{case}/Atx"].tobytes()
    np.testing.assert_allclose(s.A @ x, g[f"{case}/Ax"], rtol=1e-12, atol=1e-12 * np.abs(g[f"{case}/Ax"]).max())
    jac = s.A.ctx.jacobi_diag().cpu().numpy()
    assert jac.tobytes() == g[f"{case}/jac"].tobytes()


@pytest.mark.parametrize("case", NEUMANN_CASES)
def test_neumann_cgnr_faithful_bit_exact(case, systems, golden):
    from paper_1807_00410_b200.solver import solve_normal_cg
    s, g = systems[case], golden["neumann"]
    meta = golden["neumann_meta"]["cases"][case]["cg0"]
    x, rep = solve_normal_cg(s, tol=1e-9, max_iter=300, mode="faithful", blas_threads=FIX_BLAS[0],
                             blas_kernel=FIX_BLAS[1])
    assert rep.iterations == meta["iterations"] and rep.converged == meta["converged"]
    assert x.tobytes() == g[f"{case}/cg0/x"].tobytes()
    assert np.array(rep.normal_history).tobytes() == g[f"{case}/cg0/nh"].tobytes()
    assert np.array(rep.primal_history).tobytes() == g[f"{case}/cg0/ph"].tobytes()


@pytest.mark.parametrize("case", NEUMANN_CASES)
def test_neumann_cgnr_fast(case, systems, golden):
    """Fast mode (FMA, tree reductions): same trajectory to round-off early on;
    converged fixtures converge."""
    from paper_1807_00410_b200.solver import solve_normal_cg
    s, g = systems[case], golden["neumann"]
    meta = golden["neumann_meta"]["cases"][case]["cg0"]
    x, rep = solve_normal_cg(s, tol=1e-9, max_iter=300)
    nh = g[f"{case}/cg0/nh"]
    k = min(10, len(nh), len(rep.normal_history))
    np.testing.assert_allclose(rep.normal_history[:k], nh[:k], rtol=1e-6, atol=1e-12 * nh[0])
    if meta["converged"]:
        assert rep.converged and rep.normal_residual <= 1e-9
        xr = g[f"{case}/cg0/x"]
        np.testing.assert_allclose(x, xr, rtol=0, atol=1e-6 * max(np.abs(xr).max(), 1e-300))


def test_neumann_larger_grid_matches_oracle():
    """A 32-wide grid beyond the fixtures: device assembly == or_csr_bc, and
    the faithful solve == oracle CGNR over it."""
    from paper_1807_00410_b200.solver import assemble, solve_normal_cg
    spec = replace(rand_spec(3, (33, 9, 7), 91), bc="neumann")
    s = assemble(build_tables(3), spec)
    o = StencilOracle(build_tables(3), spec)
    A, Ao = s.A.to_scipy(), o.csr()
    assert np.array_equal(A.indptr, Ao.indptr) and np.array_equal(A.indices, Ao.indices)
    assert A.data.tobytes() == Ao.data.tobytes() and s.Q.tobytes() == o.rhs.tobytes()
    x, rep = solve_normal_cg(s, tol=1e-8, max_iter=60, mode="faithful", blas_threads=8, blas_kernel=0)
    xo, ro = o.cgnr(tol=1e-8, max_iter=60, blas_threads=8, blas_kernel=0)
    assert rep.iterations == ro["iterations"] and x.tobytes() == xo.tobytes()


def test_neumann_solve_pn_and_run(tmp_path):
    """solve_pn and the batch run honour bc="neumann" (cli.py --bc)."""
    from paper_1807_00410_b200 import run as prun
    from paper_1807_00410_b200.solver import solve_pn
    spec = replace(rand_spec(2, (8, 6, 5), 8), bc="neumann")
    coll, rep, xs = solve_pn(2, spec, tol=1e-10, max_iter=2000, mode="faithful", blas_threads=8, blas_kernel=0,
                             return_staggered=True)
    o = StencilOracle(build_tables(2), spec)
    xo, ro = o.cgnr(tol=1e-10, max_iter=2000, blas_threads=8, blas_kernel=0)
    assert xs.tobytes() == xo.tobytes()
    assert coll.tobytes() == o.unstagger(xo).tobytes()
    cfg = prun.config_from_mapping({"problem": "cfg1", "res": 8, "bc": "neumann", "out": str(tmp_path),
                                    "tol": 1e-6})
    report = prun.run(cfg, log=lambda *_: None)
    assert report.iterations > 0
    assert "bc neumann" in (tmp_path / "solve.log").read_text()


def test_assemble_csr_errors():
    from paper_1807_00410_b200.solver import PnContext
    spec = rand_spec(1, (4, 4, 4), 3)
    ctx = PnContext(build_tables(1), spec.res, spec.h)
    ctx.set_fields(spec)
    with pytest.raises(ValueError):
        ctx.assemble_csr("periodic")
    csr, _ = ctx.assemble_csr("dirichlet")
    with pytest.raises(NotImplementedError):
        csr.assemble_csr("neumann")
