"""General stencil programs on the device (CDA: field-dependent couplings,
equations.py:213-237): pn_assemble_general evaluates the compiled
coefficient programs per voxel and builds the reference's CSR; the CSR
operator solves it.  Checked against the reference fixtures
(tests/golden/cda.npz) and the numpy oracle."""

from dataclasses import replace

import numpy as np
import pytest

from cases import CDA_CASES, cda_inputs, probe_vector, rand_spec
from oracle import general_oracle as go
from oracle.oracle import CsrOracle
from paper_1807_00410_b200.general import build_cda_program

pytestmark = pytest.mark.gpu

FIX_BLAS = (8, 0)


@pytest.fixture(scope="module")
def systems():
    from paper_1807_00410_b200.solver import assemble
    return {name: assemble(*cda_inputs(name)) for name in CDA_CASES}


@pytest.mark.parametrize("case", CDA_CASES)
def test_cda_assembly_bit_exact(case, systems, golden):
    s, g = systems[case], golden["cda"]
    A = s.A.to_scipy()
    assert np.array_equal(A.indptr, g[f"{case}/indptr"]) and np.array_equal(A.indices, g[f"{case}/indices"])
    assert A.data.tobytes() == g[f"{case}/data"].tobytes()
    assert s.Q.tobytes() == g[f"{case}/Q"].tobytes()


@pytest.mark.parametrize("case", CDA_CASES)
def test_cda_products_and_faithful_solve(case, systems, golden):
    from paper_1807_00410_b200.solver import solve_normal_cg, unstagger
    s, g = systems[case], golden["cda"]
    meta = golden["cda_meta"]["cases"][case]["cg0"]
    x = probe_vector(s.A.shape[0])
    assert s.A.matvec(x, mode="faithful").tobytes() == g[f"{case}/Ax"].tobytes()
    assert s.A.T.matvec(x, mode="faithful").tobytes() == g[f"{case}/Atx"].tobytes()
    xs, rep = solve_normal_cg(s, tol=1e-10, max_iter=500, mode="faithful", blas_threads=FIX_BLAS[0],
                              blas_kernel=FIX_BLAS[1])
    assert rep.iterations == meta["iterations"] and rep.converged == meta["converged"]
    assert xs.tobytes() == g[f"{case}/cg0/x"].tobytes()
    assert np.array(rep.normal_history).tobytes() == g[f"{case}/cg0/nh"].tobytes()
    prog, spec = cda_inputs(case)
    assert unstagger(xs, prog, spec.res).tobytes() == g[f"{case}/unstagger"].tobytes()
    assert s.A.ctx.unstagger(xs).cpu().numpy().tobytes() == g[f"{case}/unstagger"].tobytes()


@pytest.mark.parametrize("case", CDA_CASES)
def test_cda_fast_solve_converges(case, systems, golden):
    from paper_1807_00410_b200.solver import solve_normal_cg
    s, g = systems[case], golden["cda"]
    xs, rep = solve_normal_cg(s, tol=1e-10, max_iter=2000)
    assert rep.converged
    xr = g[f"{case}/cg0/x"]
    scale = max(np.abs(xr).max(), 1e-300)
    np.testing.assert_allclose(xs, xr, rtol=0, atol=1e-7 * scale)


def test_cda_larger_grid_and_solve_pn():
    """Beyond the fixtures: a 48x20x16 CDA system == oracle; solve_pn on the
    restated program == oracle CGNR + unstagger, bit for bit."""
    from paper_1807_00410_b200.solver import assemble, solve_pn
    spec = replace(rand_spec(1, (48, 20, 16), 54), bc="dirichlet")
    prog = build_cda_program(3)
    s = assemble(prog, spec)
    A, Q = go.assemble(prog, spec)
    Ad = s.A.to_scipy()
    assert np.array_equal(Ad.indices, A.indices) and Ad.data.tobytes() == A.data.tobytes()
    assert s.Q.tobytes() == Q.tobytes()
    coll, rep, xs = solve_pn(prog, spec, tol=1e-9, max_iter=3000, mode="faithful", blas_threads=8, blas_kernel=0,
                             return_staggered=True)
    xo, ro = CsrOracle(A).cgnr(Q, tol=1e-9, max_iter=3000, blas_threads=8, blas_kernel=0)
    assert rep.iterations == ro["iterations"] and xs.tobytes() == xo.tobytes()
    assert coll.tobytes() == go.unstagger(xo, prog, spec.res).tobytes()


def test_cda_run_writes_reference_field(tmp_path):
    """`run --method cda` (cli.py:114,156): the written field is the oracle's
    CGNR solution, unstaggered, bit for bit (faithful mode)."""
    from paper_1807_00410_b200 import fields as fio
    from paper_1807_00410_b200 import run as prun
    cfg = prun.config_from_mapping({"problem": "cfg1", "method": "cda", "res": 10, "mode": "faithful",
                                    "out": str(tmp_path), "tol": 1e-8})
    report = prun.run(cfg, log=lambda *_: None)
    spec = prun.build_problem(cfg)
    A, Q = go.assemble(build_cda_program(3), spec)
    xo, ro = CsrOracle(A).cgnr(Q, tol=1e-8)
    assert report.iterations == ro["iterations"] and report.converged
    meta, coll = fio.read_field(tmp_path / "field.pnfld")
    assert meta["order"] == 0 and meta["unknowns"] == 1
    assert coll.tobytes() == go.unstagger(xo, build_cda_program(3), spec.res).tobytes()
    assert "method cda" in (tmp_path / "solve.log").read_text()
