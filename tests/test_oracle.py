"""The C oracle (oracle/pn_oracle.c) pinned against the reference: committed
fixtures everywhere, the live reference where it is mounted."""

import hashlib

import numpy as np
import pytest

from cases import ALL_CASES, CASES, NEUMANN_CASES, case_inputs, probe_vector, rand_spec
from oracle.oracle import StencilOracle, ddot
from paper_1807_00410_b200.configs import make_config
from paper_1807_00410_b200.program import build_tables

FIX_BLAS = (8, 0)   # fixtures were generated with OpenBLAS SkylakeX, 8 threads


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def oracles():
    return {name: StencilOracle(*case_inputs(name)) for name in ALL_CASES}


@pytest.mark.parametrize("case", ALL_CASES)
def test_oracle_assembly_matches_golden(case, oracles, golden):
    o, g = oracles[case], golden["cases"]
    A = o.csr()
    assert np.array_equal(A.indptr, g[f"{case}/indptr"])
    assert np.array_equal(A.indices, g[f"{case}/indices"])
    assert A.data.tobytes() == g[f"{case}/data"].tobytes()
    assert o.rhs.tobytes() == g[f"{case}/Q"].tobytes()
    assert o.jacobi_diag().tobytes() == g[f"{case}/jac"].tobytes()


@pytest.mark.parametrize("case", ALL_CASES)
def test_oracle_apply_matches_golden(case, oracles, golden):
    o, g = oracles[case], golden["cases"]
    x = probe_vector(o.R)
    assert o.apply(x).tobytes() == g[f"{case}/Ax"].tobytes()
    assert o.apply(x, transpose=True).tobytes() == g[f"{case}/Atx"].tobytes()


@pytest.mark.parametrize("case", ALL_CASES)
def test_oracle_cgnr_matches_golden(case, oracles, golden):
    o, g, meta = oracles[case], golden["cases"], golden["cases_meta"]["cases"][case]
    for jac in (0, 1):
        x, rep = o.cgnr(tol=1e-9, max_iter=400, jacobi=bool(jac), blas_threads=FIX_BLAS[0], blas_kernel=FIX_BLAS[1])
        k = f"{case}/cg{jac}"
        assert rep["iterations"] == meta[f"cg{jac}"]["iterations"]
        assert x.tobytes() == g[k + "/x"].tobytes()
        assert np.array(rep["normal_history"]).tobytes() == g[k + "/nh"].tobytes()
        assert np.array(rep["primal_history"]).tobytes() == g[k + "/ph"].tobytes()
        assert rep["normal_residual"] == meta[f"cg{jac}"]["normal_residual"]
    xs = g[f"{case}/cg0/x"]
    assert o.unstagger(xs).tobytes() == g[f"{case}/unstagger"].tobytes()


def test_oracle_config1_bit_identical_to_reference(golden):
    cfg = make_config(1)
    want = golden["configs"]["cfg1"]
    o = StencilOracle(build_tables(cfg.N), cfg.spec)
    assert sha(o.rhs) == want["Q_sha256"]
    x, rep = o.cgnr(tol=cfg.tol, max_iter=cfg.max_iter, blas_threads=FIX_BLAS[0], blas_kernel=FIX_BLAS[1])
    assert rep["iterations"] == want["iterations"] == 169
    assert sha(x) == want["x_sha256"]
    assert rep["normal_history"] == want["normal_history"]


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_ddot_emulation_properties(kernel, threads):
    """Exact on integer-valued data (no rounding anywhere), symmetric in its
    arguments, and chunk results combine in order."""
    rng = np.random.default_rng(threads)
    for n in (0, 1, 15, 16, 17, 31, 33, 10000, 10001, 123457):
        x = rng.integers(-8, 8, n).astype(float)
        y = rng.integers(-8, 8, n).astype(float)
        assert ddot(x, y, threads, kernel) == float(np.sum(x * y))
        z = rng.normal(size=n)
        assert ddot(z, x, threads, kernel) == ddot(x, z, threads, kernel)


@pytest.mark.reference
def test_ddot_emulation_matches_numpy_blas(ref):
    from oracle.oracle import blas_pin
    th, kn = blas_pin()
    rng = np.random.default_rng(7)
    for n in list(range(1, 80)) + [9999, 10000, 10001, 65537, 1000003]:
        x = rng.normal(size=n)
        y = rng.normal(size=n) * np.exp(rng.normal(size=n))
        assert ddot(x, y, th, kn) == float(x @ y)
        assert np.sqrt(ddot(x, x, th, kn)) == float(np.linalg.norm(x))


@pytest.mark.reference
@pytest.mark.parametrize("case", ["p3_456", "p7_343", "p5_3233"])
def test_oracle_matches_live_reference(case, ref):
    from pnrte.equations import build_pn
    from pnrte.solver import assemble, solve_normal_cg
    from pnrte.stencil import compile_program
    _, N, res, seed = [c for c in CASES if c[0] == case][0]
    spec = rand_spec(N, res, seed)
    s = assemble(compile_program(build_pn(N, 3)), spec)
    o = StencilOracle(build_tables(N), spec)
    x, rep = o.cgnr(tol=1e-10, max_iter=500, jacobi=True)
    xr, rr = solve_normal_cg(s, tol=1e-10, max_iter=500, jacobi=True)
    assert rep["iterations"] == rr.iterations and x.tobytes() == xr.tobytes()


# ---------------------------------------------------------------- Neumann --
@pytest.mark.parametrize("case", NEUMANN_CASES)
def test_oracle_neumann_matches_golden(case, golden):
    """or_csr_bc / or_setup_bc against the reference's bc="neumann" assembly:
    clipped writes, summed duplicates, unpinned RHS; CGNR over that CSR."""
    o = StencilOracle(*case_inputs(case))
    g, meta = golden["neumann"], golden["neumann_meta"]["cases"][case]
    A = o.csr()
    assert np.array_equal(A.indptr, g[f"{case}/indptr"])
    assert np.array_equal(A.indices, g[f"{case}/indices"])
    assert A.data.tobytes() == g[f"{case}/data"].tobytes()
    assert o.rhs.tobytes() == g[f"{case}/Q"].tobytes()
    assert o.jacobi_diag().tobytes() == g[f"{case}/jac"].tobytes()
    x = probe_vector(o.R)
    assert o.apply(x).tobytes() == g[f"{case}/Ax"].tobytes()
    assert o.apply(x, transpose=True).tobytes() == g[f"{case}/Atx"].tobytes()
    xs, rep = o.cgnr(tol=1e-9, max_iter=300, blas_threads=FIX_BLAS[0], blas_kernel=FIX_BLAS[1])
    assert rep["iterations"] == meta["cg0"]["iterations"]
    assert xs.tobytes() == g[f"{case}/cg0/x"].tobytes()
    assert np.array(rep["normal_history"]).tobytes() == g[f"{case}/cg0/nh"].tobytes()


def test_neumann_redirects_instead_of_dropping():
    """The reference's own Neumann check (test_solver.py:73-79): redirected
    writes keep more entries than Dirichlet's dropped ones."""
    from dataclasses import replace
    spec = rand_spec(1, (4, 4, 4), 5)
    nd = StencilOracle(build_tables(1), spec).csr().nnz
    nn = StencilOracle(build_tables(1), replace(spec, bc="neumann")).csr().nnz
    assert nn > nd


@pytest.mark.reference
def test_oracle_neumann_matches_live_reference(ref):
    from dataclasses import replace
    from pnrte.equations import build_pn
    from pnrte.solver import assemble
    from pnrte.stencil import compile_program
    spec = replace(rand_spec(4, (4, 3, 5), 77), bc="neumann")
    s = assemble(compile_program(build_pn(4, 3)), spec)
    A = StencilOracle(build_tables(4), spec).csr()
    assert np.array_equal(A.indices, s.A.indices) and A.data.tobytes() == s.A.data.tobytes()


@pytest.mark.parametrize("idx", [3, 4])
def test_oracle_perfcfg_assembly_and_products(idx, golden):
    """The config-3/4 generators at 32^3 (floor 1): the oracle reproduces the
    live reference's assembly and products (tests/golden/perfcfg.json)."""
    import json
    from paper_1807_00410_b200.configs import solve_spec
    want = json.loads((golden["dir"] / "perfcfg.json").read_text())[f"cfg{idx}_n32"]
    cfg = make_config(idx, n=32)
    o = StencilOracle(build_tables(cfg.N), solve_spec(cfg))
    A = o.csr()
    assert sha(A.indices.astype(np.int32)) == want["A_indices_sha256"]
    assert sha(A.data) == want["A_data_sha256"]
    assert sha(o.rhs) == want["Q_sha256"]
    x = probe_vector(o.R)
    assert sha(o.apply(x)) == want["Ax_sha256"]
    assert sha(o.apply(x, True)) == want["Atx_sha256"]


def test_oracle_perfcfg3_solve_matches_reference(golden):
    """The whole config-3-generator CGNR at 32^3 (452 iterations to 1e-6): the
    oracle's trajectory is the reference's, bit for bit."""
    import json
    from paper_1807_00410_b200.configs import solve_spec
    want = json.loads((golden["dir"] / "perfcfg.json").read_text())["cfg3_n32"]
    cfg = make_config(3, n=32)
    o = StencilOracle(build_tables(cfg.N), solve_spec(cfg))
    x, rep = o.cgnr(tol=cfg.tol, max_iter=cfg.max_iter, blas_threads=FIX_BLAS[0], blas_kernel=FIX_BLAS[1])
    assert rep["iterations"] == want["iterations"]
    assert sha(x) == want["x_sha256"]
    assert rep["normal_history"] == want["normal_history"]
    assert sha(o.unstagger(x)) == want["unstagger_sha256"]
