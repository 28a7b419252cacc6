"""Solver semantics of the reference tests (test_solver.py) on the device
path, edge cases, the drop-in API, and the slab decomposition (loopback
group of z-slab contexts on one GPU: P slabs == 1 slab, bit for bit)."""

import ctypes

import numpy as np
import pytest

from cases import rand_spec
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.problems import ProblemSpec, phase_fields
from paper_1807_00410_b200.program import build_tables, q_name


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

pytestmark = pytest.mark.gpu


def homogeneous_spec(res, sigma_t=1.0, sigma_s=0.0, q=0.0, extent=1.0):
    """test_solver.py:21-31."""
    shape = (res,) * 3
    f = {"sigma_t": np.full(shape, sigma_t), "sigma_s": np.full(shape, sigma_s),
         "p_0": np.full(shape, 1 / np.sqrt(4 * np.pi)), q_name(0, 0): np.full(shape, q)}
    return ProblemSpec(dim=3, origin=(0.0,) * 3, extent=(extent,) * 3, res=shape, fields=f)


def test_single_voxel_is_diagonal():
    """test_solver.py:38-45: 1x1x1 Dirichlet keeps only collision entries."""
    from paper_1807_00410_b200.solver import assemble
    s = assemble(build_tables(1), homogeneous_spec(1, sigma_t=1.0))
    A = s.A.to_scipy().toarray()
    np.testing.assert_allclose(A, np.eye(4), atol=1e-14)


def test_center_row_p1_has_seven_nonzeros():
    """test_solver.py:48-55."""
    from paper_1807_00410_b200.solver import assemble
    s = assemble(build_tables(1), homogeneous_spec(3))
    assert s.A.to_scipy().getrow(13 * 4).nnz == 7


def test_adjoint_consistency():
    """test_solver.py:82-92 on the fast device operator."""
    from paper_1807_00410_b200.solver import assemble
    s = assemble(build_tables(3), rand_spec(3, (32, 5, 4), 3))
    rng = np.random.default_rng(0)
    for _ in range(5):
        u, v = rng.normal(size=s.A.shape[0]), rng.normal(size=s.A.shape[0])
        lhs, rhs = float((s.A @ u) @ v), float(u @ (s.A.T @ v))
        assert abs(lhs - rhs) <= 1e-12 * (1 + abs(lhs))


def test_nonconvergence_reported_not_raised():
    from paper_1807_00410_b200.solver import assemble, solve_normal_cg
    s = assemble(build_tables(3), rand_spec(3, (32, 4, 4), 5))
    for mode in ("fast", "faithful"):
        _, rep = solve_normal_cg(s, tol=1e-14, max_iter=3, mode=mode)
        assert not rep.converged and rep.iterations == 3 and len(rep.normal_history) == 3


def test_tol_must_be_positive():
    from paper_1807_00410_b200.solver import assemble, solve_normal_cg
    s = assemble(build_tables(1), homogeneous_spec(2))
    with pytest.raises(ValueError):
        solve_normal_cg(s, tol=0.0)


def test_zero_rhs_returns_zero_converged():
    """solver.py:211-216."""
    from paper_1807_00410_b200.solver import assemble, solve_normal_cg
    s = assemble(build_tables(1), homogeneous_spec(4, q=0.0))
    x, rep = solve_normal_cg(s, tol=1e-8)
    assert rep.converged and rep.iterations == 0 and not np.any(x)
    assert rep.normal_residual == 0.0 and rep.primal_residual == 0.0


def test_max_iter_zero_and_warm_start():
    from paper_1807_00410_b200.solver import assemble, solve_normal_cg
    s = assemble(build_tables(3), rand_spec(3, (32, 4, 3), 8))
    x, rep = solve_normal_cg(s, tol=1e-10, max_iter=2000)
    x2, rep2 = solve_normal_cg(s, tol=1e-10, max_iter=0, x0=x)
    assert rep2.iterations == 0 and np.array_equal(x2, x)
    _, rep3 = solve_normal_cg(s, tol=1e-6, max_iter=2000, x0=x)
    assert rep3.iterations <= 1


def test_primal_tol_and_histories():
    """test_solver.py:148-155."""
    from paper_1807_00410_b200.solver import assemble, solve_normal_cg
    s = assemble(build_tables(1), rand_spec(1, (32, 6, 5), 9))
    _, rep = solve_normal_cg(s, tol=1e-10, max_iter=5000, primal_tol=1e-12)
    assert rep.converged and rep.normal_history[-1] <= 1e-10 and rep.primal_history[-1] <= 1e-12
    assert len(rep.primal_history) == len(rep.normal_history) == rep.iterations


def test_jacobi_consistent():
    """test_solver.py:136-145."""
    from paper_1807_00410_b200.solver import assemble, solve_normal_cg
    s = assemble(build_tables(3), rand_spec(3, (32, 5, 4), 10))
    x0, r0 = solve_normal_cg(s, tol=1e-12, max_iter=5000)
    x1, r1 = solve_normal_cg(s, tol=1e-12, max_iter=5000, jacobi=True)
    assert r0.converged and r1.converged
    np.testing.assert_allclose(x0, x1, atol=1e-6 * np.abs(x0).max())


def test_dim_mismatch_raises():
    from paper_1807_00410_b200.solver import assemble
    f = {"sigma_t": np.ones((3, 3)), "sigma_s": np.zeros((3, 3))}
    spec2 = ProblemSpec(dim=2, origin=(0, 0), extent=(1, 1), res=(3, 3), fields=f)
    with pytest.raises(ValueError):
        assemble(build_tables(1), spec2)


def test_uniform_fields_segmented_path():
    """Scalar (0-d) sigma fields are materialised for the segmented kernel."""
    from paper_1807_00410_b200.solver import PnContext
    from oracle.oracle import StencilOracle
    spec = rand_spec(5, (32, 4, 4), 12, uniform_sigma=True)
    spec = ProblemSpec(3, spec.origin, spec.extent, spec.res,
                       dict(spec.fields, sigma_t=np.float64(4.0), sigma_s=np.float64(3.0)))
    c = PnContext(build_tables(5), spec.res, spec.h)
    c.set_fields(spec)
    o = StencilOracle(build_tables(5), spec)
    x = np.random.default_rng(1).normal(size=o.R)
    y = c.apply(x, 0, "fast").cpu().numpy()
    assert np.linalg.norm(y - o.apply(x)) <= 1e-13 * np.linalg.norm(o.apply(x))


def test_solve_pn_end_to_end():
    """Order + fields in, collocated (N+1)^2 coefficients out (cli.py:136-155)."""
    from paper_1807_00410_b200.solver import solve_pn
    from oracle.oracle import StencilOracle
    cfg = make_config(3, n=32)
    spec = solve_spec(cfg)
    coll, rep, xs = solve_pn(cfg.N, spec, tol=1e-6, max_iter=20000, return_staggered=True)
    assert rep.converged and coll.shape == (32, 32, 32, 36)
    o = StencilOracle(build_tables(cfg.N), spec)
    assert coll.tobytes() == o.unstagger(xs).tobytes()
    # the reference's result record (solver.py:53-59) through the package-level names
    import paper_1807_00410_b200 as pkg
    f = pkg.solve_pn(cfg.N, spec, tol=1e-6, max_iter=20000, as_field=True)
    assert isinstance(f, pkg.SolutionField) and f.spec is spec and f.report.iterations == rep.iterations
    assert f.collocated.tobytes() == coll.tobytes() and f.staggered.tobytes() == xs.tobytes()
    assert f.unknowns[:4] == [(0, 0), (1, -1), (1, 0), (1, 1)] and len(f.unknowns) == 36


def _group(tables, spec, n_slabs):
    from paper_1807_00410_b200.solver import PnContext
    nz = spec.res[2]
    out = []
    for r in range(n_slabs):
        c = PnContext(tables, spec.res, spec.h, z0=r * nz // n_slabs, nz_local=nz // n_slabs, rank=r, world=n_slabs)
        c.set_fields(spec)
        out.append(c)
    return out


@pytest.mark.parametrize("N,res,slabs", [(1, (32, 8, 8), 2), (3, (32, 6, 8), 4), (7, (32, 4, 4), 2), (5, (32, 8, 12), 3), (7, (64, 8, 10), 2),
                                         (3, (7, 5, 6), 3)])
@pytest.mark.parametrize("bulk", ["0", "1"])
def test_loopback_slabs_match_single_slab(N, res, slabs, bulk, monkeypatch):
    """z-slab decomposition (halo planes + all-gathered plane partials) gives
    the single-GPU result bit for bit, for the operator and the full solve;
    with the segmented kernel's cp.async (bulk=0) and bulk/TMA (bulk=1)
    staging paths (the plane-range launches of the interior / boundary planes
    differ between the two).  Grids with nx % 32 != 0 run the table operator
    on slabs, so the single context is pinned to it too (PNRTE_SEG_PAD=0; the
    zero-padded segmented path is checked in test_padded_segmented_path)."""
    import torch
    monkeypatch.setenv("PNRTE_SEG_BULK", bulk)
    monkeypatch.setenv("PNRTE_SEG_PAD", "0")
    monkeypatch.setenv("PNRTE_SMALL_MAX", "0")   # the launch chain, as the slab group runs
    from paper_1807_00410_b200 import _lib
    from paper_1807_00410_b200.solver import PnContext
    spec = rand_spec(N, res, 31)
    t = build_tables(N)
    one = PnContext(t, res, spec.h)
    one.set_fields(spec)
    grp = _group(t, spec, slabs)
    L = _lib.load()
    x = torch.tensor(np.random.default_rng(2).normal(size=one.R_local), dtype=torch.float64, device="cuda")
    R_l = grp[0].R_local
    for mode in (0, 1):
        for tr in (0, 1):
            want = one.apply(x, tr, "faithful" if mode else "fast")
            ys = [torch.empty(R_l, dtype=torch.float64, device="cuda") for _ in grp]
            xs = [x[r * R_l:(r + 1) * R_l].contiguous() for r in range(slabs)]
            hs = (ctypes.c_void_p * slabs)(*[g.handle.value for g in grp])
            xp = (ctypes.c_void_p * slabs)(*[v.data_ptr() for v in xs])
            yp = (ctypes.c_void_p * slabs)(*[v.data_ptr() for v in ys])
            _lib.check(L.pn_group_apply(hs, slabs, tr, mode, xp, yp, None))
            got = torch.cat(ys)
            assert torch.equal(got, want), (mode, tr)
    xo, ro = one.solve(tol=1e-9, max_iter=300, mode="fast")
    xs = [torch.empty(R_l, dtype=torch.float64, device="cuda") for _ in grp]
    opts = _lib.SolveOpts(1e-9, 300, -1.0, 0, 0, 8, 0, 0)
    rep = _lib.Report()
    hs = (ctypes.c_void_p * slabs)(*[g.handle.value for g in grp])
    xp = (ctypes.c_void_p * slabs)(*[v.data_ptr() for v in xs])
    _lib.check(L.pn_group_solve(hs, slabs, ctypes.byref(opts), xp, ctypes.byref(rep), None, None, 0, None))
    assert rep.iterations == ro.iterations
    assert torch.equal(torch.cat(xs), xo)


@pytest.mark.parametrize("N,res", [(1, (7, 5, 6)), (3, (33, 6, 5)), (5, (40, 9, 7)), (7, (17, 4, 5)), (2, (65, 3, 4))])
def test_padded_segmented_path(N, res, monkeypatch):
    """nx % 32 != 0 on one slab: the segmented operator on the zero-padded
    solve layout (last 32-voxel row partial) against the table operator
    (PNRTE_SEG_PAD=0) and the C oracle, for A, A^T, the fused reductions
    (solve) and Jacobi: products within rounding, solves to the same
    iteration count and field."""
    from oracle.oracle import StencilOracle
    from paper_1807_00410_b200.solver import PnContext
    spec = rand_spec(N, res, 55 + N)
    t = build_tables(N)
    out = {}
    monkeypatch.setenv("PNRTE_SMALL_MAX", "0")   # the segmented solve, not the one-launch small path
    for pad in ("1", "0"):
        monkeypatch.setenv("PNRTE_SEG_PAD", pad)
        c = PnContext(t, res, spec.h)
        c.set_fields(spec)
        x = np.random.default_rng(9).normal(size=c.R_local)
        ys = [c.apply(x, tr, "fast").cpu().numpy() for tr in (0, 1)]
        sols = [c.solve(tol=1e-10, max_iter=3000, jacobi=j, mode="fast") for j in (False, True)]
        out[pad] = (ys, sols)
    o = StencilOracle(t, spec)
    for tr in (0, 1):
        want = o.apply(np.random.default_rng(9).normal(size=o.R), bool(tr))
        assert rel(out["1"][0][tr], want) <= 1e-13
        assert rel(out["1"][0][tr], out["0"][0][tr]) <= 1e-13
    for (xa, ra), (xb, rb) in zip(out["1"][1], out["0"][1]):
        assert ra.converged and rb.converged
        assert abs(ra.iterations - rb.iterations) <= 1
        assert rel(xa.cpu().numpy(), xb.cpu().numpy()) <= 1e-8


# ---------------------------------------------------------------------------
# generic CSR systems (test_solver.py:99-145 of the reference)
# ---------------------------------------------------------------------------

def _csr_system(A, b):
    import scipy.sparse as sp
    from paper_1807_00410_b200.solver import SparseSystem
    return SparseSystem(A=sp.csr_matrix(A), Q=b, res=(len(b),), n_unknowns=1)


def test_csr_identity_single_iteration():
    import scipy.sparse as sp
    from paper_1807_00410_b200.solver import solve_normal_cg
    b = np.zeros(6)
    b[0] = 1.0
    x, rep = solve_normal_cg(_csr_system(sp.identity(6, format="csr"), b), tol=1e-12)
    np.testing.assert_allclose(x, b, atol=1e-12)
    assert rep.converged and rep.iterations == 1


def test_csr_matches_dense_lu():
    from paper_1807_00410_b200.solver import solve_normal_cg
    rng = np.random.default_rng(1)
    n = 50
    A = rng.normal(size=(n, n)) + n * np.eye(n)
    b = A @ rng.normal(size=n)
    x, rep = solve_normal_cg(_csr_system(A, b), tol=1e-12, max_iter=2000)
    assert rep.converged
    np.testing.assert_allclose(x, np.linalg.solve(A, b), atol=1e-8)


def test_csr_nonconvergence_and_jacobi():
    from paper_1807_00410_b200.solver import solve_normal_cg
    rng = np.random.default_rng(2)
    A = rng.normal(size=(40, 40)) + np.diag(np.logspace(0, 6, 40))
    _, rep = solve_normal_cg(_csr_system(A, rng.normal(size=40)), tol=1e-14, max_iter=3)
    assert not rep.converged and rep.iterations == 3 and len(rep.normal_history) == 3
    rng = np.random.default_rng(3)
    A = rng.normal(size=(60, 60)) + np.diag(rng.uniform(5, 500, 60))
    b = rng.normal(size=60)
    x0, r0 = solve_normal_cg(_csr_system(A, b), tol=1e-12, max_iter=5000)
    x1, r1 = solve_normal_cg(_csr_system(A, b), tol=1e-12, max_iter=5000, jacobi=True)
    assert r0.converged and r1.converged
    np.testing.assert_allclose(x0, x1, atol=1e-6)


@pytest.mark.parametrize("n", [1, 37, 3001])
def test_csr_products_ragged_rows(n):
    """Generic CSR with empty rows, single entries and long rows (up to 300
    entries, odd and even lengths): the fast product (two lanes per row,
    shuffle fold) within rounding of scipy, the faithful product (one thread
    per row, stored order, mul-then-add) bit-identical to scipy's csr_matvec,
    for A and A^T."""
    import scipy.sparse as sp
    import torch
    from paper_1807_00410_b200.solver import PnContext
    rng = np.random.default_rng(n)
    lens = rng.choice([0, 1, 2, 3, 7, 10, 33, 300], size=n, p=[.15, .15, .1, .1, .2, .2, .05, .05])
    rows, cols = [], []
    for i, L in enumerate(lens):
        c = np.sort(rng.choice(n, size=min(int(L), n), replace=False))
        rows += [i] * len(c)
        cols += list(c)
    A = sp.csr_matrix((rng.normal(size=len(rows)), (rows, cols)), shape=(n, n))
    A.sort_indices()
    x = rng.normal(size=n)
    c = PnContext.from_csr(A)
    for tr, M in ((False, A), (True, A.T.tocsr())):
        want = M @ x
        fast = c.apply(x, transpose=tr).cpu().numpy()
        scale = abs(M) @ np.abs(x)
        assert np.all(np.abs(fast - want) <= 1e-13 * scale)   # ~ 900 ulp of sum |a x|, rows up to 300
        faithful = c.apply(x, transpose=tr, mode="faithful").cpu().numpy()
        assert faithful.tobytes() == want.tobytes()
    torch.cuda.synchronize()


@pytest.mark.parametrize("case", ["p3_456", "p7_343", "p1_3286"])
@pytest.mark.parametrize("jac", [0, 1])
def test_csr_faithful_bit_identical_to_reference(case, jac, golden):
    """The reference's own assembled CSR (fixture), solved on the device in
    faithful mode: bit-identical to solve_normal_cg on that matrix."""
    import scipy.sparse as sp
    from paper_1807_00410_b200.solver import SparseSystem, solve_normal_cg
    g, meta = golden["cases"], golden["cases_meta"]["cases"][case]
    n = len(g[f"{case}/indptr"]) - 1
    A = sp.csr_matrix((g[f"{case}/data"], g[f"{case}/indices"], g[f"{case}/indptr"]), shape=(n, n))
    s = SparseSystem(A=A, Q=g[f"{case}/Q"], res=(n,), n_unknowns=1)
    x, rep = solve_normal_cg(s, tol=1e-9, max_iter=400, jacobi=bool(jac), mode="faithful", blas_threads=8,
                             blas_kernel=0)
    assert rep.iterations == meta[f"cg{jac}"]["iterations"]
    assert x.tobytes() == g[f"{case}/cg{jac}/x"].tobytes()
    assert np.array(rep.normal_history).tobytes() == g[f"{case}/cg{jac}/nh"].tobytes()


# ---------------------------------------------------------------------------
# C ABI error behaviour and native-path evidence
# ---------------------------------------------------------------------------

def test_abi_error_codes():
    import ctypes
    import scipy.sparse as sp
    from paper_1807_00410_b200 import _lib
    from paper_1807_00410_b200.solver import PnContext
    L = _lib.load()
    spec = rand_spec(1, (4, 4, 4), 1)
    c = PnContext(build_tables(1), spec.res, spec.h)
    with pytest.raises(ValueError):                        # bad field slot
        _lib.check(L.pn_set_field(c.handle, 999, 0, 0.0, None, None))
    with pytest.raises(ValueError):                        # setup not called
        c.solve(tol=1e-6)
    c.set_fields(spec)
    with pytest.raises(ValueError):                        # tol <= 0 (solver.py:200-201)
        c.solve(tol=0.0)
    csr = PnContext.from_csr(sp.identity(5, format="csr"))
    with pytest.raises(NotImplementedError):               # stencil-only entry point
        csr.unstagger(np.zeros(5))
    with pytest.raises(ValueError):                        # CSR solve needs b
        csr.solve(tol=1e-6)
    assert "tolerance" in L.pn_last_error().decode() or L.pn_last_error()


def test_native_kernels_ran():
    """The solve runs in libpnrte_b200.so: its kernel counter moves and the
    library is mapped into this process."""
    from paper_1807_00410_b200 import _lib
    from paper_1807_00410_b200.solver import PnContext
    spec = rand_spec(3, (32, 4, 4), 3)
    c = PnContext(build_tables(3), spec.res, spec.h)
    c.set_fields(spec)
    n0 = c.kernel_launches()
    c.solve(tol=1e-8, max_iter=50)
    assert c.kernel_launches() > n0
    maps = open("/proc/self/maps").read()
    assert str(_lib.LIB_PATH) in maps


# ---------------------------------------------------------------------------
# 2-D programs (reference test_solver.py:82-92, 148-155 use the checkerboard)
# ---------------------------------------------------------------------------

def test_2d_matvec_adjoint_consistency():
    from cases import tables_2d
    from paper_1807_00410_b200.problems import make_checkerboard
    from paper_1807_00410_b200.solver import assemble
    s = assemble(tables_2d(2), make_checkerboard(15))
    assert s.A.shape[0] == 15 * 15 * 6
    rng = np.random.default_rng(0)
    for _ in range(5):
        u, v = rng.normal(size=s.A.shape[0]), rng.normal(size=s.A.shape[0])
        lhs, rhs = float((s.A @ u) @ v), float(u @ (s.A.T @ v))
        assert abs(lhs - rhs) <= 1e-12 * (1 + abs(lhs))


def test_2d_cg_residual_histories_recorded():
    from cases import tables_2d
    from paper_1807_00410_b200.problems import make_checkerboard
    from paper_1807_00410_b200.solver import assemble, solve_normal_cg, unstagger
    s = assemble(tables_2d(1), make_checkerboard(15))
    x, rep = solve_normal_cg(s, tol=1e-10, max_iter=5000)
    assert rep.converged and rep.normal_history[-1] <= 1e-10
    assert len(rep.primal_history) == len(rep.normal_history)
    assert rep.primal_residual < 1e-8
    coll = unstagger(x, tables_2d(1), (15, 15))
    assert coll.shape == (15, 15, 3)


def test_2d_checkerboard_71_size():
    """test_solver.py:58-61: the full checkerboard P1 system has 71*71*3 rows."""
    from cases import tables_2d
    from paper_1807_00410_b200.problems import make_checkerboard
    from paper_1807_00410_b200.solver import assemble
    assert assemble(tables_2d(1), make_checkerboard()).A.shape[0] == 71 * 71 * 3


def test_nccl_call_patterns_on_one_rank():
    """The NCCL calls of the slab path (communicator from a unique id, grouped
    send / recv of a plane, in-place all-gather of plane sums) captured into a
    CUDA graph on a forked stream and replayed, on a one-rank communicator:
    library, linkage and capture of NCCL work on this box (one GPU cannot show
    two ranks agreeing; the loopback groups and the gloo tests cover that)."""
    from paper_1807_00410_b200.distributed import nccl_selftest
    nccl_selftest(0, 256 * 256 * 4)


def test_solve_host_composite_through_the_c_abi():
    """pn_solve_host (include/pnrte_b200.h): plain host pointers in and out, as
    a cgo / JNI binding would call it -- no torch tensor crosses the boundary.
    Faithful solve of a small P3 system == the oracle's bits; fast solve equal
    to PnContext.solve's."""
    from paper_1807_00410_b200 import _lib
    from paper_1807_00410_b200.solver import PnContext
    from oracle.oracle import StencilOracle
    N, res = 3, (32, 6, 5)
    spec = rand_spec(N, res, 515)
    t = build_tables(N)
    c = PnContext(t, res, spec.h)
    c.set_fields(spec)
    L = _lib.load()

    def run(mode):
        o = _lib.SolveOpts()
        o.tol, o.max_iter, o.primal_tol, o.jacobi, o.mode = 1e-8, 600, -1.0, 0, mode
        o.blas_threads, o.blas_kernel, o.check_every = 8, 0, 0
        x = np.full(c.R_local, np.nan)
        hn, hp = np.zeros(600), np.zeros(600)
        rep = _lib.Report()
        _lib.check(L.pn_solve_host(c.handle, ctypes.byref(o), x.ctypes.data_as(ctypes.c_void_p), ctypes.byref(rep),
                                   hn.ctypes.data_as(ctypes.c_void_p), hp.ctypes.data_as(ctypes.c_void_p), 600))
        return x, rep, hn[:rep.iterations]

    xo, ro = StencilOracle(t, spec).cgnr(tol=1e-8, max_iter=600, blas_threads=8, blas_kernel=0)
    x, rep, hn = run(1)
    assert rep.iterations == ro["iterations"] and bool(rep.converged) and x.tobytes() == xo.tobytes()
    assert hn.tolist() == ro["normal_history"]
    xf, repf, _ = run(0)
    xs, rs = c.solve(tol=1e-8, max_iter=600)
    assert repf.iterations == rs.iterations and xf.tobytes() == xs.cpu().numpy().tobytes()


@pytest.mark.parametrize("N,res", [(7, (64, 9, 6)), (7, (64, 70, 9)), (3, (80, 13, 4)), (4, (96, 130, 5)), (1, (64, 9, 6))])
def test_fused_residual_update_is_bit_identical_to_the_chain(N, res, monkeypatch):
    """Opt-in k_seg_fr (PNRTE_SEG_FUSE_R=1): r -= alpha w inside the A^T apply launch,
    handed over through L2 under ticket order and release / acquire flags.  Same
    arithmetic and partial slots as k_r + k_seg: fixed-iteration solves (with and
    without Jacobi) and a converged solve give the same solution and histories."""
    from paper_1807_00410_b200.solver import PnContext
    monkeypatch.setenv("PNRTE_SEG_BULK", "1")
    monkeypatch.setenv("PNRTE_SMALL_MAX", "0")
    spec = rand_spec(N, res, 70 + N)
    got = []
    for fuse in ("0", "1"):
        monkeypatch.setenv("PNRTE_SEG_FUSE_R", fuse)
        c = PnContext(build_tables(N), res, spec.h)
        c.set_fields(spec)
        runs = []
        for kw in (dict(tol=1e-30, max_iter=40), dict(tol=1e-30, max_iter=40, jacobi=True), dict(tol=1e-7, max_iter=4000)):
            x, rep = c.solve(**kw)
            runs.append((x.cpu().numpy().tobytes(), rep.iterations, rep.normal_history, rep.primal_history))
        # fields set again on the same context (the ticket counter and the chunk flags start over together)
        c.set_fields(spec)
        x, rep = c.solve(tol=1e-30, max_iter=40)
        assert (x.cpu().numpy().tobytes(), rep.iterations, rep.normal_history, rep.primal_history) == runs[0]
        got.append(runs)
        del c
    assert got[0] == got[1]
