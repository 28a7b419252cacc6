"""One-launch small-system CGNR (launch_cg_small, PNRTE_SMALL_MAX): the
iteration loop of solve_normal_cg (solver.py:231-253) as one cooperative
kernel, checked against the launch-chain fast path (PNRTE_SMALL_MAX=0) and the
C oracle of the reference solve: same iteration count within +-1, field and
residual histories within the fast-mode tolerances."""

import numpy as np
import pytest

from cases import rand_spec
from paper_1807_00410_b200.problems import ProblemSpec
from paper_1807_00410_b200.program import build_tables

pytestmark = pytest.mark.gpu

ALWAYS, NEVER = str(1 << 40), "0"


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _solve(spec, N, small, monkeypatch, **kw):
    from paper_1807_00410_b200.solver import PnContext
    monkeypatch.setenv("PNRTE_SMALL_MAX", small)
    c = PnContext(build_tables(N), spec.res, spec.h)
    c.set_fields(spec)
    n0 = c.kernel_launches()
    x, rep = c.solve(**kw)
    return x.cpu().numpy(), rep, c.kernel_launches() - n0


def _field_phase(spec, seed):
    """p_1 as a field: the fast operator uses the stored diagonal."""
    rng = np.random.default_rng(seed)
    f = dict(spec.fields)
    f["p_1"] = 0.05 + 0.1 * rng.random(spec.res)
    return ProblemSpec(3, spec.origin, spec.extent, spec.res, f)


CASES = [(1, (32, 32, 32)), (3, (32, 6, 5)), (5, (17, 9, 7)), (7, (8, 8, 8)), (2, (40, 3, 4)), (1, (1, 1, 1)),
         (4, (5, 7, 1))]


@pytest.mark.parametrize("N,res", CASES)
@pytest.mark.parametrize("jacobi", [False, True])
def test_small_solve_matches_chain_and_oracle(N, res, jacobi, monkeypatch):
    from oracle.oracle import StencilOracle
    spec = rand_spec(N, res, 70 + N)
    kw = dict(tol=1e-10, max_iter=3000, jacobi=jacobi)
    xs, rs, ls = _solve(spec, N, ALWAYS, monkeypatch, **kw)
    xc, rc, lc = _solve(spec, N, NEVER, monkeypatch, **kw)
    xo, ro = StencilOracle(build_tables(N), spec).cgnr(**kw)
    assert rs.converged and rc.converged
    assert abs(rs.iterations - ro["iterations"]) <= 1 and abs(rs.iterations - rc.iterations) <= 1
    assert rel(xs, xo) <= 1e-8 and rel(xs, xc) <= 1e-8
    assert len(rs.normal_history) == rs.iterations == len(rs.primal_history)
    n = min(rs.iterations, rc.iterations)
    hs, hc = np.array(rs.normal_history[:n]), np.array(rc.normal_history[:n])
    big = hc > 1e-3
    assert np.all(np.abs(hs[big] - hc[big]) <= 1e-6 * hc[big])
    # final residuals recomputed as in solver.py:254-255 (at the bottom of the
    # solve they differ by the summation-order noise only)
    assert rs.normal_residual <= 1e-9 and rs.primal_residual <= 2 * rc.primal_residual + 1e-14
    # the loop is one launch: setup + final residual kernels around it only
    assert ls < lc


def test_small_solve_stored_diagonal(monkeypatch):
    from oracle.oracle import StencilOracle
    N, res = 3, (12, 10, 9)
    spec = _field_phase(rand_spec(N, res, 5), 6)
    kw = dict(tol=1e-10, max_iter=3000)
    xs, rs, _ = _solve(spec, N, ALWAYS, monkeypatch, **kw)
    xo, ro = StencilOracle(build_tables(N), spec).cgnr(**kw)
    assert rs.converged and abs(rs.iterations - ro["iterations"]) <= 1
    assert rel(xs, xo) <= 1e-8


def test_small_solve_max_iter_primal_tol_warm_start(monkeypatch):
    from oracle.oracle import StencilOracle
    N, res = 3, (16, 8, 8)
    spec = rand_spec(N, res, 9)
    o = StencilOracle(build_tables(N), spec)
    # stops at max_iter, not converged, histories of max_iter entries
    xs, rs, _ = _solve(spec, N, ALWAYS, monkeypatch, tol=1e-14, max_iter=7)
    xo, ro = o.cgnr(tol=1e-14, max_iter=7)
    assert not rs.converged and rs.iterations == 7 == ro["iterations"] and len(rs.normal_history) == 7
    assert rel(xs, xo) <= 1e-12
    # primal tolerance as a second stop condition
    xs, rs, _ = _solve(spec, N, ALWAYS, monkeypatch, tol=1e-3, primal_tol=1e-9, max_iter=3000)
    xo, ro = o.cgnr(tol=1e-3, primal_tol=1e-9, max_iter=3000)
    assert rs.converged and abs(rs.iterations - ro["iterations"]) <= 1 and rs.primal_residual <= 1e-9
    # warm start from the solution: converges at once
    from paper_1807_00410_b200.solver import PnContext
    monkeypatch.setenv("PNRTE_SMALL_MAX", ALWAYS)
    c = PnContext(build_tables(N), spec.res, spec.h)
    c.set_fields(spec)
    x1, r1 = c.solve(tol=1e-10, max_iter=3000)
    x2, r2 = c.solve(tol=1e-8, max_iter=3000, x0=x1)
    assert r2.iterations <= 1 and rel(x2.cpu().numpy(), x1.cpu().numpy()) <= 1e-9


def test_small_solve_repeatable(monkeypatch):
    """Fixed-order block partials: two solves are bit-identical."""
    N, res = 5, (20, 6, 7)
    spec = rand_spec(N, res, 3)
    a, ra, _ = _solve(spec, N, ALWAYS, monkeypatch, tol=1e-9, max_iter=3000)
    b, rb, _ = _solve(spec, N, ALWAYS, monkeypatch, tol=1e-9, max_iter=3000)
    assert ra.iterations == rb.iterations and a.tobytes() == b.tobytes()


def test_small_solve_falls_back_when_grid_not_resident(monkeypatch):
    """A cooperative grid larger than what is resident (other work on the SMs)
    is refused by the driver; the solve then runs the launch chain on the same
    reference-layout vectors instead of failing."""
    from oracle.oracle import StencilOracle
    N, res = 3, (16, 8, 8)
    spec = rand_spec(N, res, 13)
    monkeypatch.setenv("PNRTE_SMALL_GRID", "2048")   # > 4 CTAs x 148 SMs
    xf, rf, lf = _solve(spec, N, ALWAYS, monkeypatch, tol=1e-10, max_iter=3000)
    monkeypatch.delenv("PNRTE_SMALL_GRID")
    xs, rs, ls = _solve(spec, N, ALWAYS, monkeypatch, tol=1e-10, max_iter=3000)
    xo, ro = StencilOracle(build_tables(N), spec).cgnr(tol=1e-10, max_iter=3000)
    assert rf.converged and abs(rf.iterations - ro["iterations"]) <= 1 and rel(xf, xo) <= 1e-8
    assert lf > ls   # the chain ran
