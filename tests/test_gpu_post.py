"""Post-processing on the device (solver.py:299-343):
fluence and trilinear interpolation bit-identical to the reference's
arithmetic, radiance reconstruction within rounding of the libm-based
basis; the reference's own reconstruction tests (test_solver.py:208-268)."""

import math

import numpy as np
import pytest

from oracle import post_oracle as po
from paper_1807_00410_b200.program import build_tables
from test_post import spec_of

pytestmark = pytest.mark.gpu

SQRT_4PI = math.sqrt(4 * math.pi)


def test_fluence_bit_exact():
    from paper_1807_00410_b200.solver import fluence
    coll = np.random.default_rng(1).normal(size=(7, 6, 5, 16))
    assert fluence(coll).tobytes() == (SQRT_4PI * coll[..., 0]).tobytes()
    c2 = np.random.default_rng(2).normal(size=(9, 8, 3))
    assert fluence(c2).tobytes() == (SQRT_4PI * c2[..., 0]).tobytes()


@pytest.mark.parametrize("res", [(5, 4, 3), (1, 6, 2), (9, 7)])
def test_trilinear_bit_exact(res):
    from paper_1807_00410_b200.solver import trilinear
    spec = spec_of(res, origin=tuple(-0.25 * (k + 1) for k in range(len(res))))
    rng = np.random.default_rng(len(res))
    grid = rng.normal(size=res)
    lo = np.asarray(spec.origin)
    hi = lo + np.asarray(spec.extent)
    pts = rng.uniform(lo - 0.1, hi + 0.1, size=(400, len(res)))   # includes the clamped rim and beyond
    pts[:5] = lo
    pts[5:10] = hi
    got = trilinear(grid, spec, pts)
    want = np.array([po.trilinear(grid, spec, p) for p in pts])
    assert got.tobytes() == want.tobytes()
    assert trilinear(grid, spec, pts[17]) == want[17]


def test_reconstruct_matches_oracle_batched():
    from paper_1807_00410_b200.solver import reconstruct_radiance, unknown_order
    spec = spec_of((6, 5, 4), origin=(-1.0, 0.0, 0.5))
    unknowns = unknown_order(build_tables(5))
    rng = np.random.default_rng(5)
    coll = rng.normal(size=(6, 5, 4, len(unknowns)))
    lo = np.asarray(spec.origin)
    pts = rng.uniform(lo, lo + np.asarray(spec.extent), size=(40, 3))
    dirs = rng.normal(size=(24, 3))
    dirs[0] = (0, 0, 1)
    dirs[1] = (0, 0, -2)
    dirs[2] = (1, 0, 0)
    got = reconstruct_radiance(coll, unknowns, spec, pts, dirs)
    want = np.array([[po.reconstruct_radiance(coll, unknowns, spec, p, d) for d in dirs] for p in pts])
    scale = np.abs(want).max()
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-13 * scale)


def test_reconstruct_constant_field_unit_radiance():
    """test_solver.py:208-222."""
    from paper_1807_00410_b200.solver import reconstruct_radiance, unknown_order
    spec = spec_of((4, 4, 4), h=0.25)
    coll = np.zeros((4, 4, 4, 4))
    coll[..., 0] = math.sqrt(4 * math.pi)
    rng = np.random.default_rng(7)
    for _ in range(10):
        val = reconstruct_radiance(coll, unknown_order(1), spec, rng.uniform(0.1, 0.9, 3), rng.normal(size=3))
        assert val == pytest.approx(1.0, rel=1e-12)


def test_reconstruct_fluence_integral():
    """test_solver.py:225-244, batched over the quadrature directions."""
    from paper_1807_00410_b200.solver import fluence, reconstruct_radiance, unknown_order
    spec = spec_of((3, 3, 3), h=1 / 3)
    coll = np.random.default_rng(8).normal(size=(3, 3, 3, 9))
    theta, phi, w = po.sphere_quadrature(32, 64)
    th = np.broadcast_to(theta, w.shape).ravel()
    ph = np.broadcast_to(phi, w.shape).ravel()
    dirs = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], axis=1)
    rad = reconstruct_radiance(coll, unknown_order(2), spec, np.array([[0.5, 0.5, 0.5]]), dirs)
    total = float(np.sum(w.ravel() * rad[0]))
    assert total == pytest.approx(fluence(coll)[1, 1, 1], abs=1e-8)


def test_reconstruct_at_center_is_basis_dot():
    """test_solver.py:247-259."""
    from paper_1807_00410_b200.solver import reconstruct_radiance, unknown_order
    spec = spec_of((4, 4, 4), h=0.25)
    coll = np.random.default_rng(9).normal(size=(4, 4, 4, 4))
    unknowns = unknown_order(1)
    x = tuple(spec.centers(k)[2] for k in range(3))
    omega = (0.3, -0.5, 0.9)
    got = reconstruct_radiance(coll, unknowns, spec, x, omega)
    th = math.acos(omega[2] / np.linalg.norm(omega))
    ph = math.atan2(omega[1], omega[0])
    want = sum(coll[2, 2, 2, c] * po.real_sh(l, m, th, ph) for c, (l, m) in enumerate(unknowns))
    assert got == pytest.approx(want, rel=1e-12)


def test_reconstruct_out_of_domain_errors():
    from paper_1807_00410_b200.solver import OutOfDomainError, reconstruct_radiance, unknown_order
    spec = spec_of((4, 4, 4), h=0.25)
    with pytest.raises(OutOfDomainError):
        reconstruct_radiance(np.zeros((4, 4, 4, 4)), unknown_order(1), spec, (1.5, 0.5, 0.5), (0, 0, 1))


def test_device_tensors_stay_on_device():
    import torch
    from paper_1807_00410_b200.solver import fluence, reconstruct_radiance, unknown_order
    spec = spec_of((4, 4, 4), h=0.25)
    coll = torch.randn(4, 4, 4, 4, dtype=torch.float64, device="cuda")
    f = fluence(coll)
    assert f.is_cuda and torch.equal(f, SQRT_4PI * coll[..., 0])
    r = reconstruct_radiance(coll, unknown_order(1), spec, np.full((3, 3), 0.5), np.eye(3))
    assert r.is_cuda and tuple(r.shape) == (3, 3)
