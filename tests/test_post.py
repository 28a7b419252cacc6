"""Post-processing oracle (oracle/post_oracle.py) pinned against the live
reference (solver.py:299-343, sh.py:33-101, 172-199)."""

import math

import numpy as np
import pytest

from oracle import post_oracle as po
from paper_1807_00410_b200.problems import ProblemSpec


def spec_of(res, h=0.5, origin=None):
    """Cubic-voxel spec with unit fields (only the geometry matters here)."""
    dim = len(res)
    f = {"sigma_t": np.ones(res), "sigma_s": np.zeros(res)}
    return ProblemSpec(dim=dim, origin=origin or (0.0,) * dim, extent=tuple(r * h for r in res), res=tuple(res),
                       fields=f)


def test_real_sh_orthonormal():
    theta, phi, w = po.sphere_quadrature(24, 48)
    lms = [(l, m) for l in range(4) for m in range(-l, l + 1)]
    G = np.zeros((len(lms), len(lms)))
    for a, (l1, m1) in enumerate(lms):
        for b, (l2, m2) in enumerate(lms):
            G[a, b] = sum(w[i, j] * po.real_sh(l1, m1, theta[i, 0], phi[0, j]) * po.real_sh(l2, m2, theta[i, 0],
                                                                                           phi[0, j])
                          for i in range(0, 24, 1) for j in range(0, 48, 1))
    np.testing.assert_allclose(G, np.eye(len(lms)), atol=1e-12)


@pytest.mark.reference
def test_post_oracle_matches_live_reference(ref):
    from pnrte import sh
    from pnrte.solver import reconstruct_radiance, trilinear
    rng = np.random.default_rng(3)
    for l in range(8):
        for m in range(-l, l + 1):
            for _ in range(3):
                th, ph = rng.uniform(0, math.pi), rng.uniform(-math.pi, math.pi)
                assert po.real_sh(l, m, th, ph) == sh.real_sh(l, m, th, ph)
    theta, phi, w = po.sphere_quadrature(8, 16)
    t2, p2, w2 = sh.sphere_quadrature(8, 16)
    assert np.array_equal(theta, t2) and np.array_equal(phi, p2) and np.array_equal(w, w2)
    spec = spec_of((5, 4, 3), origin=(-1.0, -0.5, 0.25))
    coll = rng.normal(size=(5, 4, 3, 9))
    unknowns = [(l, m) for l in range(3) for m in range(-l, l + 1)]
    for _ in range(20):
        x = rng.uniform([-1.0, -0.5, 0.25], [1.5, 1.5, 1.75])
        assert po.trilinear(coll[..., 4], spec, x) == trilinear(coll[..., 4], spec, x)
        om = rng.normal(size=3)
        assert po.reconstruct_radiance(coll, unknowns, spec, x, om) == reconstruct_radiance(coll, unknowns, spec, x,
                                                                                            om)
