"""Input contract and config generators."""

import hashlib

import numpy as np
import pytest

from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.problems import (ProblemSpec, SingularRiskError, field_slot, floor_sigma_t,
                                            validate_for_solve, zonal_phase_coefficients)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a)).tobytes()).hexdigest()


@pytest.mark.reference
def test_phase_coefficients_bit_identical(ref):
    from pnrte.sh import zonal_phase_coefficients as z
    for g in (0.0, 0.3, 0.6, 0.8, 0.9):
        assert zonal_phase_coefficients(g, 8) == z(g, 8)


@pytest.mark.parametrize("idx", [1, 2])
def test_config_fields_pinned(idx, golden):
    cfg = make_config(idx)
    want = golden["configs"][f"cfg{idx}"]["fields_sha256"]
    assert {k: sha(v) for k, v in sorted(cfg.spec.fields.items())} == want


@pytest.mark.parametrize("idx", [3, 4])
def test_small_cloud_configs_pinned(idx, golden):
    cfg = make_config(idx, n=32)
    want = golden["configs"][f"cfg{idx}_n32_fields_sha256"]
    assert {k: sha(v) for k, v in sorted(cfg.spec.fields.items())} == want
    st = cfg.spec.fields["sigma_t"]
    assert 0.0 < float(np.mean(st == 0.0)) < 0.9      # genuine vacuum
    with pytest.raises(SingularRiskError):
        validate_for_solve(cfg.spec)
    validate_for_solve(solve_spec(cfg))


def test_spec_validation_mirrors_reference():
    f = {"sigma_t": np.ones((2, 2, 2)), "sigma_s": np.full((2, 2, 2), 2.0)}
    with pytest.raises(ValueError):
        ProblemSpec(3, (0, 0, 0), (1, 1, 1), (2, 2, 2), f)
    f = {"sigma_t": np.ones((2, 2, 2)), "sigma_s": np.zeros((2, 2, 2))}
    with pytest.raises(ValueError):
        ProblemSpec(3, (0, 0, 0), (1, 2, 1), (2, 2, 2), f)
    s = ProblemSpec(3, (0, 0, 0), (1, 1, 1), (2, 2, 2), f)
    assert field_slot(s, "Q_0_0") == (0, 0.0, None)
    with pytest.raises(KeyError):
        field_slot(s, "bogus")
    with pytest.raises(ValueError):
        floor_sigma_t(s, 0.0)
    fl = floor_sigma_t(s, 3.0)
    assert np.all(fl.field_array("sigma_t") == 3.0) and fl.sigma_t_floor == 3.0


@pytest.mark.reference
@pytest.mark.parametrize("n", [15, 21, 71])
def test_checkerboard_generator_bit_identical(n, ref):
    from pnrte.problems import make_checkerboard as ref_cb
    from paper_1807_00410_b200.problems import make_checkerboard
    a, b = make_checkerboard(n), ref_cb(n)
    assert a.res == b.res and a.extent == b.extent and a.dim == b.dim == 2
    for k in b.fields:
        assert np.asarray(a.fields[k]).tobytes() == np.asarray(b.fields[k]).tobytes(), k


@pytest.mark.parametrize("idx,n", [(3, 32), (4, 32), (5, 24)])
def test_slab_generation_equals_planes_of_the_grid(idx, n):
    """configs.make_config(..., planes=(k0, k1)) generates exactly the global
    z-planes [k0, k1) of every field (one rank's share of a slab run)."""
    from paper_1807_00410_b200.configs import make_config
    full = make_config(idx, n=n)
    for k0, k1 in ((0, 5), (3, 17), (n - 6, n), (0, n)):
        part = make_config(idx, n=n, planes=(k0, k1))
        assert part.spec.z_planes == (k0, k1 - k0)
        for name, v in full.spec.fields.items():
            w = part.spec.fields[name]
            if np.ndim(v) == 0:
                assert w == v
            else:
                assert np.ascontiguousarray(np.asarray(v)[:, :, k0:k1]).tobytes() == np.ascontiguousarray(w).tobytes()


def test_package_exports_the_reference_solve_path_names():
    """The package root mirrors the solve-path names of pnrte/__init__.py:17-25
    (importing does no CUDA work)."""
    import paper_1807_00410_b200 as pkg
    for name in ("ProblemSpec", "floor_sigma_t", "make_checkerboard", "SolveReport", "SolutionField", "SparseSystem",
                 "assemble", "fluence", "reconstruct_radiance", "solve_normal_cg", "unstagger", "solve_pn"):
        assert hasattr(pkg, name), name
    f = pkg.SolutionField(staggered=None, collocated=None, unknowns=[(0, 0)], spec=None, report=pkg.SolveReport())
    assert f.report.iterations == 0 and not f.report.converged
