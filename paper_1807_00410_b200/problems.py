"""Solver input contract: the problem container and its admission rules.

Mirrors the reference's ProblemSpec (problems.py:28-70), validate_for_solve
(:78-84) and floor_sigma_t (:87-97) so the drop-in accepts the same objects.
Any object with ``dim``, ``res``, ``extent``, ``h``, ``bc`` and
``field_array(name)`` (the reference's own ProblemSpec included) is accepted
by the solver entry points.

Fields are numpy arrays indexed [i, j, k] (x first, z fastest in memory);
the device upload transposes them once to the x-fastest voxel order of the
unknown vector (solver.py:4-6).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np


class SingularRiskError(RuntimeError):
    """The extinction field contains vacuum (problems.py:23-25)."""


@dataclass(frozen=True)
class ProblemSpec:
    dim: int
    origin: tuple
    extent: tuple
    res: tuple
    fields: dict = field(repr=False)
    bc: str = "dirichlet"
    sigma_t_floor: float = 0.0
    name: str = ""
    # (k0, n_planes): the array fields hold only the global z-planes
    # [k0, k0 + n_planes) (shape (nx, ny, n_planes)) -- one rank's share of a
    # slab decomposition (configs.make_config(..., planes=)); None = whole grid
    z_planes: tuple | None = None

    @property
    def field_shape(self):
        if self.z_planes is None:
            return tuple(self.res)
        return (self.res[0], self.res[1], int(self.z_planes[1]))

    def __post_init__(self):
        hs = {self.extent[k] / self.res[k] for k in range(self.dim)}
        if len(hs) != 1:
            raise ValueError("voxels must be cubic: extent/res equal per axis")
        if self.bc not in ("dirichlet", "neumann"):
            raise ValueError(f"unknown boundary condition {self.bc!r}")
        st, ss = self.fields["sigma_t"], self.fields["sigma_s"]
        if not (np.all(np.isfinite(st)) and np.all(np.isfinite(ss))):
            raise ValueError("non-finite parameter field")
        if np.any(ss > st + 1e-12):
            raise ValueError("sigma_s must not exceed sigma_t")

    @property
    def h(self):
        return self.extent[0] / self.res[0]

    def field_array(self, name):
        if name in self.fields:
            arr = self.fields[name]
            if np.ndim(arr) == 0:
                return np.full(self.field_shape, float(arr))
            return arr
        if name.startswith("p_") or name.startswith("Q_"):
            return np.zeros(self.field_shape)
        raise KeyError(f"unknown parameter field {name!r}")

    def centers(self, axis):
        return self.origin[axis] + (np.arange(self.res[axis]) + 0.5) * self.h


def make_checkerboard(res=71):
    """2-D lattice problem (problems.py:104-127): 7x7 domain, absorbing
    checkerboard on the inner 5x5 blocks, unit isotropic emitter in the centre
    block.  Restated so 2-D fixtures can be rebuilt without the reference."""
    n = res
    xs = (np.arange(n) + 0.5) * (7.0 / n)
    bx = np.floor(xs).astype(int)
    BX, BY = np.meshgrid(bx, bx, indexing="ij")
    absorber = ((BX + BY) % 2 == 0) & (BX >= 1) & (BX <= 5) & (BY >= 1) & (BY <= 5) & ~((BX == 3) & (BY == 3))
    sigma_t = np.where(absorber, 10.0, 1.0)
    sigma_s = np.where(absorber, 0.0, 1.0)
    q00 = np.where((BX == 3) & (BY == 3), 1.0 / math.sqrt(4.0 * math.pi), 0.0)
    fields = {"sigma_t": sigma_t, "sigma_s": sigma_s, "Q_0_0": q00}
    fields.update(phase_fields(0.0, 8))
    return ProblemSpec(dim=2, origin=(0.0, 0.0), extent=(7.0, 7.0), res=(n, n), fields=fields,
                       bc="dirichlet", sigma_t_floor=1.0, name="checkerboard")


def validate_for_solve(spec):
    """Admission: any sigma_t <= 0 makes the system singular."""
    st = np.asarray(spec.field_array("sigma_t"))
    if float(st.min()) <= 0.0:
        raise SingularRiskError(
            "sigma_t contains vacuum (min <= 0); raise the floor "
            "(floor_sigma_t) before solving")


def floor_sigma_t(spec, tau):
    """sigma_t' = max(sigma_t, tau), sigma_s unchanged (problems.py:87-97)."""
    if tau <= 0:
        raise ValueError("floor must be positive")
    fields = dict(spec.fields)
    fields["sigma_t"] = np.maximum(spec.field_array("sigma_t"), tau)
    return replace(spec, fields=fields, sigma_t_floor=tau)


def field_slot(spec, name):
    """(kind, scalar, array) for one device field slot without materialising
    scalars or absent coefficients: kind 0 = zero, 1 = uniform, 2 = array."""
    fields = getattr(spec, "fields", None)
    if fields is not None and name in fields:
        arr = fields[name]
        if np.ndim(arr) == 0:
            return 1, float(arr), None
        arr = np.asarray(arr, dtype=np.float64)
        want = tuple(getattr(spec, "field_shape", spec.res))
        if tuple(arr.shape) != want:
            raise ValueError(f"field {name!r} has shape {arr.shape}, expected {want}")
        return 2, 0.0, arr
    if fields is None:
        arr = np.asarray(spec.field_array(name), dtype=np.float64)
        return 2, 0.0, arr
    if name.startswith("p_") or name.startswith("Q_"):
        return 0, 0.0, None
    raise KeyError(f"unknown parameter field {name!r}")


# ---------------------------------------------------------------------------
# Henyey-Greenstein zonal phase coefficients (sh.py:172-223), restated so the
# configs can be generated where the reference is absent.  The numpy
# expressions keep the reference's order, so the values are bit-identical
# (tests/test_problems.py pins them).
# ---------------------------------------------------------------------------

def _legendre_m0(l, x):
    """P_l(x) by the upward recurrence of sh.py:45-60 at m = 0."""
    pmm = np.ones_like(x)
    if l == 0:
        return pmm
    pmmp1 = x * 1 * pmm
    if l == 1:
        return pmmp1
    for ll in range(2, l + 1):
        pll = (x * (2 * ll - 1) * pmmp1 - (ll - 1) * pmm) / ll
        pmm, pmmp1 = pmmp1, pll
    return pmmp1


def zonal_phase_coefficients(g, N, n_theta=64, n_phi=128):
    """p^{l,0}, l = 0..N, of an HG lobe by Gauss-Legendre x trapezoid
    projection (sh.py:172-199, 210-223)."""
    xg, wx = np.polynomial.legendre.leggauss(n_theta)
    theta = np.arccos(xg)[:, None]
    phi = (np.arange(n_phi) * 2.0 * math.pi / n_phi)[None, :]
    w = wx[:, None] * np.full((1, n_phi), 2.0 * math.pi / n_phi)
    th = theta + 0 * phi
    mu = np.cos(th)
    fv = (1.0 - g * g) / (4.0 * math.pi * (1.0 + g * g - 2.0 * g * mu) ** 1.5)
    xa = np.clip(np.asarray(np.cos(th), dtype=float), -1.0, 1.0)
    out = []
    for l in range(N + 1):
        norm = math.sqrt((2 * l + 1) / (4 * math.pi)
                         * math.factorial(l) / math.factorial(l))
        basis = norm * _legendre_m0(l, xa)
        out.append(float(np.sum(w * fv * basis)))
    return out


def phase_fields(g, N):
    """{p_l: np.float64} as the reference generators store them (:73-75)."""
    return {f"p_{l}": np.float64(c) for l, c in enumerate(zonal_phase_coefficients(g, N))}
