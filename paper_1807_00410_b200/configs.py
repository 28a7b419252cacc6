"""Seeded synthetic inputs for the five BASELINE.json configurations.

There is no dataset: every configuration is procedural.  Generators follow
SURVEY.md s8(d) (choices marked [decision] there are restated here), use the
reference's RNG (``np.random.default_rng(seed)``, problems.py:174), extent 2
(h = 2/n) and vacuum (Dirichlet) boundaries.  Fields are [i, j, k] C-order
float64 like the reference's generators (problems.py:3-4); p_l come from the
quadrature projection (sh.py:220-223) as np.float64 scalars.

  cfg 1  P1 32^3  homogeneous sigma_t=8, albedo 0.9, g=0, unit source in the
         2^3 centre voxels [15,16]^3 (power-preserving, problems.py:145)
  cfg 2  P3 64^3  sigma_t = 1 + 19*box3(u), albedo U[0.5,0.99), g=0.3,
         Gaussian blob sigma=4 voxels at 31.5 (unit power, problems.py:204)
  cfg 3  P5 128^3 4-octave value noise (period 32), cut 0.4, sigma_t<=50,
         albedo 0.95, g=0.6, z=0 emission slab Q_l0 = p_l(g=0.9)
  cfg 4  P7 256^3 same noise with period 64, sigma_t<=100, albedo 0.99,
         g=0.8, four 2^3 emitters at rng.integers(8,248,(4,3))
  cfg 5  P5 512^3 cfg-3 generator at 512^3, fixed 200 iterations
Configs 3-5 contain vacuum (sigma_t = 0); converging solves use
floor_sigma_t(spec, 1.0) (problems.py:87-97), throughput runs need no floor.

Configs 3-5 take ``planes=(k0, k1)``: only the global z-planes [k0, k1) of
every field are generated (the spec's ``z_planes``), bit-identical to the
same planes of the whole grid -- the random draws are the small noise
lattices and emitter positions, consumed in the same order either way.  A
rank of a slab decomposition generates just its share (config 5: 1.07 GB
per 512^3 field).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .problems import ProblemSpec, floor_sigma_t, phase_fields
from .program import q_name

SQRT_4PI = math.sqrt(4.0 * math.pi)


@dataclass(frozen=True)
class Config:
    index: int
    N: int
    spec: ProblemSpec
    tol: float
    max_iter: int
    floor: float | None      # sigma_t floor for converging solves
    description: str


def _spec(n, fields, name, planes=None):
    zp = None if planes is None else (int(planes[0]), int(planes[1]) - int(planes[0]))
    return ProblemSpec(dim=3, origin=(-1.0,) * 3, extent=(2.0,) * 3, res=(n, n, n),
                       fields=fields, bc="dirichlet", name=name, z_planes=zp)


def _zrange(n, planes):
    k0, k1 = (0, n) if planes is None else (int(planes[0]), int(planes[1]))
    if not (0 <= k0 < k1 <= n):
        raise ValueError(f"planes {planes} outside 0..{n}")
    return k0, k1


def _shape3(n):
    return (int(n),) * 3 if np.ndim(n) == 0 else tuple(int(v) for v in n)


def value_noise(rng, n, cells, planes=None):
    """Trilinear interpolation of a seeded (cells+1)^3 lattice, the pattern of
    problems.py:178-192 (z-planes [k0, k1) only when ``planes`` is given).
    ``n`` / ``cells`` may be per-axis triples (box grids of the weak-scaling
    workload); scalars give the cubic configs."""
    shape, cl = _shape3(n), _shape3(cells)
    k0, k1 = _zrange(shape[2], planes)
    lattice = rng.random(tuple(c + 1 for c in cl))
    ax = []
    for m, c in zip(shape, cl):
        t = np.linspace(0.0, c, m, endpoint=False)
        i0 = np.floor(t).astype(int)
        ax.append((i0, t - i0, np.minimum(i0 + 1, c)))
    (ix0, frx, ix1), (iy0, fry, iy1), (iz0, frz, iz1) = ax
    out = np.zeros((shape[0], shape[1], k1 - k0))
    fx, fy, fz = frx[:, None, None], fry[None, :, None], frz[None, None, k0:k1]
    for dx, wx in ((ix0, 1 - fx), (ix1, fx)):
        for dy, wy in ((iy0, 1 - fy), (iy1, fy)):
            for dz, wz in ((iz0[k0:k1], 1 - fz), (iz1[k0:k1], fz)):
                out += (wx * wy * wz) * lattice[np.ix_(dx, dy, dz)]
    return out


def cloud_density(rng, n, base_period, octaves=4, persistence=0.5, cut=0.4, planes=None):
    shape = _shape3(n)
    k0, k1 = _zrange(shape[2], planes)
    amps = [persistence ** o for o in range(octaves)]
    noise = np.zeros((shape[0], shape[1], k1 - k0))
    for o in range(octaves):
        cells = tuple(max(1, (m * (2 ** o)) // base_period) for m in shape)
        noise += amps[o] * value_noise(rng, shape, cells, planes)
    noise /= sum(amps)
    return np.clip((noise - cut) / (1.0 - cut), 0.0, 1.0)


def config1(seed=0, n=32):
    h = 2.0 / n
    q = np.zeros((n, n, n))
    c = n // 2
    q[c - 1:c + 1, c - 1:c + 1, c - 1:c + 1] = 1.0 / (8 * h ** 3 * SQRT_4PI)
    fields = {"sigma_t": np.full((n,) * 3, 8.0), "sigma_s": np.full((n,) * 3, 7.2),
              q_name(0, 0): q}
    fields.update(phase_fields(0.0, 1))
    return Config(1, 1, _spec(n, fields, "cfg1"), 1e-6, 50000, None,
                  f"P1 {n}^3 homogeneous sigma_t=8 albedo=0.9 g=0 centre source")


def config2(seed=0, n=64):
    from scipy.ndimage import uniform_filter
    rng = np.random.default_rng(seed)
    u = rng.random((n,) * 3)
    st = 1.0 + 19.0 * uniform_filter(u, 3, mode="nearest")
    albedo = rng.uniform(0.5, 0.99, (n,) * 3)
    h = 2.0 / n
    idx = np.arange(n) - (n / 2 - 0.5)
    r2 = idx[:, None, None] ** 2 + idx[None, :, None] ** 2 + idx[None, None, :] ** 2
    blob = np.exp(-r2 / (2 * 4.0 ** 2))
    q = blob / (blob.sum() * h ** 3 * SQRT_4PI)
    fields = {"sigma_t": st, "sigma_s": albedo * st, q_name(0, 0): q}
    fields.update(phase_fields(0.3, 3))
    return Config(2, 3, _spec(n, fields, "cfg2"), 1e-6, 50000, None,
                  f"P3 {n}^3 heterogeneous box-filtered sigma_t in [1,20] albedo U[0.5,0.99) g=0.3")


def config3(seed=0, n=128, base_period=None, planes=None):
    N = 5
    k0, k1 = _zrange(n, planes)
    rng = np.random.default_rng(seed)
    bp = base_period if base_period is not None else max(1, n // 4)
    st = 50.0 * cloud_density(rng, n, bp, planes=planes)
    fields = {"sigma_t": st, "sigma_s": 0.95 * st}
    pe = phase_fields(0.9, N)
    for l in range(N + 1):
        q = np.zeros((n, n, k1 - k0))
        if k0 == 0:
            q[:, :, 0] = float(pe[f"p_{l}"])
        fields[q_name(l, 0)] = q
    fields.update(phase_fields(0.6, N))
    return Config(3, N, _spec(n, fields, "cfg3", planes), 1e-6, 50000, 1.0,
                  f"P5 {n}^3 4-octave cloud (period {bp}) sigma_t in [0,50] albedo 0.95 g=0.6 z=0 slab")


def config4(seed=0, n=256, planes=None):
    N = 7
    k0, k1 = _zrange(n, planes)
    rng = np.random.default_rng(seed)
    st = 100.0 * cloud_density(rng, n, max(1, n // 4), planes=planes)
    h = 2.0 / n
    q = np.zeros((n, n, k1 - k0))
    lo, hi = (8, n - 8) if n > 24 else (0, n - 1)
    for (i, j, k) in rng.integers(lo, hi, (4, 3)):
        for kk in range(k, k + 2):        # emitters overlapping [k0, k1)
            if k0 <= kk < k1:
                q[i:i + 2, j:j + 2, kk - k0] += 1.0 / (8 * h ** 3 * SQRT_4PI)
    fields = {"sigma_t": st, "sigma_s": 0.99 * st, q_name(0, 0): q}
    fields.update(phase_fields(0.8, N))
    return Config(4, N, _spec(n, fields, "cfg4", planes), 1e-6, 50000, 1.0,
                  f"P7 {n}^3 4-octave cloud sigma_t in [0,100] albedo 0.99 g=0.8 four 2^3 emitters")


def config5(seed=0, n=512, planes=None):
    c = config3(seed=seed, n=n, base_period=n // 4, planes=planes)
    return Config(5, 5, c.spec, 1e-300, 200, None,
                  f"P5 {n}^3 cfg-3 generator, fixed 200 iterations")


def weak_config(k, seed=0, n=256, planes=None):
    """Weak-scaling companion of config 5: the config-3
    generator (P5, cloud cut 0.4, sigma_t <= 50, albedo 0.95, g = 0.6, z = 0
    emission slab) on an (n, n, n k) box with the h of n^3 (h = 2/n), noise
    base period n/4 -- k GPUs each own one n^3 slab.  Fixed 200 iterations."""
    N = 5
    shape = (n, n, n * k)
    k0, k1 = _zrange(shape[2], planes)
    rng = np.random.default_rng(seed)
    st = 50.0 * cloud_density(rng, shape, max(1, n // 4), planes=planes)
    fields = {"sigma_t": st, "sigma_s": 0.95 * st}
    pe = phase_fields(0.9, N)
    for l in range(N + 1):
        q = np.zeros((n, n, k1 - k0))
        if k0 == 0:
            q[:, :, 0] = float(pe[f"p_{l}"])
        fields[q_name(l, 0)] = q
    fields.update(phase_fields(0.6, N))
    zp = None if planes is None else (k0, k1 - k0)
    h = 2.0 / n
    spec = ProblemSpec(dim=3, origin=(-1.0,) * 3, extent=(2.0, 2.0, h * n * k), res=shape, fields=fields,
                       bc="dirichlet", name=f"weak{k}", z_planes=zp)
    return Config(0, N, spec, 1e-300, 200, None, f"P5 {n}x{n}x{n * k} cfg-3 generator (weak scaling, {k} GPUs)")


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make_config(index, **kw):
    return CONFIGS[index](**kw)


def solve_spec(cfg):
    """The spec a converging solve uses (floored when the config has vacuum)."""
    return floor_sigma_t(cfg.spec, cfg.floor) if cfg.floor else cfg.spec
