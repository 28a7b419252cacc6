"""ORACLE — TEST INFRASTRUCTURE ONLY (never imported by the product package).

Scalar restatement of the reference's post-processing (pkg/src/pnrte/
solver.py:299-343) and of the real spherical-harmonic basis it uses
(sh.py:33-101, complex Condon-Shortley form combined into the real basis).
Pinned against the live reference in tests/test_post.py.
"""

from __future__ import annotations

import math

import numpy as np

SQRT_4PI = math.sqrt(4.0 * math.pi)


def assoc_legendre(l, m, x):
    """Phase-free P^{l,m}(x), 0 <= m <= l (sh.py:33-58)."""
    x = min(max(float(x), -1.0), 1.0)
    somx2 = math.sqrt(1.0 - x * x)
    pmm, fact = 1.0, 1.0
    for _ in range(m):
        pmm = pmm * (fact * somx2)
        fact += 2.0
    if l == m:
        return pmm
    pmmp1 = x * (2 * m + 1) * pmm
    for ll in range(m + 2, l + 1):
        pll = (x * (2 * ll - 1) * pmmp1 - (ll + m - 1) * pmm) / (ll - m)
        pmm, pmmp1 = pmmp1, pll
    return pmmp1


def complex_sh(l, m, theta, phi):
    if m < 0:
        return (-1) ** m * np.conj(complex_sh(l, -m, theta, phi))
    norm = math.sqrt((2 * l + 1) / (4 * math.pi) * math.factorial(l - m) / math.factorial(l + m))
    return (-1) ** m * norm * np.exp(1j * m * phi) * assoc_legendre(l, m, math.cos(theta))


def real_sh(l, m, theta, phi):
    if m == 0:
        return float(np.real(complex_sh(l, 0, theta, phi)))
    if m < 0:
        return float(np.real((1j / math.sqrt(2)) * (complex_sh(l, m, theta, phi)
                                                     - (-1) ** m * complex_sh(l, -m, theta, phi))))
    return float(np.real((1 / math.sqrt(2)) * (complex_sh(l, -m, theta, phi)
                                                + (-1) ** m * complex_sh(l, m, theta, phi))))


def trilinear(comp, spec, x):
    res, h = spec.res, spec.h
    t, i0 = [], []
    for k in range(spec.dim):
        s = (x[k] - spec.origin[k]) / h - 0.5
        s = min(max(s, 0.0), res[k] - 1.0)
        base = min(int(math.floor(s)), res[k] - 2) if res[k] > 1 else 0
        i0.append(base)
        t.append(s - base)
    acc = 0.0
    for corner in range(2 ** spec.dim):
        w = 1.0
        idx = []
        for k in range(spec.dim):
            bit = (corner >> k) & 1
            w *= t[k] if bit else (1.0 - t[k])
            idx.append(min(i0[k] + bit, res[k] - 1))
        acc += w * comp[tuple(idx)]
    return acc


def reconstruct_radiance(coll, unknowns, spec, x, omega):
    omega = np.asarray(omega, dtype=float)
    omega = omega / np.linalg.norm(omega)
    theta = math.acos(max(-1.0, min(1.0, omega[2])))
    phi = math.atan2(omega[1], omega[0])
    val = 0.0
    for comp, (l, m) in enumerate(unknowns):
        val += trilinear(coll[..., comp], spec, x) * real_sh(l, m, theta, phi)
    return val


def sphere_quadrature(n_theta, n_phi):
    """Gauss-Legendre in cos(theta) x trapezoid in phi (sh.py:172-199)."""
    xg, wx = np.polynomial.legendre.leggauss(n_theta)
    theta = np.arccos(xg)[:, None]
    phi = (np.arange(n_phi) * 2.0 * math.pi / n_phi)[None, :]
    w = wx[:, None] * np.full((1, n_phi), 2.0 * math.pi / n_phi)
    return theta, phi, w
