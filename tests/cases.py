"""Seeded small problems shared by the golden generator and the tests.

Deterministic on every machine (numpy default_rng); no dependency on the
reference, so the GPU box can rebuild the same inputs.
"""

import numpy as np

from paper_1807_00410_b200.problems import ProblemSpec, phase_fields
from paper_1807_00410_b200.program import q_name

# (name, N, res, seed): ragged grids, single voxel, thin slabs, 32-wide rows
# (segmented kernel) and grids above the OpenBLAS 10000-element threading cut
CASES = [
    ("p1_567", 1, (5, 6, 7), 11),
    ("p1_111", 1, (1, 1, 1), 12),
    ("p1_213", 1, (2, 1, 3), 13),
    ("p2_445", 2, (4, 4, 5), 14),
    ("p3_456", 3, (4, 5, 6), 15),
    ("p3_333", 3, (3, 3, 3), 16),
    ("p4_344", 4, (3, 4, 4), 17),
    ("p5_345", 5, (3, 4, 5), 18),
    ("p6_334", 6, (3, 3, 4), 19),
    ("p7_343", 7, (3, 4, 3), 20),
    ("p1_3286", 1, (32, 8, 6), 21),
    ("p3_3245", 3, (32, 4, 5), 22),
    ("p5_3233", 5, (32, 3, 3), 23),
    ("p7_3222", 7, (32, 2, 2), 24),
]


# 2-D programs (checkerboard, problems.py:104-127): (name, N, res); tables
# from the restated 2-D builder (build_tables(N, 2)), the spec from make_checkerboard
CASES_2D = [
    ("cb_p1_15", 1, 15),
    ("cb_p2_15", 2, 15),
    ("cb_p3_21", 3, 21),
]


# Neumann boundaries (bc="neumann": writes redirected into the domain,
# solver.py:133-135,146-147), served by the device CSR assembly
CASES_NEUMANN = [
    ("n_p1_567", 1, (5, 6, 7), 41),
    ("n_p2_445", 2, (4, 4, 5), 42),
    ("n_p3_3245", 3, (32, 4, 5), 43),
    ("n_p5_345", 5, (3, 4, 5), 44),
    ("n_p7_343", 7, (3, 4, 3), 45),
    ("n_p1_111", 1, (1, 1, 1), 46),
]
CASES_NEUMANN_2D = [("ncb_p2_15", 2, 15), ("ncb_p3_21", 3, 21)]
NEUMANN_CASES = [c[0] for c in CASES_NEUMANN] + [c[0] for c in CASES_NEUMANN_2D]


# CDA (collapsed diffusion, equations.py:213-237): field-dependent couplings,
# served by the general-program device assembly.  (name, dim, res or n, seed, bc)
CASES_CDA = [
    ("cda3_654", 3, (6, 5, 4), 51, "dirichlet"),
    ("cda3_654n", 3, (6, 5, 4), 51, "neumann"),
    ("cda3_3274", 3, (32, 7, 4), 54, "dirichlet"),
    ("cda3_111", 3, (1, 1, 1), 53, "dirichlet"),
    ("cda2_cb15", 2, 15, 0, "dirichlet"),
    ("cda2_cb15n", 2, 15, 0, "neumann"),
]
CDA_CASES = [c[0] for c in CASES_CDA]


def cda_inputs(name):
    """(program, spec) of a CDA fixture case (restated program, no reference)."""
    from dataclasses import replace
    from paper_1807_00410_b200.general import build_cda_program
    from paper_1807_00410_b200.problems import make_checkerboard
    for cname, dim, res, seed, bc in CASES_CDA:
        if cname == name:
            spec = rand_spec(1, res, seed) if dim == 3 else make_checkerboard(res)
            return build_cda_program(dim), replace(spec, bc=bc)
    raise KeyError(name)


def tables_2d(N):
    """Restated 2-D builder (equal to the reference fixtures, test_program.py)."""
    from paper_1807_00410_b200.program import build_tables
    return build_tables(N, dim=2)


def rand_spec(N, res, seed, g=0.6, q_frac=0.5, uniform_sigma=False):
    """Heterogeneous sigma_t in [0.5, 20), albedo in [0, 0.99), HG phase g,
    random emission on about q_frac of the (l, m) coefficients."""
    rng = np.random.default_rng(seed)
    if uniform_sigma:
        st = np.full(res, 4.0)
        ss = np.full(res, 3.0)
    else:
        st = rng.uniform(0.5, 20.0, res)
        ss = st * rng.uniform(0.0, 0.99, res)
    f = {"sigma_t": st, "sigma_s": ss}
    f.update(phase_fields(g, N))
    for l in range(N + 1):
        for m in range(-l, l + 1):
            if rng.random() < q_frac:
                f[q_name(l, m)] = rng.normal(size=res)
    return ProblemSpec(dim=3, origin=(0.0, 0.0, 0.0), extent=tuple(r * 0.125 for r in res), res=tuple(res),
                       fields=f)


def probe_vector(R, seed=99):
    return np.random.default_rng(seed).normal(size=R)


ALL_CASES = [c[0] for c in CASES] + [c[0] for c in CASES_2D]


def case_inputs(name):
    """(tables, spec) of a named fixture case, 3-D random or 2-D checkerboard."""
    from paper_1807_00410_b200.problems import make_checkerboard
    from paper_1807_00410_b200.program import build_tables
    for cname, N, res, seed in CASES:
        if cname == name:
            return build_tables(N), rand_spec(N, res, seed)
    for cname, N, n in CASES_2D:
        if cname == name:
            return tables_2d(N), make_checkerboard(n)
    from dataclasses import replace
    for cname, N, res, seed in CASES_NEUMANN:
        if cname == name:
            return build_tables(N), replace(rand_spec(N, res, seed), bc="neumann")
    for cname, N, n in CASES_NEUMANN_2D:
        if cname == name:
            return tables_2d(N), replace(make_checkerboard(n), bc="neumann")
    raise KeyError(name)
