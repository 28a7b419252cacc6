"""ORACLE — TEST INFRASTRUCTURE ONLY (never imported by the product package).

numpy restatement of the reference's assemble() for arbitrary stencil
programs (pkg/src/pnrte/solver.py:96-186) with the expression evaluator of
cas.py:465-517: every coefficient is evaluated over whole numpy grids, the
COO triplets are masked (Dirichlet) or clipped (Neumann) and handed to
scipy's coo_matrix(...).tocsr().  Independent of the device path's postfix
compiler (paper_1807_00410_b200/general.py); pinned against the live
reference and the committed CDA fixtures (tests/golden/cda.npz).
"""

from __future__ import annotations

import numpy as np


def _kind(n):
    return type(n).__name__


def evaluate(e, h, sampler):
    """cas.py:478-517 for Num / Sym(h) / FieldSample / Add / Mul / Pow."""
    k = _kind(e)
    if k == "Num":
        return e.value
    if k == "Sym":
        if e.name != "h":
            raise KeyError(e.name)
        return h
    if k == "FieldSample":
        return sampler(e.name, e.pos)
    if k == "Add":
        acc = evaluate(e.children[0], h, sampler)
        for c in e.children[1:]:
            acc = acc + evaluate(c, h, sampler)
        return acc
    if k == "Mul":
        acc = evaluate(e.children[0], h, sampler)
        for c in e.children[1:]:
            acc = acc * evaluate(c, h, sampler)
        return acc
    if k == "Pow":
        return evaluate(e.base, h, sampler) ** e.exponent
    raise ValueError(f"unsupported node {k}")


def _needed_pad(program):
    pad = 1
    stack = []
    for row in program.rows:
        stack.append(row.residual)
        for e in row.entries:
            pad = max(pad, max(abs(o) // 2 + 1 for o in e.offset))
            stack.append(e.coeff)
    while stack:
        n = stack.pop()
        k = _kind(n)
        if k == "FieldSample" and n.pos is not None:
            pad = max(pad, max(abs(p) // 2 + 1 for p in n.pos))
        elif k in ("Add", "Mul"):
            stack.extend(n.children)
        elif k == "Pow":
            stack.append(n.base)
    return pad


def field_array(spec, name):
    f = spec.fields
    if name in f:
        a = f[name]
        return np.full(spec.res, float(a)) if np.ndim(a) == 0 else np.asarray(a, np.float64)
    if name.startswith("p_") or name.startswith("Q_"):
        return np.zeros(spec.res)
    raise KeyError(name)


def assemble(program, spec):
    """(A csr, Q) exactly as solver.py:96-186 builds them."""
    import scipy.sparse as sp
    res = tuple(spec.res)
    dim = program.dim
    U = len(program.rows)
    R = int(np.prod(res)) * U
    h = spec.h
    pad = _needed_pad(program)
    cache = {}

    def sampler(name, pos):
        if name not in cache:
            cache[name] = np.pad(field_array(spec, name), pad, mode="edge")
        sl = tuple(slice(pad + p // 2, pad + p // 2 + res[k]) for k, p in enumerate(pos))
        return cache[name][sl]

    grids = np.indices(res)

    def flat(*idx):
        out = np.zeros(res, dtype=np.int64)
        stride = 1
        for k in range(dim):
            out = out + idx[k] * stride
            stride *= res[k]
        return out

    vox = flat(*grids)
    neumann = spec.bc == "neumann"
    rows_acc, cols_acc, data_acc = [], [], []
    rhs = np.zeros(R)
    for row in program.rows:
        eq = program.unknown_index[row.index]
        row_ids = (vox * U + eq).ravel()
        row_boundary = None
        if not neumann:
            row_boundary = np.zeros(res, dtype=bool)
            for k in range(dim):
                if row.location[k] == 1:
                    row_boundary |= grids[k] == res[k] - 1
        for e in row.entries:
            coeff = np.broadcast_to(np.asarray(evaluate(e.coeff, h, sampler), dtype=float), res)
            home = program.placement.offsets[e.target]
            disp = [(e.offset[k] - home[k]) // 2 for k in range(dim)]
            t = [grids[k] + disp[k] for k in range(dim)]
            if neumann:
                t = [np.clip(t[k], 0, res[k] - 1) for k in range(dim)]
                mask = None
            else:
                ind = np.ones(res, dtype=bool)
                interior = np.ones(res, dtype=bool)
                for k in range(dim):
                    ind &= (t[k] >= 0) & (t[k] <= res[k] - 1)
                    if home[k] == 1:
                        interior &= t[k] <= res[k] - 2
                if e.target == row.index and all(d == 0 for d in disp):
                    mask = ind
                else:
                    mask = ind & interior & ~row_boundary
                t = [np.clip(t[k], 0, res[k] - 1) for k in range(dim)]
            cols = (flat(*t) * U + program.unknown_index[e.target]).ravel()
            vals = coeff.ravel()
            if mask is not None:
                keep = mask.ravel()
                rows_acc.append(row_ids[keep]); cols_acc.append(cols[keep]); data_acc.append(vals[keep])
            else:
                rows_acc.append(row_ids); cols_acc.append(cols); data_acc.append(vals)
        r = np.broadcast_to(np.asarray(-evaluate(row.residual, h, sampler), dtype=float), res)
        if row_boundary is not None:
            r = np.where(row_boundary, 0.0, r)
        rhs[row_ids] = r.ravel()
    A = sp.coo_matrix((np.concatenate(data_acc), (np.concatenate(rows_acc), np.concatenate(cols_acc))),
                      shape=(R, R)).tocsr()
    return A, rhs


def unstagger(u, program, res):
    """solver.py:275-296."""
    res = tuple(res)
    U = len(program.rows)
    out = np.empty(res + (U,))
    for lm, comp in program.unknown_index.items():
        grid = np.asarray(u)[comp::U].reshape(res, order="F")
        for k in range(program.dim):
            if program.placement.offsets[lm][k] == 1:
                lower = np.concatenate([np.take(grid, [0], axis=k), np.take(grid, range(0, res[k] - 1), axis=k)],
                                       axis=k)
                grid = 0.5 * (grid + lower)
        out[..., comp] = grid
    return out
