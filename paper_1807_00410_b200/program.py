"""P_N staggered-grid stencil tables: the operator definition the kernels run.

The reference turns the P_N moment equations into expression trees
(equations.py:191-210), places every unknown on a staggered grid
(stencil.py:81-123), discretises and factors each row into stencil entries
(stencil.py:142-237) and then interprets those trees over the whole grid in
``assemble`` (solver.py:96-186).  On B200 the trees are not interpreted per
voxel; they are flattened once, on the host, into plain tables:

* one ``Row`` per SH component (comp = l(l+1)+m, equations.py:69-84) with its
  staggered ``location`` (parity per axis, 0 = voxel centre, 1 = +half voxel);
* per row the ``Entry`` list in the reference's order (sorted by target (l,m)
  then doubled-unit offset, stencil.py:231): each entry is either the
  field-dependent diagonal (a sum of product ``Term`` s over sigma_t/sigma_s/p_l
  samples, evaluated in expression-tree order) or a constant transport weight
  ``w * h**-1`` whose target voxel is displaced by at most one voxel along one
  axis;
* per row the residual terms (RHS = -residual, solver.py:177-181).

Two producers of the same tables:

``build_tables(N)``
    a restatement, for 3-D P_N, of build_pn + assign_placement +
    compile_program (no computer algebra: the discretisation rules of
    stencil.py:142-174 are applied directly to the known equation shape).
``tables_from_program(program)``
    reads a reference ``StencilProgram`` (duck-typed walk of its Expr trees,
    cas.py:56-193), which is what the drop-in ``assemble(program, spec)``
    receives.

Both produce bit-identical tables (pinned by tests/test_program.py against the
reference and against tests/golden/tables_N*.json).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

AXES = 3


class PlacementError(Exception):
    """Inconsistent staggered-grid parity (mirrors stencil.py:35)."""


class InvalidOrderError(ValueError):
    """P_N order below 1 (mirrors equations.py:30, raised at :193-194)."""


class UnsupportedProgramError(ValueError):
    """A stencil program outside the matrix-free P_N form (e.g. CDA's
    field-dependent off-diagonals, equations.py:213-237)."""


# ---------------------------------------------------------------------------
# table types
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Term:
    """One product term: ``coef * f0 * f1 ...`` evaluated left to right
    (cas.py:499-503).  ``coef`` None means the product starts at f0.
    factors: ((field_name, (sx, sy, sz)), ...) with voxel-offset sites."""

    coef: float | None
    factors: tuple


@dataclass(frozen=True)
class Entry:
    target: int          # target component index
    target_lm: tuple     # (l, m) of the target
    offset: tuple        # absolute doubled-unit offset (StencilEntry.offset)
    disp: tuple          # voxel displacement of the target sample
    diag: bool           # field-dependent diagonal entry
    weights: tuple       # off-diagonal: value = sum_i (w_i * h**-1), in order
    terms: tuple         # diagonal: sum of Terms, in order


@dataclass(frozen=True)
class Row:
    comp: int
    lm: tuple
    location: tuple      # parity per axis (doubled-unit row location)
    entries: tuple       # reference order
    rhs_terms: tuple     # residual Terms; RHS = -(sum of terms)


@dataclass(frozen=True)
class PnTables:
    N: int
    U: int
    rows: tuple          # indexed by component
    dim: int = 3         # 2-D programs are embedded as nz = 1 grids (z parity / offsets 0)

    @property
    def lm(self):
        return [r.lm for r in self.rows]

    @property
    def parity(self):
        return [r.location for r in self.rows]

    def field_names(self):
        names = set()
        for r in self.rows:
            for e in r.entries:
                for t in e.terms:
                    names.update(f for f, _ in t.factors)
            for t in r.rhs_terms:
                names.update(f for f, _ in t.factors)
        return sorted(names)


# ---------------------------------------------------------------------------
# index maps and SH coupling numbers (restated from equations.py / sh.py)
# ---------------------------------------------------------------------------

def q_name(l, m):
    """Emission field name Q^{l,m} (equations.py:41-43)."""
    return f"Q_{l}_{'n' if m < 0 else ''}{abs(m)}"


def p_name(l):
    """Zonal phase field name p^{l,0} (equations.py:46-48)."""
    return f"p_{l}"


def comp_index(l, m):
    """3-D flat SH index l(l+1)+m (equations.py:77-78)."""
    return l * (l + 1) + m


def num_unknowns(N):
    return (N + 1) ** 2


def lambda_l(l):
    """sqrt(4 pi / (2l+1)) (sh.py:141-143)."""
    return math.sqrt(4.0 * math.pi / (2 * l + 1))


# (numerator, denominator) factor pairs of the six coupling coefficients,
# sh.py:106-138; value = sqrt(num/den), 0 when num == 0.
_COUPLING = {
    "a": (lambda l, m: (l - m + 1) * (l + m + 1), lambda l: (2 * l + 3) * (2 * l + 1)),
    "b": (lambda l, m: (l - m) * (l + m), lambda l: (2 * l + 1) * (2 * l - 1)),
    "c": (lambda l, m: (l + m + 1) * (l + m + 2), lambda l: (2 * l + 3) * (2 * l + 1)),
    "d": (lambda l, m: (l - m) * (l - m - 1), lambda l: (2 * l + 1) * (2 * l - 1)),
    "e": (lambda l, m: (l - m + 1) * (l - m + 2), lambda l: (2 * l + 3) * (2 * l + 1)),
    "f": (lambda l, m: (l + m) * (l + m - 1), lambda l: (2 * l + 1) * (2 * l - 1)),
}


def coupling(kind, l, m):
    num_f, den_f = _COUPLING[kind]
    num, den = num_f(l, m), den_f(l)
    if num == 0:
        return 0.0
    if num * den < 0:
        raise ValueError(f"negative radicand for {kind}^({l},{m})")
    return math.sqrt(num / den)


_SQRT2 = math.sqrt(2.0)
_HALF = 0.5
_INV_SQRT2 = 1.0 / math.sqrt(2.0)


def _beta(axis, m):
    """beta_x / beta_y selectors (sh.py:149-165)."""
    gate, double = (-1, 1) if axis == 0 else (1, -1)
    if m == gate:
        return 0.0
    if m == double:
        return _SQRT2
    return 1.0


def transport_couplings(l, m):
    """(axis, (l_t, m_t), weight) transport couplings of equation (l, m).

    Restates equations.py:116-176 term by term; the float expressions keep
    the reference's evaluation order so the weights are bit-identical.
    """
    out = []

    def emit(axis, lt, mt, w):
        if lt >= 0 and abs(mt) <= lt and w != 0.0:
            out.append((axis, (lt, mt), w))

    if m == 0:
        c = coupling("c", l - 1, -1) if l - 1 >= 1 else 0.0
        d = coupling("d", l + 1, -1)
        a = coupling("a", l - 1, 0) if l >= 1 else 0.0
        b = coupling("b", l + 1, 0)
        for axis, mt in ((0, 1), (1, -1)):
            emit(axis, l - 1, mt, -_INV_SQRT2 * c)
            emit(axis, l + 1, mt, +_INV_SQRT2 * d)
        emit(2, l - 1, 0, a)
        emit(2, l + 1, 0, b)
        return out

    bx, by = _beta(0, m), _beta(1, m)
    mc = m - 1 if m < 0 else -m - 1  # c/d coupling order argument
    me = m + 1 if m < 0 else -m + 1  # e/f coupling order argument
    c = coupling("c", l - 1, mc) if l - 1 >= abs(mc) else 0.0
    d = coupling("d", l + 1, mc)
    e = coupling("e", l - 1, me) if l - 1 >= abs(me) else 0.0
    f = coupling("f", l + 1, me)
    mza = m if m < 0 else -m
    a = coupling("a", l - 1, mza) if l - 1 >= abs(m) else 0.0
    b = coupling("b", l + 1, mza)
    if m < 0:
        emit(0, l - 1, m - 1, -_HALF * c)
        emit(0, l + 1, m - 1, +_HALF * d)
        emit(0, l - 1, m + 1, +_HALF * bx * e)
        emit(0, l + 1, m + 1, -_HALF * bx * f)
        emit(1, l - 1, -m + 1, +_HALF * c)
        emit(1, l + 1, -m + 1, -_HALF * d)
        emit(1, l - 1, -m - 1, +_HALF * by * e)
        emit(1, l + 1, -m - 1, -_HALF * by * f)
    else:
        emit(0, l - 1, m + 1, -_HALF * c)
        emit(0, l + 1, m + 1, +_HALF * d)
        emit(0, l - 1, m - 1, +_HALF * bx * e)
        emit(0, l + 1, m - 1, -_HALF * bx * f)
        emit(1, l - 1, -m - 1, -_HALF * c)
        emit(1, l + 1, -m - 1, +_HALF * d)
        emit(1, l - 1, -m + 1, -_HALF * by * e)
        emit(1, l + 1, -m + 1, +_HALF * by * f)
    emit(2, l - 1, m, a)
    emit(2, l + 1, m, b)
    return out


def scope(N, dim=3):
    """(l, m) carried at order N; the 2-D reduction (z-independence) keeps
    only even l + m (equations.py:51-64)."""
    return [(l, m) for l in range(N + 1) for m in range(-l, l + 1) if dim == 3 or (l + m) % 2 == 0]


def _in_scope(lm, N, dim=3):
    l, m = lm
    return 0 <= l <= N and abs(m) <= l and (dim == 3 or (l + m) % 2 == 0)


# ---------------------------------------------------------------------------
# restated builder
# ---------------------------------------------------------------------------

def _placement(N, dim=3):
    """Per-axis parity 2-colouring of the coupling graph seeded by (0,0) at
    the voxel centre (stencil.py:81-123); 2-D drops the z couplings."""
    unknowns = scope(N, dim)
    edges = []
    for lm in unknowns:
        for axis, tgt, _ in transport_couplings(*lm):
            if dim == 2 and axis == 2:
                continue
            if _in_scope(tgt, N, dim):
                par = tuple(1 if k == axis else 0 for k in range(AXES))
                edges.append((lm, tgt, par))
    off = {unknowns[0]: (0, 0, 0)}
    changed = True
    while changed:
        changed = False
        for a, b, par in edges:
            if a in off and b not in off:
                off[b] = tuple((off[a][k] + par[k]) % 2 for k in range(AXES))
                changed = True
            elif b in off and a not in off:
                off[a] = tuple((off[b][k] + par[k]) % 2 for k in range(AXES))
                changed = True
    for a, b, par in edges:
        want = tuple((off[a][k] + par[k]) % 2 for k in range(AXES))
        if off[b] != want:
            raise PlacementError(f"parity conflict between {a} and {b}")
    for lm in unknowns:
        off.setdefault(lm, (0, 0, 0))
    return off


def _sites(location):
    """Voxel-centre sites averaged at a staggered location, x outermost
    (stencil.py:130-139 with parameters at centres)."""
    sites = [()]
    for p in location:
        if p % 2 == 0:
            sites = [s + (p // 2,) for s in sites]
        else:
            sites = [s + (q,) for s in sites for q in ((p - 1) // 2, (p + 1) // 2)]
    return sites


def comp_index_dim(l, m, N, dim):
    """Flat unknown index: l(l+1)+m in 3-D, the rank among the even-parity
    pairs in (l, m) order in 2-D (equations.py:85-103)."""
    if dim == 3:
        return comp_index(l, m)
    return scope(N, 2).index((l, m))


def build_tables(N, dim=3):
    """Tables of compile_program(build_pn(N, dim)) without computer algebra.
    2-D programs (equations.py:191-210 with dim = 2: odd l + m dropped, no z
    transport) are embedded as nz = 1 grids: z parity 0, z offsets 0."""
    if N < 1:
        raise InvalidOrderError(f"order must be >= 1, got {N}")
    if dim not in (2, 3):
        raise ValueError(f"dim must be 2 or 3, got {dim}")
    unknowns = scope(N, dim)
    place = _placement(N, dim)
    rows = []
    for lm in unknowns:
        l, m = lm
        loc = place[lm]
        # transport: D_axis(L_t) -> (L_t@loc+e - L_t@loc-e) * h^-1; the
        # coefficient of each sample is Num(+-w) * h^-1 (stencil.py:143-151)
        coeffs = {}
        for axis, tgt, w in transport_couplings(l, m):
            if (dim == 2 and axis == 2) or not _in_scope(tgt, N, dim):
                continue
            for sgn in (+1, -1):
                off = tuple(loc[k] + (sgn if k == axis else 0) for k in range(AXES))
                wv = w if sgn > 0 else w * -1.0
                coeffs.setdefault((tgt, off), []).append(wv)
        sites = _sites(loc)
        n = len(sites)
        lam = lambda_l(l)
        # sigma_t L: n terms 1/n * sigma_t@s (bare sample when n == 1)
        terms = [Term(None if n == 1 else 1.0 / n, (("sigma_t", s),)) for s in sites]
        # -lambda_l sigma_s p_l L: coefficient -lambda * (1/n) * (1/n),
        # sigma_s site outer, p site inner (cas.py:332-336 expansion order)
        cst = -1.0 * lam
        if n > 1:
            cst = cst * (1.0 / n) * (1.0 / n)
        for s1 in sites:
            for s2 in sites:
                terms.append(Term(cst, (("sigma_s", s1), (p_name(l), s2))))
        entries = []
        for (tgt, off), ws in coeffs.items():
            home = place[tgt]
            disp = tuple((off[k] - home[k]) // 2 for k in range(AXES))
            entries.append(Entry(comp_index_dim(*tgt, N, dim), tgt, off, disp, False, tuple(ws), ()))
        entries.append(Entry(comp_index_dim(l, m, N, dim), lm, loc, (0, 0, 0), True, (), tuple(terms)))
        entries.sort(key=lambda e: (e.target_lm, e.offset))
        rc = -1.0 if n == 1 else -1.0 * (1.0 / n)
        rhs = tuple(Term(rc, ((q_name(l, m), s),)) for s in sites)
        rows.append(Row(comp_index_dim(l, m, N, dim), lm, loc, tuple(entries), rhs))
    rows.sort(key=lambda r: r.comp)
    return PnTables(N=N, U=len(rows), rows=tuple(rows), dim=dim)


# ---------------------------------------------------------------------------
# reference StencilProgram reader (duck-typed; no import of the reference)
# ---------------------------------------------------------------------------

def _kind(node):
    return type(node).__name__


def _site(pos):
    s = tuple(p // 2 for p in pos)
    return s + (0,) * (AXES - len(s))


def _pad3(t):
    t = tuple(t)
    return t + (0,) * (AXES - len(t))


def _term(node):
    k = _kind(node)
    if k == "FieldSample":
        return Term(None, ((node.name, _site(node.pos)),))
    if k == "Num":
        return Term(float(node.value), ())
    if k != "Mul":
        raise UnsupportedProgramError(f"unsupported coefficient term {node!r}")
    kids = list(node.children)
    coef = None
    if _kind(kids[0]) == "Num":
        coef = float(kids.pop(0).value)
    facs = []
    for c in kids:
        if _kind(c) != "FieldSample" or c.pos is None:
            raise UnsupportedProgramError(f"unsupported factor {c!r}")
        facs.append((c.name, _site(c.pos)))
    return Term(coef, tuple(facs))


def _terms(expr):
    kids = expr.children if _kind(expr) == "Add" else (expr,)
    return tuple(_term(t) for t in kids)


def _hinv_weights(expr):
    """Off-diagonal coefficient Num(w)*h^-1 (or a sum of such)."""
    kids = expr.children if _kind(expr) == "Add" else (expr,)
    ws = []
    for t in kids:
        if (_kind(t) == "Pow" and _kind(t.base) == "Sym"
                and t.base.name == "h" and t.exponent == -1):
            ws.append(1.0)             # w == 1 folds away (cas.py:258-259)
            continue
        ch = getattr(t, "children", ())
        if (_kind(t) != "Mul" or len(ch) != 2 or _kind(ch[0]) != "Num"
                or _kind(ch[1]) != "Pow" or _kind(ch[1].base) != "Sym"
                or ch[1].base.name != "h" or ch[1].exponent != -1):
            raise UnsupportedProgramError(
                f"off-diagonal coefficient is not constant*h^-1: {expr!r}")
        ws.append(float(ch[0].value))
    return tuple(ws)


def tables_from_program(program):
    """Flatten a reference StencilProgram (stencil.py:205-217) into tables."""
    if program.dim not in (2, 3):
        raise UnsupportedProgramError("programs must be 2-D or 3-D")
    U = len(program.rows)
    place = {k: _pad3(v) for k, v in program.placement.offsets.items()}
    rows = []
    for row in program.rows:
        comp = program.unknown_index[row.index]
        loc = _pad3(row.location)
        entries = []
        for e in row.entries:
            home = place[e.target]
            off = _pad3(e.offset)
            disp = tuple((off[k] - home[k]) // 2 for k in range(AXES))
            tc = program.unknown_index[e.target]
            is_diag = tc == comp and disp == (0, 0, 0)
            if is_diag:
                entries.append(Entry(tc, tuple(e.target), off, disp,
                                     True, (), _terms(e.coeff)))
            else:
                if sum(1 for d in disp if d != 0) > 1 or any(abs(d) > 1 for d in disp):
                    raise UnsupportedProgramError("stencil reach beyond one voxel")
                entries.append(Entry(tc, tuple(e.target), off, disp,
                                     False, _hinv_weights(e.coeff), ()))
        res = row.residual
        rhs = () if (_kind(res) == "Num" and float(res.value) == 0.0) else _terms(res)
        rows.append(Row(comp, tuple(row.index), loc, tuple(entries), rhs))
    rows.sort(key=lambda r: r.comp)
    if [r.comp for r in rows] != list(range(U)):
        raise UnsupportedProgramError("component indices are not 0..U-1")
    return PnTables(N=program.N, U=U, rows=tuple(rows), dim=program.dim)


def as_tables(program_or_N, dim=3):
    """Accept an order N (with the problem's dim), our PnTables, or a
    reference StencilProgram."""
    if isinstance(program_or_N, PnTables):
        return program_or_N
    if isinstance(program_or_N, int):
        return build_tables(program_or_N, dim=dim)
    return tables_from_program(program_or_N)


# ---------------------------------------------------------------------------
# canonical-form checks used by the fast (recomputed-diagonal) kernels
# ---------------------------------------------------------------------------

def canonical_diag(tables):
    """True when every diagonal is  sum_s (1/n) sigma_t@s
    + sum_{s1,s2} (-lambda_l/n^2) sigma_s@s1 p_l@s2  over the staggered
    site set of its row: then diag = avg(sigma_t) - lambda_l p_l avg(sigma_s)
    for spatially uniform p_l, which the fast kernels recompute on the fly."""
    if tables.dim != 3 or tables.U != (tables.N + 1) ** 2:
        return False
    ref = build_tables(tables.N)
    for a, b in zip(ref.rows, tables.rows):
        da = [e for e in a.entries if e.diag][0]
        db = [e for e in b.entries if e.diag][0]
        if da.terms != db.terms:
            return False
    return True


def from_json(d):
    """Inverse of to_json (tables of 2-D programs come from fixtures)."""
    def term(t):
        return Term(t[0], tuple((f, tuple(site)) for f, site in t[1]))
    rows = []
    for r in d["rows"]:
        ents = tuple(Entry(e["target"], tuple(e["lm"]), tuple(e["offset"]), tuple(e["disp"]), e["diag"],
                           tuple(e["weights"]), tuple(term(t) for t in e["terms"])) for e in r["entries"])
        rows.append(Row(r["comp"], tuple(r["lm"]), tuple(r["location"]), ents, tuple(term(t) for t in r["rhs"])))
    return PnTables(N=d["N"], U=d["U"], rows=tuple(rows), dim=d.get("dim", 3))


def to_json(tables):
    """Stable JSON-able dump (golden fixture format)."""
    def term(t):
        return [t.coef, [[f, list(s)] for f, s in t.factors]]
    out = {"N": tables.N, "U": tables.U, "rows": []}
    if tables.dim != 3:
        out["dim"] = tables.dim
    for r in tables.rows:
        out["rows"].append({
            "comp": r.comp, "lm": list(r.lm), "location": list(r.location),
            "entries": [{"target": e.target, "lm": list(e.target_lm),
                         "offset": list(e.offset), "disp": list(e.disp),
                         "diag": e.diag, "weights": list(e.weights),
                         "terms": [term(t) for t in e.terms]}
                        for e in r.entries],
            "rhs": [term(t) for t in r.rhs_terms],
        })
    return out


# ---------------------------------------------------------------------------
# flat packing for the C-ABI (include/pnrte_b200.h) and the C oracle
# ---------------------------------------------------------------------------

# direction codes of a one-voxel displacement; 0 = same voxel
DIR_CODES = {(0, 0, 0): 0, (-1, 0, 0): 1, (1, 0, 0): 2, (0, -1, 0): 3,
             (0, 1, 0): 4, (0, 0, -1): 5, (0, 0, 1): 6}
# ascending flat-index order of the voxels a row touches (x fastest):
# z-1 < y-1 < x-1 < same < x+1 < y+1 < z+1  (scipy csr column order)
DIR_RANK = {5: 0, 3: 1, 1: 2, 0: 3, 2: 4, 4: 5, 6: 6}
NEG_DIR = {0: 0, 1: 2, 2: 1, 3: 4, 4: 3, 5: 6, 6: 5}


def field_slots(N_or_tables):
    """Device field slot order: sigma_t, sigma_s, p_0..p_N, Q_lm by comp
    (for a 3-D order N, or for the rows of given tables, e.g. 2-D)."""
    if isinstance(N_or_tables, PnTables):
        t = N_or_tables
        names = ["sigma_t", "sigma_s"] + [p_name(l) for l in range(t.N + 1)]
        return names + [q_name(*r.lm) for r in t.rows]
    N = N_or_tables
    names = ["sigma_t", "sigma_s"] + [p_name(l) for l in range(N + 1)]
    names += [q_name(l, m) for (l, m) in sorted(scope(N), key=lambda lm: comp_index(*lm))]
    return names


def parity_bits(loc):
    return (loc[0] & 1) | ((loc[1] & 1) << 1) | ((loc[2] & 1) << 2)


def site_code(s):
    return (s[0] & 1) | ((s[1] & 1) << 1) | ((s[2] & 1) << 2)


def entry_value(weights, h):
    """Off-diagonal value exactly as cas.evaluate forms it: w * (h ** -1),
    summed left to right when an entry carries several parts."""
    acc = None
    hinv = h ** -1
    for w in weights:
        v = w * hinv
        acc = v if acc is None else acc + v
    return acc


def pack_tables(tables, h):
    """Flatten tables (+ grid spacing h) into int32/float64 numpy arrays."""
    import numpy as np
    U = tables.U
    slots = {n: i for i, n in enumerate(field_slots(tables))}
    par = np.array([parity_bits(r.location) for r in tables.rows], np.int32)
    lam = np.array([lambda_l(r.lm[0]) for r in tables.rows], np.float64)
    lidx = np.array([r.lm[0] for r in tables.rows], np.int32)

    # A rows in ascending column order
    a_ptr, a_tgt, a_dir, a_w, a_diag = [0], [], [], [], []
    # transposed: column c gathers entries (row c', dir of source voxel)
    trans = [[] for _ in range(U)]
    for r in tables.rows:
        ents = []
        for e in r.entries:
            d = DIR_CODES[e.disp]
            val = 0.0 if e.diag else entry_value(e.weights, h)
            ents.append((DIR_RANK[d], e.target, d, val, int(e.diag)))
            trans[e.target].append((DIR_RANK[NEG_DIR[d]], r.comp, NEG_DIR[d], val, int(e.diag)))
        ents.sort()
        for _, t, d, val, dg in ents:
            a_tgt.append(t); a_dir.append(d); a_w.append(val); a_diag.append(dg)
        a_ptr.append(len(a_tgt))
    t_ptr, t_src, t_dir, t_w, t_diag = [0], [], [], [], []
    for c in range(U):
        for _, s, d, val, dg in sorted(trans[c]):
            t_src.append(s); t_dir.append(d); t_w.append(val); t_diag.append(dg)
        t_ptr.append(len(t_src))

    # term programs: diagonal then rhs, each [U+1] ranges into one term pool
    coef, hascoef, nf, fld, site = [], [], [], [], []

    def push(terms):
        for t in terms:
            if len(t.factors) > 2:
                raise UnsupportedProgramError("more than two field factors in a term")
            coef.append(0.0 if t.coef is None else t.coef)
            hascoef.append(0 if t.coef is None else 1)
            nf.append(len(t.factors))
            fs = [slots[f] for f, _ in t.factors] + [0] * (2 - len(t.factors))
            ss = [site_code(s) for _, s in t.factors] + [0] * (2 - len(t.factors))
            for s in (x for _, x in t.factors):
                if any(v not in (0, 1) for v in s):
                    raise UnsupportedProgramError("field site outside {0,1}^3")
            fld.extend(fs); site.extend(ss)

    d_ptr = [0]
    for r in tables.rows:
        push([e for e in r.entries if e.diag][0].terms)
        d_ptr.append(len(coef))
    r_ptr = [len(coef)]
    for r in tables.rows:
        push(r.rhs_terms)
        r_ptr.append(len(coef))
    i32 = lambda a: np.ascontiguousarray(np.array(a, dtype=np.int32))
    f64 = lambda a: np.ascontiguousarray(np.array(a, dtype=np.float64))
    return {
        "N": tables.N, "U": U, "n_fields": len(slots), "par": par, "lam": lam, "lidx": lidx,
        "a_ptr": i32(a_ptr), "a_tgt": i32(a_tgt), "a_dir": i32(a_dir), "a_w": f64(a_w), "a_diag": i32(a_diag),
        "t_ptr": i32(t_ptr), "t_src": i32(t_src), "t_dir": i32(t_dir), "t_w": f64(t_w), "t_diag": i32(t_diag),
        "d_ptr": i32(d_ptr), "r_ptr": i32(r_ptr), "term_coef": f64(coef), "term_hascoef": i32(hascoef),
        "term_nf": i32(nf), "term_f": i32(fld), "term_site": i32(site),
    }
