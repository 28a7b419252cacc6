"""General stencil programs: field-dependent coefficients on the device.

The matrix-free P_N kernels assume every off-diagonal coefficient is a
constant times h^-1.  Programs outside that form --
the collapsed diffusion (CDA) system of equations.py:213-237, whose
couplings are -(1.5 sigma_t@a + 1.5 sigma_t@b)^-1 h^-2 -- are assembled
here into an explicit device CSR system (pn_assemble_general) and solved by
the CSR operator.

Every coefficient, diagonal and residual expression is compiled into a small
postfix program evaluated per voxel on the device with the reference's
arithmetic (cas.py:465-517 evaluated over numpy arrays, solver.py:115-123):

  * field-free subtrees (h powers, numeric factors) are folded here with
    Python scalar arithmetic, exactly as ``evaluate`` computes them;
  * n-ary Add / Mul fold left to right; a leading run of scalar operands is
    folded first (the reference's accumulator is still a Python scalar
    there), every later operand is one IEEE op on the array;
  * ``array ** e`` follows numpy's fast paths: -1 -> reciprocal, 2 -> square,
    0.5 -> sqrt, 1 -> identity, 0 -> ones; other exponents go through libm
    pow and are rejected (no bit-exact device equivalent);
  * FieldSample(name, pos) reads the voxel (i, j, k) + pos // 2 with edge
    replication (solver.py:62-64, 118-123).

Programs are accepted duck-typed: the reference's StencilProgram or the
restated ``build_cda_program`` below.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .program import UnsupportedProgramError

AXES = 3

OP_END, OP_NUM, OP_FIELD, OP_ADD, OP_MUL, OP_RECIP, OP_SQUARE, OP_SQRT, OP_ONE = range(9)
MAX_STACK = 16


# ---------------------------------------------------------------------------
# minimal expression / program types (same attribute names as cas.py / stencil.py)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Num:
    value: float


@dataclass(frozen=True)
class Sym:
    name: str


@dataclass(frozen=True)
class FieldSample:
    name: str
    pos: tuple


@dataclass(frozen=True)
class Add:
    children: tuple


@dataclass(frozen=True)
class Mul:
    children: tuple


@dataclass(frozen=True)
class Pow:
    base: object
    exponent: object


@dataclass(frozen=True)
class StencilEntry:
    target: tuple
    offset: tuple
    coeff: object


@dataclass(frozen=True)
class StencilRow:
    index: tuple
    location: tuple
    entries: tuple
    residual: object


@dataclass(frozen=True)
class Placement:
    offsets: dict


@dataclass(frozen=True)
class StencilProgram:
    N: int
    dim: int
    rows: tuple
    unknown_index: dict
    placement: Placement


def build_cda_program(dim=3):
    """compile_program(build_cda(dim)) restated: one cell-centred unknown
    L^{0,0}; per axis the neighbour couplings -(1.5 sigma_t@a + 1.5
    sigma_t@b)^-1 h^-1 h^-1 and a diagonal that sums the six (four in 2-D)
    face terms, + sigma_t - lambda_0 sigma_s p_0; residual -Q_0_0.
    Entries ordered by offset (stencil.py row compilation); expression trees
    as the reference's CAS leaves them (tests pin them against it)."""
    if dim not in (2, 3):
        raise ValueError("CDA programs are 2-D or 3-D")
    zero = (0,) * dim
    hinv = Pow(Sym("h"), -1)

    def at(axis, d):
        return tuple(d if k == axis else 0 for k in range(dim))

    def face(a, b):
        return Pow(Add((Mul((Num(1.5), FieldSample("sigma_t", a))), Mul((Num(1.5), FieldSample("sigma_t", b))))), -1)

    def lo(axis):
        return face(at(axis, -2), zero)

    def hi(axis):
        return face(zero, at(axis, 2))

    entries = {}
    for axis in range(dim):
        entries[at(axis, -2)] = Mul((Num(-1.0), lo(axis), hinv, hinv))
        entries[at(axis, 2)] = Mul((Num(-1.0), hi(axis), hinv, hinv))
    diag_terms = []
    for axis in range(dim):
        diag_terms.append(Mul((hi(axis), hinv, hinv)))
        diag_terms.append(Mul((lo(axis), hinv, hinv)))
    lam0 = math.sqrt(4.0 * math.pi / 1)
    diag_terms.append(FieldSample("sigma_t", zero))
    diag_terms.append(Mul((Num(-1.0 * lam0), FieldSample("sigma_s", zero), FieldSample("p_0", zero))))
    entries[zero] = Add(tuple(diag_terms))
    ents = tuple(StencilEntry((0, 0), off, entries[off]) for off in sorted(entries))
    row = StencilRow((0, 0), zero, ents, Mul((Num(-1.0), FieldSample("Q_0_0", zero))))
    return StencilProgram(N=0, dim=dim, rows=(row,), unknown_index={(0, 0): 0},
                          placement=Placement({(0, 0): zero}))


# ---------------------------------------------------------------------------
# expression -> postfix program
# ---------------------------------------------------------------------------

def _kind(n):
    return type(n).__name__


def _has_field(n):
    k = _kind(n)
    if k == "FieldSample":
        return True
    if k in ("Add", "Mul"):
        return any(_has_field(c) for c in n.children)
    if k == "Pow":
        return _has_field(n.base)
    if k in ("Num", "Sym"):
        return False
    raise UnsupportedProgramError(f"unsupported node in a coefficient: {k}")


def _scalar(n, h):
    """Python-scalar evaluation of a field-free subtree (cas.py:478-505)."""
    k = _kind(n)
    if k == "Num":
        return n.value
    if k == "Sym":
        if n.name != "h":
            raise UnsupportedProgramError(f"unbound symbol {n.name!r}")
        return h
    if k == "Add":
        acc = _scalar(n.children[0], h)
        for c in n.children[1:]:
            acc = acc + _scalar(c, h)
        return acc
    if k == "Mul":
        acc = _scalar(n.children[0], h)
        for c in n.children[1:]:
            acc = acc * _scalar(c, h)
        return acc
    if k == "Pow":
        return _scalar(n.base, h) ** n.exponent
    raise UnsupportedProgramError(f"unsupported node {k}")


_POW_OPS = {-1: OP_RECIP, 2: OP_SQUARE, 0.5: OP_SQRT}


class _Emitter:
    def __init__(self, h, dim):
        self.h = h
        self.dim = dim
        self.ops = []
        self.consts = []
        self.samples = {}
        self.fields = {}
        self.depth = 0
        self.max_depth = 0

    def _push(self, op, arg):
        self.ops += [op, arg]
        if op in (OP_NUM, OP_FIELD):
            self.depth += 1
            self.max_depth = max(self.max_depth, self.depth)
        elif op in (OP_ADD, OP_MUL):
            self.depth -= 1

    def num(self, v):
        self.consts.append(float(v))
        self._push(OP_NUM, len(self.consts) - 1)

    def sample(self, node):
        if node.pos is None:
            raise UnsupportedProgramError("field sample without a position")
        pos = tuple(node.pos) + (0,) * (AXES - len(node.pos))
        off = tuple(p // 2 for p in pos)
        slot = self.fields.setdefault(node.name, len(self.fields))
        key = (slot,) + off
        idx = self.samples.setdefault(key, len(self.samples))
        self._push(OP_FIELD, idx)

    def emit(self, n):
        if not _has_field(n):
            self.num(_scalar(n, self.h))
            return
        k = _kind(n)
        if k == "FieldSample":
            self.sample(n)
        elif k in ("Add", "Mul"):
            op = OP_ADD if k == "Add" else OP_MUL
            kids = list(n.children)
            if not _has_field(kids[0]):
                # the accumulator stays a Python scalar until the first array operand
                acc = _scalar(kids.pop(0), self.h)
                while kids and not _has_field(kids[0]):
                    v = _scalar(kids.pop(0), self.h)
                    acc = acc + v if op == OP_ADD else acc * v
                self.num(acc)
            else:
                self.emit(kids.pop(0))
            for c in kids:
                self.emit(c)
                self._push(op, 0)
        elif k == "Pow":
            e = n.exponent
            self.emit(n.base)
            if e == 1:
                return
            if e == 0:
                self._push(OP_ONE, 0)
                return
            if e not in _POW_OPS:
                raise UnsupportedProgramError(f"array ** {e!r} has no bit-exact device form")
            self._push(_POW_OPS[e], 0)
        else:
            raise UnsupportedProgramError(f"unsupported node {k}")

    def code(self, n):
        start = len(self.ops) // 2
        self.depth = 0
        self.emit(n)
        self.ops += [OP_END, 0]
        if self.max_depth > MAX_STACK:
            raise UnsupportedProgramError("coefficient expression too deep for the device evaluator")
        return start


@dataclass
class GeneralTables:
    """Host arrays of pn_general_desc (include/pnrte_b200.h)."""
    dim: int
    U: int
    lm: list
    par: np.ndarray
    e_ptr: np.ndarray
    e_tgt: np.ndarray
    e_dx: np.ndarray
    e_dy: np.ndarray
    e_dz: np.ndarray
    e_diag: np.ndarray
    e_code: np.ndarray
    r_code: np.ndarray
    ops: np.ndarray
    consts: np.ndarray
    s_slot: np.ndarray
    s_dx: np.ndarray
    s_dy: np.ndarray
    s_dz: np.ndarray
    field_names: list


def compile_general(program, h):
    """Flatten a stencil program into GeneralTables for grid spacing h
    (solver.py:127-181: masks need the row location and target home parity;
    coefficients become postfix programs)."""
    dim = program.dim
    if dim not in (2, 3):
        raise UnsupportedProgramError("programs must be 2-D or 3-D")
    U = len(program.rows)
    pad = lambda t: tuple(t) + (0,) * (AXES - len(t))  # noqa: E731
    place = {k: pad(v) for k, v in program.placement.offsets.items()}
    em = _Emitter(float(h), dim)
    rows = sorted(program.rows, key=lambda r: program.unknown_index[r.index])
    if [program.unknown_index[r.index] for r in rows] != list(range(U)):
        raise UnsupportedProgramError("component indices are not 0..U-1")
    par = np.zeros(U, np.int32)
    e_ptr = [0]
    cols = {k: [] for k in ("tgt", "dx", "dy", "dz", "diag", "code")}
    r_code = np.full(U, -1, np.int32)
    for c, row in enumerate(rows):
        loc = pad(row.location)
        par[c] = sum(1 << k for k in range(AXES) if loc[k] == 1)
        for e in row.entries:
            home = place[e.target]
            off = pad(e.offset)
            disp = tuple((off[k] - home[k]) // 2 for k in range(AXES))
            tc = program.unknown_index[e.target]
            cols["tgt"].append(tc)
            cols["dx"].append(disp[0]); cols["dy"].append(disp[1]); cols["dz"].append(disp[2])
            cols["diag"].append(int(tc == c and disp == (0, 0, 0)))
            cols["code"].append(em.code(e.coeff))
        e_ptr.append(len(cols["tgt"]))
        r_code[c] = em.code(row.residual)
    home_par = np.zeros(U, np.int32)
    for lm, c in program.unknown_index.items():
        home_par[c] = sum(1 << k for k in range(AXES) if place[lm][k] == 1)
    if not np.array_equal(home_par, par):
        raise UnsupportedProgramError("row locations differ from the placement of their unknowns")
    samples = sorted(em.samples.items(), key=lambda kv: kv[1])
    i32 = lambda v: np.ascontiguousarray(v, np.int32)  # noqa: E731
    names = sorted(em.fields, key=em.fields.get)
    return GeneralTables(
        dim=dim, U=U, lm=[r.index for r in rows], par=par, e_ptr=i32(e_ptr), e_tgt=i32(cols["tgt"]),
        e_dx=i32(cols["dx"]), e_dy=i32(cols["dy"]), e_dz=i32(cols["dz"]), e_diag=i32(cols["diag"]),
        e_code=i32(cols["code"]), r_code=r_code, ops=i32(em.ops),
        consts=np.ascontiguousarray(em.consts if em.consts else [0.0], np.float64),
        s_slot=i32([k[0] for k, _ in samples] or [0]), s_dx=i32([k[1] for k, _ in samples] or [0]),
        s_dy=i32([k[2] for k, _ in samples] or [0]), s_dz=i32([k[3] for k, _ in samples] or [0]),
        field_names=names)


def is_general(program):
    """True when a program needs this path (not the constant-weight P_N form)."""
    from .program import PnTables, tables_from_program
    if isinstance(program, (int, PnTables)):
        return False
    try:
        tables_from_program(program)
    except UnsupportedProgramError:
        return True
    return False
