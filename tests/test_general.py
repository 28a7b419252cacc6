"""General stencil programs (CDA, equations.py:213-237) on the host side:
the restated program equals the reference's compiled one, the numpy oracle
(oracle/general_oracle.py) reproduces the reference's assembly bit for bit,
and the postfix programs the device evaluates (general.py) give the
oracle's coefficients when interpreted here with numpy."""

import numpy as np
import pytest

from cases import CDA_CASES, cda_inputs, probe_vector
from oracle import general_oracle as go
from oracle.oracle import CsrOracle
from paper_1807_00410_b200 import general as G
from paper_1807_00410_b200.program import UnsupportedProgramError, build_tables

FIX_BLAS = (8, 0)


def _tree(n):
    k = type(n).__name__
    if k == "Num":
        return ("N", float(n.value))
    if k == "Sym":
        return ("S", n.name)
    if k == "FieldSample":
        return ("F", n.name, tuple(n.pos))
    if k in ("Add", "Mul"):
        return (k,) + tuple(_tree(c) for c in n.children)
    if k == "Pow":
        return ("Pow", _tree(n.base), n.exponent)
    return (k,)


def _run(gt, pc, spec, res3):
    """numpy interpreter of one postfix program over the whole grid."""
    grids = np.indices(res3)
    st = []
    while True:
        op, a = gt.ops[2 * pc], gt.ops[2 * pc + 1]
        pc += 1
        if op == G.OP_END:
            return st[0]
        if op == G.OP_NUM:
            st.append(np.full(res3, gt.consts[a]))
        elif op == G.OP_FIELD:
            arr = go.field_array(spec, gt.field_names[gt.s_slot[a]]).reshape(res3)
            idx = tuple(np.clip(grids[k] + (gt.s_dx, gt.s_dy, gt.s_dz)[k][a], 0, res3[k] - 1) for k in range(3))
            st.append(arr[idx])
        elif op in (G.OP_ADD, G.OP_MUL):
            b = st.pop()
            st[-1] = st[-1] + b if op == G.OP_ADD else st[-1] * b
        elif op == G.OP_RECIP:
            st[-1] = 1.0 / st[-1]
        elif op == G.OP_SQUARE:
            st[-1] = st[-1] * st[-1]
        elif op == G.OP_SQRT:
            st[-1] = np.sqrt(st[-1])
        elif op == G.OP_ONE:
            st[-1] = np.ones(res3)
        else:
            raise AssertionError(op)


@pytest.mark.parametrize("case", CDA_CASES)
def test_oracle_matches_golden(case, golden):
    prog, spec = cda_inputs(case)
    g = golden["cda"]
    A, Q = go.assemble(prog, spec)
    assert np.array_equal(A.indptr, g[f"{case}/indptr"]) and np.array_equal(A.indices, g[f"{case}/indices"])
    assert A.data.tobytes() == g[f"{case}/data"].tobytes() and Q.tobytes() == g[f"{case}/Q"].tobytes()
    x = probe_vector(A.shape[0])
    assert (A @ x).tobytes() == g[f"{case}/Ax"].tobytes()
    xs, rep = CsrOracle(A).cgnr(Q, tol=1e-10, max_iter=500, blas_threads=FIX_BLAS[0], blas_kernel=FIX_BLAS[1])
    assert xs.tobytes() == g[f"{case}/cg0/x"].tobytes()
    assert rep["iterations"] == golden["cda_meta"]["cases"][case]["cg0"]["iterations"]
    assert go.unstagger(xs, prog, spec.res).tobytes() == g[f"{case}/unstagger"].tobytes()


@pytest.mark.parametrize("case", CDA_CASES)
def test_postfix_programs_equal_oracle(case):
    """Interpreting the compiled programs gives the oracle's diagonal,
    couplings and RHS bit for bit (Dirichlet masks applied afterwards)."""
    prog, spec = cda_inputs(case)
    gt = G.compile_general(prog, spec.h)
    res3 = tuple(spec.res) + (1,) * (3 - len(spec.res))
    row = prog.rows[0]

    def sampler(name, pos):
        pad = 2
        arr = np.pad(go.field_array(spec, name), pad, mode="edge")
        return arr[tuple(slice(pad + p // 2, pad + p // 2 + spec.res[k]) for k, p in enumerate(pos))]

    for e, pc in zip(row.entries, gt.e_code):
        want = np.broadcast_to(np.asarray(go.evaluate(e.coeff, spec.h, sampler), float), spec.res)
        got = _run(gt, int(pc), spec, res3).reshape(spec.res)
        assert got.tobytes() == np.ascontiguousarray(want).tobytes()
    want = np.broadcast_to(np.asarray(-go.evaluate(row.residual, spec.h, sampler), float), spec.res)
    got = -_run(gt, int(gt.r_code[0]), spec, res3).reshape(spec.res)
    assert got.tobytes() == np.ascontiguousarray(want).tobytes()


def test_compile_shapes_and_detection():
    p3 = G.build_cda_program(3)
    gt = G.compile_general(p3, 0.25)
    assert gt.U == 1 and list(gt.e_ptr) == [0, 7] and gt.e_diag.tolist() == [0, 0, 0, 1, 0, 0, 0]
    assert gt.field_names == ["sigma_t", "sigma_s", "p_0", "Q_0_0"]
    assert G.is_general(p3) and not G.is_general(3) and not G.is_general(build_tables(2))
    assert (gt.e_dx.tolist(), gt.e_dy.tolist(), gt.e_dz.tolist()) == (
        [-1, 0, 0, 0, 0, 0, 1], [0, -1, 0, 0, 0, 1, 0], [0, 0, -1, 0, 1, 0, 0])


def test_unsupported_exponent_rejected():
    bad = G.Pow(G.FieldSample("sigma_t", (0, 0, 0)), 3)
    em = G._Emitter(0.1, 3)
    with pytest.raises(UnsupportedProgramError):
        em.code(bad)
    em = G._Emitter(0.1, 3)
    em.code(G.Pow(G.Sym("h"), 3))           # field-free: folded on the host
    assert em.consts == [0.1 ** 3]


@pytest.mark.reference
@pytest.mark.parametrize("dim", [2, 3])
def test_restated_cda_program_equals_reference(dim, ref):
    from pnrte.equations import build_cda
    from pnrte.stencil import compile_program
    rp, mp = compile_program(build_cda(dim)), G.build_cda_program(dim)
    ra, ma = rp.rows[0], mp.rows[0]
    assert [tuple(e.offset) for e in ra.entries] == [tuple(e.offset) for e in ma.entries]
    assert [_tree(e.coeff) for e in ra.entries] == [_tree(e.coeff) for e in ma.entries]
    assert _tree(ra.residual) == _tree(ma.residual)
    assert dict(rp.placement.offsets) == dict(mp.placement.offsets) and rp.unknown_index == mp.unknown_index
    assert G.is_general(rp)


@pytest.mark.reference
def test_oracle_matches_live_reference(ref):
    from dataclasses import replace
    from pnrte.equations import build_cda
    from pnrte.solver import assemble
    from pnrte.stencil import compile_program
    from cases import rand_spec
    for bc in ("dirichlet", "neumann"):
        spec = replace(rand_spec(1, (5, 7, 3), 61), bc=bc)
        s = assemble(compile_program(build_cda(3)), spec)
        A, Q = go.assemble(G.build_cda_program(3), spec)
        assert A.data.tobytes() == s.A.data.tobytes() and np.array_equal(A.indices, s.A.indices)
        assert Q.tobytes() == s.Q.tobytes()
