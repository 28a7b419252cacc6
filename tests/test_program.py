"""Stencil tables: restated builder == reference StencilProgram, pinned by
committed fixtures (tests/golden/tables_N*.json from tools/make_goldens.py)."""

import json

import pytest

from paper_1807_00410_b200.program import (InvalidOrderError, build_tables, canonical_diag, field_slots,
                                           pack_tables, tables_from_program, to_json, transport_couplings)


@pytest.mark.parametrize("N", range(1, 8))
def test_tables_match_golden(N, golden):
    want = json.loads((golden["dir"] / f"tables_N{N}.json").read_text())
    assert to_json(build_tables(N)) == want


@pytest.mark.reference
@pytest.mark.parametrize("N", range(1, 8))
def test_tables_match_live_reference(N, ref):
    from pnrte.equations import build_pn
    from pnrte.stencil import compile_program
    assert tables_from_program(compile_program(build_pn(N, 3))) == build_tables(N)


@pytest.mark.reference
@pytest.mark.parametrize("N", [1, 3, 6])
def test_transport_couplings_match_reference(N, ref):
    from pnrte.equations import transport_couplings as ref_tc
    for l in range(N + 1):
        for m in range(-l, l + 1):
            assert transport_couplings(l, m) == ref_tc(l, m)


def test_p1_is_mac_layout():
    """test_stencil.py:21-26: (1,1) on x faces, (1,-1) y, (1,0) z."""
    t = build_tables(1)
    loc = {r.lm: r.location for r in t.rows}
    assert loc[(0, 0)] == (0, 0, 0) and loc[(1, 1)] == (1, 0, 0)
    assert loc[(1, -1)] == (0, 1, 0) and loc[(1, 0)] == (0, 0, 1)


@pytest.mark.parametrize("N", [1, 3, 5, 7])
def test_half_offset_and_reach(N):
    """Every off-diagonal entry reaches at most one voxel along one axis
    (test_stencil.py:35-50,202-205) and the diagonal is canonical."""
    t = build_tables(N)
    for r in t.rows:
        for e in r.entries:
            if not e.diag:
                assert sum(abs(d) for d in e.disp) <= 1
    assert canonical_diag(t)


def test_entry_counts():
    """Appendix A of SURVEY.md: entries per row mean/max for N=1,3,5,7."""
    want = {1: (4.0, 7), 3: (9.75, 15), 5: (12.89, 21), 7: (14.69, 21)}
    for N, (mean, mx) in want.items():
        t = build_tables(N)
        n = [len(r.entries) for r in t.rows]
        assert round(sum(n) / len(n), 2) == mean and max(n) == mx


def test_invalid_order():
    with pytest.raises(InvalidOrderError):
        build_tables(0)


def test_pack_orders_columns_ascending():
    """Packed A rows are in scipy column order: z-1, y-1, x-1, same (comp
    ascending), x+1, y+1, z+1."""
    rank = {5: 0, 3: 1, 1: 2, 0: 3, 2: 4, 4: 5, 6: 6}
    pk = pack_tables(build_tables(5), 0.1)
    for prefix, oth in (("a", "a_tgt"), ("t", "t_src")):
        ptr = pk[f"{prefix}_ptr"]
        for c in range(pk["U"]):
            keys = [(rank[int(pk[f"{prefix}_dir"][e])], int(pk[oth][e])) for e in range(ptr[c], ptr[c + 1])]
            assert keys == sorted(keys)
    assert len(field_slots(5)) == pk["n_fields"] == 2 + 6 + 36


@pytest.mark.parametrize("N", [1, 2, 3])
def test_2d_tables_roundtrip_golden(N, golden):
    from paper_1807_00410_b200.program import from_json
    want = json.loads((golden["dir"] / f"tables_N{N}_2d.json").read_text())
    t = from_json(want)
    assert t.dim == 2 and to_json(t) == want
    pk = pack_tables(t, 0.1)
    assert set(pk["par"].tolist()) <= {0, 1, 2, 3}     # no z staggering in 2-D


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_2d_builder_matches_reference_fixtures(N, golden):
    """build_tables(N, 2) restates compile_program(build_pn(N, 2))
    (equations.py:51-103,179-210): equal to the reference's tables."""
    from paper_1807_00410_b200.program import build_tables
    t = build_tables(N, dim=2)
    assert t.dim == 2
    assert to_json(t) == json.loads((golden["dir"] / f"tables_N{N}_2d.json").read_text())


@pytest.mark.reference
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6])
def test_2d_builder_matches_live_reference(N, ref):
    from pnrte.equations import build_pn
    from pnrte.stencil import compile_program
    from paper_1807_00410_b200.program import build_tables
    assert to_json(build_tables(N, dim=2)) == to_json(tables_from_program(compile_program(build_pn(N, 2))))


@pytest.mark.reference
@pytest.mark.parametrize("N", [1, 2, 3])
def test_2d_tables_match_live_reference(N, ref, golden):
    from pnrte.equations import build_pn
    from pnrte.stencil import compile_program
    t = tables_from_program(compile_program(build_pn(N, 2)))
    assert to_json(t) == json.loads((golden["dir"] / f"tables_N{N}_2d.json").read_text())
