"""PNFLD1 / profile / config formats and the run front door (CPU parts)."""

import numpy as np
import pytest

from paper_1807_00410_b200 import fields as fio
from paper_1807_00410_b200.run import ConfigError, RunConfig, config_from_mapping, main, make_pointsource


def test_field_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    coll = rng.normal(size=(3, 4, 5, 9))
    fio.write_field(tmp_path / "f.pnfld", coll, 2)
    meta, back = fio.read_field(tmp_path / "f.pnfld")
    assert meta == {"dim": 3, "res": (3, 4, 5), "order": 2, "unknowns": 9}
    assert back.tobytes() == coll.tobytes()


def test_reads_reference_writer_layout(tmp_path):
    """The reference writer ends the header with one newline (fields.py:31-38);
    such files are read correctly (the reference's own reader cannot, :53)."""
    coll = np.arange(2 * 3 * 2 * 4, dtype=float).reshape(2, 3, 2, 4) / 7.0
    header = "\n".join(["PNFLD1", "dim 3", "res 2 3 2", "order 1", "unknowns 4", "endian little", ""])
    flat = np.ascontiguousarray(coll.reshape(12, 4, order="F"), dtype="<f8")
    (tmp_path / "ref.pnfld").write_bytes(header.encode("ascii") + flat.tobytes())
    meta, back = fio.read_field(tmp_path / "ref.pnfld")
    assert meta["res"] == (2, 3, 2) and back.tobytes() == coll.tobytes()


@pytest.mark.reference
def test_reads_files_of_the_live_reference_writer(tmp_path, ref):
    from pnrte.fields import write_field
    coll = np.random.default_rng(1).normal(size=(4, 3, 2, 4))
    write_field(tmp_path / "x.pnfld", coll, 1)
    assert fio.read_field(tmp_path / "x.pnfld")[1].tobytes() == coll.tobytes()


@pytest.mark.reference
def test_pointsource_matches_reference_generator(ref):
    from pnrte.problems import make_pointsource as ref_ps
    a, b = make_pointsource(16), ref_ps(16)
    assert a.res == b.res and a.extent == b.extent and a.origin == b.origin
    for k in b.fields:
        assert np.asarray(a.fields[k]).tobytes() == np.asarray(b.fields[k]).tobytes(), k


def test_profile_and_config_files(tmp_path):
    fio.write_profile(tmp_path / "p.csv", [(0.0, 1.5), (0.25, 0.75)])
    r, v = fio.read_profile(tmp_path / "p.csv")
    assert r.tolist() == [0.0, 0.25] and v.tolist() == [1.5, 0.75]
    (tmp_path / "c.txt").write_text("# run\nproblem=cfg2\norder=3\njacobi=true\n")
    cfg = config_from_mapping(fio.read_config(tmp_path / "c.txt"))
    assert cfg.problem == "cfg2" and cfg.order == 3 and cfg.jacobi is True


@pytest.mark.parametrize("mapping", [{"problem": "checkerboard"}, {"method": "sn"}, {"order": 0},
                                     {"tol": 0}, {"bogus": 1}, {"jacobi": "maybe"}, {"mode": "turbo"},
                                     {"bc": "periodic"}])
def test_config_errors(mapping):
    with pytest.raises((ConfigError, ValueError)):
        config_from_mapping(mapping)


def test_main_config_error_exit_code(tmp_path):
    assert main(["run", "--problem", "checkerboard", "--out", str(tmp_path)]) == 2
    assert main(["run", "--order", "0", "--out", str(tmp_path)]) == 2
    assert main(["bogus"]) == 2
