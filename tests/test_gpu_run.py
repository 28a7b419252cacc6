"""Device-integrated run (cli.run semantics) end to end on the GPU."""

import numpy as np
import pytest

from paper_1807_00410_b200 import fields as fio
from paper_1807_00410_b200.run import main

pytestmark = pytest.mark.gpu


def test_run_pointsource_artifacts(tmp_path):
    out = tmp_path / "out"
    rc = main(["run", "--problem", "pointsource", "--res", "16", "--order", "3", "--tol", "1e-8",
               "--out", str(out)])
    assert rc == 0
    meta, coll = fio.read_field(out / "field.pnfld")
    assert meta["res"] == (16, 16, 16) and meta["unknowns"] == 16 and np.isfinite(coll).all()
    r, v = fio.read_profile(out / "profile.csv")
    assert len(r) == 8 and v[0] > v[-1] > 0       # fluence decays away from the source
    log = (out / "solve.log").read_text()
    assert "converged True" in log


def test_run_matches_solve_pn_faithful(tmp_path):
    from paper_1807_00410_b200.run import build_problem, config_from_mapping
    from paper_1807_00410_b200.solver import solve_pn
    out = tmp_path / "o"
    assert main(["run", "--problem", "cfg1", "--tol", "1e-6", "--mode", "faithful", "--out", str(out)]) == 0
    _, coll = fio.read_field(out / "field.pnfld")
    spec = build_problem(config_from_mapping({"problem": "cfg1"}))
    want, rep = solve_pn(1, spec, tol=1e-6, mode="faithful")
    assert rep.iterations == 169 and coll.tobytes() == want.tobytes()


def test_run_nonconvergence_exit_code(tmp_path):
    assert main(["run", "--problem", "cfg2", "--max-iter", "3", "--tol", "1e-12", "--out", str(tmp_path)]) == 3
