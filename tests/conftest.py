import os
import pathlib
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

REF_SRC = pathlib.Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "reference: needs the live reference under /root/reference")


def pytest_collection_modifyitems(config, items):
    have_ref = REF_SRC.exists()
    for item in items:
        if "reference" in item.keywords and not have_ref:
            item.add_marker(pytest.mark.skip(reason="reference not mounted (GPU box)"))


@pytest.fixture(scope="session")
def ref():
    """The live reference package (only in the build container)."""
    if not REF_SRC.exists():
        pytest.skip("reference not mounted")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import pnrte
    return pnrte


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    g = ROOT / "tests" / "golden"
    return {
        "cases": np.load(g / "cases.npz"),
        "cases_meta": json.loads((g / "cases.json").read_text()),
        "configs": json.loads((g / "configs.json").read_text()),
        "neumann": np.load(g / "neumann.npz"),
        "neumann_meta": json.loads((g / "neumann.json").read_text()),
        "cda": np.load(g / "cda.npz"),
        "cda_meta": json.loads((g / "cda.json").read_text()),
        "dir": g,
    }
