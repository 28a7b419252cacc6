"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute call: this runs without a GPU)."""

import ctypes
import pathlib
import re

from paper_1807_00410_b200 import _lib

ROOT = pathlib.Path(__file__).resolve().parents[1]


def declared():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = h.read_text()
        names.update(re.findall(r"^\s*(?:int|int64_t|const char \*|void)\s*\*?\s*(pn_\w+)\s*\(", text, re.M))
    return names


def test_header_declares_entry_points():
    d = declared()
    assert {"pn_create", "pn_destroy", "pn_set_field", "pn_setup", "pn_apply", "pn_solve",
            "pn_unstagger", "pn_last_error"} <= d


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    for name in sorted(declared()):
        assert hasattr(L, name), name
        assert isinstance(getattr(L, name), ctypes._CFuncPtr)


def test_library_is_sm100a():
    data = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in data
