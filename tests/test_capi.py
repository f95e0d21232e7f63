"""CPU-side checks of the C ABI library: it loads and exports every entry
point declared in include/wbflow_b200.h (no device calls)."""
import ctypes
import os
import re

from paper_1806_04960_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "wbflow_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(wb_\w+)\(", src, re.M)))


def test_library_exports_header():
    lib = _lib.load()
    names = declared()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_bindings_cover_header():
    names = set(declared()) - {"wb_last_error"}
    assert names <= set(_lib.SIGNATURES), names - set(_lib.SIGNATURES)


def test_config_struct_layout():
    # the ctypes mirror must match the C struct (checked via offsets)
    c = _lib.WbConfig
    assert c.inflow_seg.offset == 4 * 4 + 8 * 8 + 16
    assert ctypes.sizeof(_lib.WbError) == 32
