"""CPU: the C-ABI library loads and exports every symbol the header declares
(no compute calls without a GPU)."""

import os
import re

from paper_1602_05033_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "krymat_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kry_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    assert set(header_functions()) == set(_lib.SIGNATURES)


def test_version_and_error_string():
    lib = _lib.load()
    assert lib.kry_version() >= 1
    assert isinstance(_lib.last_error(), str)


def test_operator_desc_layout_matches_header():
    # kind, variable (2x int32), then int64 n at offset 8
    assert _lib.OperatorDesc.n.offset == 8
    assert _lib.OperatorDesc.c_diag.offset == 40
    assert _lib.OperatorDesc.z_end.offset == _lib.OperatorDesc.z_begin.offset + 8
