"""The C-ABI library loads and exports every symbol include/sten.h declares; the
product package does not reach into the oracle (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "sten.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_]+\s*\*?\s*([a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("stencil_create", "stencil_apply", "bicgstab_solve", "stencil_destroy", "sten_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2010_03660_b200 as sten
    from paper_2010_03660_b200 import build
    build.build()
    L = ctypes.CDLL(sten.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    assert sten.version() == 3


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2010_03660_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", text, flags=re.M), f
                assert "liboracle" not in text, f
                assert "oracle.h" not in text, f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    import paper_2010_03660_b200 as sten
    monkeypatch.setattr(sten, "_lib", None)
    monkeypatch.setattr(sten, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(sten.StenError):
        sten.lib()
