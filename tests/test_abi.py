"""C-ABI library loads and exports every symbol include/b200sp.h declares
(CPU only: no kernel is launched)."""

import ctypes
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "b200sp.h")
LIB = os.path.join(REPO, "paper_2006_16852_b200", "libb200sp.so")


def declared_symbols():
    text = open(HEADER).read()
    names = set(re.findall(r"\b(b200sp_[a-z0-9_]+)\s*\(", text))
    # expand the typed declaration macros (T, SUF)
    for macro in re.finditer(r"#define B200SP_[A-Z]+_DECL\(T, SUF\)(.*?)\n(?!.*\\\n)", text, re.S):
        for base in re.findall(r"b200sp_([a-z0-9_]+)_##SUF", macro.group(1)):
            names.update({f"b200sp_{base}_f64", f"b200sp_{base}_f32"})
    for base in re.findall(r"b200sp_([a-z0-9_]+)_##SUF", text):
        names.update({f"b200sp_{base}_f64", f"b200sp_{base}_f32"})
    return sorted(n for n in names if "##" not in n)


def test_header_declares_a_full_api():
    names = declared_symbols()
    for must in ("b200sp_csr_spmv_classical_f64", "b200sp_csr_spmv_lb_f64", "b200sp_coo_spmv_f64",
                 "b200sp_ell_spmv_f64", "b200sp_sellp_spmv_f64", "b200sp_csr_to_ell_f64"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="libb200sp.so not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB), reason="libb200sp.so not built")
def test_binding_table_matches_header():
    from paper_2006_16852_b200 import _lib

    declared = set(declared_symbols())
    bound = set(_lib.exported_symbols())
    assert bound <= declared, sorted(bound - declared)
    _lib._load()
    assert _lib.query("version") == 1


def test_missing_library_fails_loudly(monkeypatch):
    from paper_2006_16852_b200 import _lib
    from paper_2006_16852_b200.errors import KernelNotImplemented

    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libb200sp.so")
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(KernelNotImplemented):
        _lib._load()
