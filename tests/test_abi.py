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


def _param_code(decl, suf):
    """ctypes type code of one C parameter declaration (as _lib spells them)."""
    d = " ".join(decl.replace("const", " ").split())
    if "*" in d or d.startswith("void"):
        return "p"
    base = d.split()[0]
    vt = {"f64": "double", "f32": "float"}.get(suf)
    if base in ("int64_t", "long"):
        return "l"
    if base in ("int32_t", "int", "uint32_t"):
        return "i"
    if base == "uint64_t":
        return "u"
    if base == "T" or (vt and base == vt and suf == "f32"):
        return "V"
    if base == "double":
        return "d" if suf != "f64" else "V"
    if base == "float":
        return "V"
    return "?"


def _prototype_codes():
    """{symbol: [type codes]} for every prototype spelled out in the header."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"//[^\n]*", "", text)
    text = text.replace("B200SP_JAC_DECL", "int64_t a, const int32_t *b, const int64_t *c, const uint8_t *d, "
                                           "const void *e")
    out = {}
    for m in re.finditer(r"\b(b200sp_[a-z0-9_#A-Z]+)\s*\(([^)]*)\)\s*;", text):
        name, params = m.group(1), m.group(2).strip()
        parts = [] if params in ("", "void") else [q.strip() for q in params.split(",")]
        for suf in (("f64", "f32") if "##SUF" in name else (name.rsplit("_", 1)[-1],)):
            key = name.replace("##SUF", suf)
            out[key] = [_param_code(q, suf) for q in parts]
    return out


def _prototype_arg_counts():
    """{symbol: number of parameters} for every prototype spelled out in the
    header (macro-generated ones are expanded for f64 / f32)."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"//[^\n]*", "", text)
    text = text.replace("B200SP_JAC_DECL", "a, b, c, d, e")  # the 5 block-Jacobi parameters
    out = {}
    for m in re.finditer(r"\b(b200sp_[a-z0-9_#A-Z]+)\s*\(([^)]*)\)\s*;", text):
        name, params = m.group(1), m.group(2).strip()
        n = 0 if params in ("", "void") else params.count(",") + 1
        if "##SUF" in name:
            for suf in ("f64", "f32"):
                out[name.replace("##SUF", suf)] = n
        else:
            out[name] = n
    return out


@pytest.mark.skipif(not os.path.exists(LIB), reason="libb200sp.so not built")
def test_binding_signatures_match_header_arity():
    """Every ctypes signature in _lib has as many parameters as the header's
    prototype (a mismatch would only surface as a TypeError on the GPU)."""
    from paper_2006_16852_b200 import _lib

    _lib._load()
    protos = _prototype_arg_counts()
    bad = []
    for key, fn in _lib._funcs.items():
        sym = "b200sp_" + key
        if sym in protos and len(fn.argtypes) != protos[sym]:
            bad.append((sym, len(fn.argtypes), protos[sym]))
    assert not bad, bad
    assert len([k for k in _lib._funcs if "b200sp_" + k in protos]) > 50


@pytest.mark.skipif(not os.path.exists(LIB), reason="libb200sp.so not built")
def test_binding_signatures_match_header_types():
    """Beyond the arity: every parameter's kind (int64 / int32 / pointer /
    double / value type) matches -- a pointer bound as an int (or the reverse)
    would be truncated by ctypes and fault only on the GPU box."""
    import ctypes

    from paper_2006_16852_b200 import _lib

    _lib._load()
    protos = _prototype_codes()
    rev = {ctypes.c_int64: "l", ctypes.c_int32: "i", ctypes.c_uint64: "u", ctypes.c_void_p: "p",
           ctypes.c_char_p: "p"}
    bad = []
    for key, fn in _lib._funcs.items():
        sym = "b200sp_" + key
        if sym not in protos:
            continue
        suf = key.rsplit("_", 1)[-1]
        got = []
        for t in fn.argtypes:
            if t is ctypes.c_double:
                got.append("V" if suf == "f64" else "d")
            elif t is ctypes.c_float:
                got.append("V")
            else:
                got.append(rev.get(t, "?"))
        want = protos[sym]
        if len(got) == len(want) and any(g != w for g, w in zip(got, want) if w != "?"):
            bad.append((sym, "".join(got), "".join(want)))
    assert not bad, bad
