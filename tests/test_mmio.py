"""Matrix Market reader / writer against the reference's
own behaviour (tests/golden/mmio.json, made by make_mmio_golden.py): the same
triples bit for bit, the same error class, message and line, the same written
text byte for byte. The reader is the native parser of libb200sp (host code,
no GPU needed)."""

import io
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

LIB = os.path.join(os.path.dirname(GOLDEN), "..", "paper_2006_16852_b200", "libb200sp.so")
pytestmark = pytest.mark.skipif(not os.path.exists(LIB), reason="libb200sp.so not built")

with open(os.path.join(GOLDEN, "mmio.json")) as f:
    G = json.load(f)


@pytest.mark.parametrize("name", sorted(G["read"]))
def test_read_matches_reference(name):
    from paper_2006_16852_b200 import mmio

    case = G["read"][name]
    exp = case["expect"]
    for threads in (1, 3):
        if "error" in exp:
            with pytest.raises(Exception) as ei:
                mmio.read_matrix_market_bytes(case["input"].encode(), threads=threads)
            assert type(ei.value).__name__ == exp["error"]
            assert str(ei.value) == exp["message"]
            assert getattr(ei.value, "line", None) == exp["line"]
        else:
            d = mmio.read_matrix_market_bytes(case["input"].encode(), threads=threads)
            assert [d.size.rows, d.size.cols] == exp["size"]
            assert d.rows.tolist() == exp["rows"] and d.cols.tolist() == exp["cols"]
            assert [repr(float(v)) for v in d.vals] == exp["vals"]


def test_stream_api_and_write_byte_identical(tmp_path):
    from paper_2006_16852_b200 import MatrixData, mmio

    w = G["write"]["random_dups"]
    data = MatrixData(tuple(w["size"]), w["rows"], w["cols"], w["vals"])
    s = io.StringIO()
    mmio.write_matrix_market(s, data)
    assert s.getvalue() == w["text"]
    # read(write(x)) then write again: byte-identical (canonical file)
    d2 = mmio.read_matrix_market(io.StringIO(w["text"]))
    s2 = io.StringIO()
    mmio.write_matrix_market(s2, d2)
    assert s2.getvalue() == w["text"]
    p = tmp_path / "m.mtx"
    p.write_text(w["text"])
    d3 = mmio.read_matrix_market_file(str(p))
    np.testing.assert_array_equal(d3.vals, d2.vals)
    a = G["write"]["array_2x3"]
    s3 = io.StringIO()
    mmio.write_matrix_market_array(s3, np.array(a["dense"]))
    assert s3.getvalue() == a["text"]


def test_large_parallel_parse_matches_single_thread():
    from paper_2006_16852_b200 import mmio

    rng = np.random.default_rng(0)
    n, k = 5000, 200_000
    r = rng.integers(1, n + 1, k)
    c = rng.integers(1, n + 1, k)
    v = rng.standard_normal(k)
    text = "%%MatrixMarket matrix coordinate real symmetric\n% big\n" + f"{n} {n} {k}\n" + "".join(
        f"{a} {b} {x!r}\n" for a, b, x in zip(r.tolist(), c.tolist(), v.tolist()))
    d1 = mmio.read_matrix_market_bytes(text, threads=1)
    d8 = mmio.read_matrix_market_bytes(text, threads=8)
    off = r != c
    assert d1.nnz == k + int(off.sum())
    for a, b in ((d1.rows, d8.rows), (d1.cols, d8.cols), (d1.vals, d8.vals)):
        np.testing.assert_array_equal(a, b)
    # mirrors follow their entry (src/mmio.py:98-101)
    np.testing.assert_array_equal(d1.vals[:2], [v[0]] * (2 if off[0] else 1) + ([v[1]] if not off[0] else []))
