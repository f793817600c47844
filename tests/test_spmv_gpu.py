"""SpMV / conversion / generator parity on the B200 (through the C ABI).

Oracle: the reference's own outputs (tests/golden, bitwise-pinned oracle) and
oracle/*.py. Tolerances (north_star): SpMV normwise-inf relative error
<= 1e-14 in fp64 and <= 1e-6 in fp32; conversions and generators bit-exact.
"""

import numpy as np
import pytest

from conftest import random_sparse
from oracle import convert as OC
from oracle import problems as P
from oracle import spmv as OS

pytestmark = pytest.mark.gpu

TOL = {"float64": 1e-14, "float32": 1e-6}

FORMATS = [
    ("csr", {"strategy": "classical"}),
    ("csr", {"strategy": "load_balance"}),
    ("csr", {"strategy": "load_balance", "impl": "lb2"}),
    ("csr", {"strategy": "load_balance", "impl": "lb3"}),
    ("csr", {"strategy": "stream"}),
    ("csr", {"strategy": "stream", "impl": "tma"}),
    ("csr", {"strategy": "stream", "impl": "tma", "rpt": 4, "cap": 64, "stages": 3}),
    ("csr", {"strategy": "stream", "impl": "ld"}),
    ("csr", {"strategy": "stream", "impl": "tma", "tpr": 4, "rpt": 2, "cap": 200, "stages": 3, "nt": 512}),
    ("csr", {"strategy": "stream", "impl": "tma", "tpr": 2, "rpt": 1, "nt": 512}),
    ("coo", {}),
    ("ell", {}),
    ("sellp", {}),
    ("sellp", {"slice_size": 4, "stride_factor": 2}),
    ("hybrid", {}),
    ("hybrid", {"strategy": "imbalance"}),
    ("hybrid", {"strategy": "col1"}),
]
IDS = ["csr_classical", "csr_lb", "csr_lb_rows", "csr_lb_nnz", "csr_stream", "csr_pipe", "csr_pipe_small", "csr_stream_ld", "csr_pipe_tpr4", "csr_pipe_tpr2", "coo", "ell", "sellp64", "sellp4", "hybrid_auto", "hybrid_imb",
       "hybrid_col1"]


def make(b2, exc, data, fmt, kw, dtype="float64"):
    kw = dict(kw)
    impl = kw.pop("impl", None)
    if impl in ("lb2", "lb3"):
        a = b2.matrix_from_data(exc, data, fmt, value_dtype=dtype, **kw)
        a.set_strategy("load_balance", lb_mode=int(impl[-1]))
        return a
    if impl is not None:
        rpt, cap, stages = kw.pop("rpt", None), kw.pop("cap", None), kw.pop("stages", None)
        nt, tpr = kw.pop("nt", None), kw.pop("tpr", 1)
        a = b2.matrix_from_data(exc, data, fmt, value_dtype=dtype, **kw)
        a.set_strategy(kw["strategy"], stream_impl=impl, stream_shape=(tpr, rpt or 1) if (rpt or tpr > 1) else None,
                       stream_cap=cap, stream_stages=stages, stream_consumers=nt)
        return a
    if fmt == "hybrid":
        s = kw.pop("strategy", None)
        kw["strategy"] = {None: None, "imbalance": b2.imbalance_limit(0.8),
                          "col1": b2.column_limit(1)}[s]
    return b2.matrix_from_data(exc, data, fmt, value_dtype=dtype, **kw)


def golden_data(b2, g):
    n = int(g["n"])
    return b2.MatrixData((n, n), g["rows"], g["cols"], g["vals"])


@pytest.mark.parametrize("fmt,kw", FORMATS, ids=IDS)
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_spmv_matches_reference(cuda, golden_spmv, fmt, kw, dtype):
    import paper_2006_16852_b200 as b2

    for name, g in golden_spmv.items():
        a = make(b2, cuda, golden_data(b2, g), fmt, kw, dtype)
        b = b2.Dense(cuda, g["b"], value_dtype=dtype)
        x = b2.Dense(cuda, np.full(g["b"].shape, 7.0), value_dtype=dtype)  # must be overwritten
        a.apply(b, x)
        if dtype == "float64":
            ref = g["x_csr"]
        else:
            n = int(g["n"])
            rp = OS.csr_from_triples(n, g["rows"], g["cols"], g["vals"])
            ref = OS.csr_spmv(rp, g["cols"], g["vals"].astype(np.float32).astype(np.float64),
                              g["b"].astype(np.float32).astype(np.float64))
        err = OS.rel_error_inf(np.asarray(x.data), ref)
        assert err <= TOL[dtype], (name, err)


def test_known_answer_exact(cuda, golden_spmv):
    import paper_2006_16852_b200 as b2

    g = golden_spmv["tri3"]
    for fmt, kw in FORMATS + [("dense", {})]:
        a = make(b2, cuda, golden_data(b2, g), fmt, kw)
        x = b2.Dense.zeros(cuda, 3, 1)
        a.apply(b2.Dense.vector(cuda, [1.0, 2.0, 3.0]), x)
        np.testing.assert_array_equal(x.data[:, 0], [0.0, 0.0, 4.0])


@pytest.mark.parametrize("fmt,kw", FORMATS, ids=IDS)
def test_advanced_apply_matches_reference(cuda, golden_spmv, fmt, kw):
    import paper_2006_16852_b200 as b2

    for name, g in golden_spmv.items():
        if "xadv_csr" not in g:
            continue
        alpha, beta = g["adv"]
        a = make(b2, cuda, golden_data(b2, g), fmt, kw)
        x = b2.Dense(cuda, g["x0"])
        a.apply_advanced(b2.Dense(cuda, [[alpha]]), b2.Dense(cuda, g["b"]), b2.Dense(cuda, [[beta]]), x)
        assert OS.rel_error_inf(np.asarray(x.data), g["xadv_csr"]) <= 1e-14, name
        x2 = b2.Dense(cuda, g["x0"])
        a.apply_advanced(alpha, b2.Dense(cuda, g["b"]), beta, x2)  # host scalars
        assert OS.rel_error_inf(np.asarray(x2.data), g["xadv_csr"]) <= 1e-14, name


@pytest.mark.parametrize("fmt,kw", FORMATS, ids=IDS)
def test_fused_residual(cuda, golden_spmv, fmt, kw):
    import paper_2006_16852_b200 as b2

    g = golden_spmv["st27_g8"]
    n = int(g["n"])
    a = make(b2, cuda, golden_data(b2, g), fmt, kw)
    xv = np.random.default_rng(3).standard_normal((n, 1))
    bv = np.random.default_rng(4).standard_normal((n, 1))
    r = b2.Dense.zeros(cuda, n, 1)
    a.residual(b2.Dense(cuda, xv), b2.Dense(cuda, bv), r)
    ref = OS.residual(g["rows"], g["cols"], g["vals"], xv, bv)
    assert OS.rel_error_inf(np.asarray(r.data), ref) <= 1e-14


@pytest.mark.parametrize("fmt,kw", FORMATS + [("dense", {})], ids=IDS + ["dense"])
def test_empty_and_one_by_one(cuda, fmt, kw):
    import paper_2006_16852_b200 as b2

    a = make(b2, cuda, b2.MatrixData((4, 4)), fmt, kw)
    x = b2.Dense(cuda, np.full((4, 1), 7.0))
    a.apply(b2.Dense.vector(cuda, np.ones(4)), x)
    np.testing.assert_array_equal(x.data, np.zeros((4, 1)))
    a = make(b2, cuda, b2.MatrixData((1, 1), [0], [0], [2.5]), fmt, kw)
    x = b2.Dense.zeros(cuda, 1, 1)
    a.apply(b2.Dense.vector(cuda, [3.0]), x)
    assert x.data[0, 0] == 7.5


@pytest.mark.parametrize("fmt,kw", FORMATS, ids=IDS)
def test_long_rows_straddling_tiles_and_chunks(cuda, fmt, kw):
    """One 60k-entry row first, one in the middle, one last, plus empty rows:
    exercises the merge-path carry fix-up and the Coo chunk carries."""
    import paper_2006_16852_b200 as b2

    n = 70000
    rng = np.random.default_rng(9)
    rows, cols = [], []
    for r in (0, 35000, n - 1):
        c = np.sort(rng.choice(n, 60000, replace=False))
        rows.append(np.full(c.size, r))
        cols.append(c)
    short = np.arange(1, n - 1, 3)
    rows.append(short)
    cols.append((short * 7) % n)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    vals = rng.uniform(-1, 1, rows.size)
    data = b2.MatrixData((n, n), rows, cols, vals).canonicalize()
    a = make(b2, cuda, data, fmt, kw)
    bv = rng.standard_normal((n, 1))
    x = b2.Dense(cuda, np.full((n, 1), 3.0))
    a.apply(b2.Dense(cuda, bv), x)
    rp = OS.csr_from_triples(n, data.rows, data.cols, data.vals)
    ref = OS.csr_spmv(rp, data.cols, data.vals, bv)
    assert OS.rel_error_inf(np.asarray(x.data), ref) <= 1e-14


def test_multi_rhs_columns_match_single(cuda):
    import paper_2006_16852_b200 as b2

    data = random_sparse(200, 0.05, seed=3)
    bv = np.random.default_rng(1).standard_normal((200, 3))
    for fmt, kw in FORMATS:
        a = make(b2, cuda, data, fmt, kw)
        x = b2.Dense.zeros(cuda, 200, 3)
        a.apply(b2.Dense(cuda, bv), x)
        for j in range(3):
            xj = b2.Dense.zeros(cuda, 200, 1)
            a.apply(b2.Dense(cuda, bv[:, j:j + 1]), xj)
            assert np.array_equal(np.asarray(x.data)[:, j], np.asarray(xj.data)[:, 0])


def test_repeatable_bitwise(cuda):
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import problems

    a = problems.power_law(cuda, 100000, seed=5, max_len=2000)
    b = b2.Dense(cuda, np.random.default_rng(0).standard_normal((100000, 1)))
    for fmt in ("csr_classical", "csr_lb", "csr_stream", "csr_pipe", "coo", "ell", "sellp", "hybrid"):
        m = b2.convert(a, fmt)
        x1, x2 = b2.Dense.zeros(cuda, 100000, 1), b2.Dense.zeros(cuda, 100000, 1)
        m.apply(b, x1)
        m.apply(b, x2)
        assert np.array_equal(np.asarray(x1.data), np.asarray(x2.data)), fmt


# ---------------------------------------------------------------------------
# conversions: bit-exact against the oracle layouts
# ---------------------------------------------------------------------------
def test_conversions_bit_exact(cuda, golden_spmv):
    import paper_2006_16852_b200 as b2

    for name, g in golden_spmv.items():
        n = int(g["n"])
        data = golden_data(b2, g)
        csr = b2.matrix_from_data(cuda, data, "csr")
        rp = OS.csr_from_triples(n, g["rows"], g["cols"], g["vals"])
        assert np.array_equal(np.asarray(csr.row_ptrs), rp), name
        ell = b2.convert(csr, "ell")
        eci, ev, w, st = OC.csr_to_ell(rp, g["cols"], g["vals"])
        assert (ell.width, ell.stride) == (w, st)
        assert np.array_equal(np.asarray(ell.col_idxs), eci) and np.array_equal(np.asarray(ell.vals), ev)
        for S, sf in ((64, 1), (4, 2)):
            sp = b2.convert(csr, "sellp", slice_size=S, stride_factor=sf)
            sl, ss, sci, sv = OC.csr_to_sellp(rp, g["cols"], g["vals"], S, sf)
            assert np.array_equal(np.asarray(sp.slice_lengths), sl)
            assert np.array_equal(np.asarray(sp.slice_sets), ss)
            assert np.array_equal(np.asarray(sp.col_idxs), sci) and np.array_equal(np.asarray(sp.vals), sv)
        for strat, wref in ((b2.imbalance_limit(0.8), OC.hybrid_width_imbalance(rp, 0.8)),
                            (b2.minimal_storage_limit(), OC.hybrid_width_minimal_storage(rp, 8))):
            hy = b2.convert(csr, "hybrid", strategy=strat)
            (eci, ev, w, st), (cr, cc, cv) = OC.csr_to_hybrid(rp, g["cols"], g["vals"], wref)
            assert hy.ell.width == wref, name
            assert np.array_equal(np.asarray(hy.ell.col_idxs), eci)
            assert np.array_equal(np.asarray(hy.coo.row_idxs), cr)
            assert np.array_equal(np.asarray(hy.coo.col_idxs), cc)
            assert np.array_equal(np.asarray(hy.coo.vals), cv)
        coo = b2.convert(csr, "coo")
        assert np.array_equal(np.asarray(coo.row_idxs), g["rows"])
        # every format converts back to the identical Csr
        for fmt in ("coo", "ell", "sellp", "hybrid", "dense"):
            back = b2.convert(b2.convert(csr, fmt), "csr")
            assert np.array_equal(np.asarray(back.row_ptrs), rp), (name, fmt)
            assert np.array_equal(np.asarray(back.col_idxs), g["cols"]), (name, fmt)
            assert np.array_equal(np.asarray(back.vals), g["vals"]), (name, fmt)


def test_to_data_preserves_triples(cuda):
    import paper_2006_16852_b200 as b2

    data = random_sparse(12, density=0.3, seed=5).canonicalize()
    for fmt in ("csr", "coo", "ell", "sellp", "hybrid", "dense"):
        out = b2.matrix_from_data(cuda, data, fmt).to_data().canonicalize()
        assert np.array_equal(out.rows, data.rows) and np.array_equal(out.cols, data.cols)
        assert np.array_equal(out.vals, data.vals)


# ---------------------------------------------------------------------------
# device generators: bit-exact against oracle/problems.py
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("kind,g", [("5pt", 31), ("7pt", 9), ("27pt", 7), ("convdiff", 6)])
def test_stencil_generator_bit_exact(cuda, kind, g):
    from paper_2006_16852_b200 import problems

    a = problems.stencil(cuda, kind, g)
    n, r, c, v = P.five_point(g) if kind == "5pt" else P.stencil3d(g, kind)
    rp, ci, vals = P.to_csr(n, r, c, v)
    assert np.array_equal(np.asarray(a.row_ptrs), rp)
    assert np.array_equal(np.asarray(a.col_idxs), ci)
    assert np.array_equal(np.asarray(a.vals), vals)


def test_power_law_generator_bit_exact(cuda):
    from paper_2006_16852_b200 import problems

    a = problems.power_law(cuda, 3000, seed=3, max_len=700)
    n, r, c, v = P.power_law(3000, seed=3, max_len=700)
    rp, ci, vals = P.to_csr(n, r, c, v)
    assert np.array_equal(np.asarray(a.row_ptrs), rp)
    assert np.array_equal(np.asarray(a.col_idxs), ci)
    assert np.array_equal(np.asarray(a.vals), vals)


def test_c2_full_size_properties(cuda):
    """C2 (27-point 128^3): every format reproduces the exact row sums
    (A * ones, small integers -> exact in fp64) and agrees with the oracle
    on a random vector at g=64."""
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import problems

    a = problems.stencil(cuda, "27pt", 128)
    n = a.size.rows
    assert a.nnz == 55_742_968
    ones = b2.Dense(cuda, np.ones((n, 1)))
    idx = np.arange(n)
    g = 128
    cnt = [(1 + (t > 0) + (t < g - 1)) for t in (idx // (g * g), (idx // g) % g, idx % g)]
    expect = 27.0 - cnt[0] * cnt[1] * cnt[2]  # 26 - (len - 1)
    for fmt in ("csr_classical", "csr_lb", "csr_stream", "csr_pipe", "coo", "ell", "sellp", "hybrid"):
        m = b2.convert(a, fmt)
        x = b2.Dense.zeros(cuda, n, 1)
        m.apply(ones, x)
        assert np.array_equal(np.asarray(x.data)[:, 0], expect), fmt
    a = problems.stencil(cuda, "27pt", 64)
    n, r, c, v = P.stencil3d(64, "27pt")
    rp, ci, vals = P.to_csr(n, r, c, v)
    bv = np.random.default_rng(0).standard_normal((n, 1))
    ref = OS.csr_spmv(rp, ci, vals, bv)
    for fmt in ("csr_classical", "csr_lb", "csr_stream", "csr_pipe", "coo", "ell", "sellp", "hybrid"):
        x = b2.Dense.zeros(cuda, n, 1)
        b2.convert(a, fmt).apply(b2.Dense(cuda, bv), x)
        assert OS.rel_error_inf(np.asarray(x.data), ref) <= 1e-14, fmt


def test_host_operands_migrate(cuda, host, golden_spmv):
    """apply with host b/x: H2D of b, kernel, D2H of x (the end-to-end path)."""
    import paper_2006_16852_b200 as b2

    g = golden_spmv["poisson31"]
    a = b2.matrix_from_data(cuda, golden_data(b2, g), "csr")
    b = b2.Dense(host, g["b"])
    x = b2.Dense(host, np.zeros_like(g["b"]))
    a.apply(b, x)
    assert OS.rel_error_inf(x.data, g["x_csr"]) <= 1e-14


def test_dense_blas(cuda):
    import paper_2006_16852_b200 as b2

    rng = np.random.default_rng(11)
    xv, yv = rng.standard_normal((50, 2)), rng.standard_normal((50, 2))
    x, y = b2.Dense(cuda, xv), b2.Dense(cuda, yv)
    np.testing.assert_array_equal(x.dot(y), y.dot(x))
    np.testing.assert_allclose(x.dot(y), (xv * yv).sum(axis=0), rtol=1e-14)
    np.testing.assert_allclose(x.norm2(), np.sqrt((xv * xv).sum(axis=0)), rtol=1e-14)
    y.add_scaled(0.7, x)
    y.add_scaled(-0.7, x)
    # bitwise the reference's NumPy `y += a * x` (product rounded, then added)
    ref = yv + 0.7 * xv
    ref = ref + (-0.7) * xv
    np.testing.assert_array_equal(np.asarray(y.data), ref)
    y.scale(b2.Dense(cuda, [[2.0, -1.0]]))
    np.testing.assert_array_equal(np.asarray(y.data), ref * [2.0, -1.0])


@pytest.mark.parametrize("knob,val", [("coo_minb", 6)])
def test_coo_kernel_variants(cuda, golden_spmv, knob, val):
    """Every Coo kernel variant (b200sp_set_tuning) reproduces the reference,
    including rows spanning many chunks and empty rows."""
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import _lib

    default = {"coo_minb": 1}[knob]
    _lib.set_tuning(knob, val)
    try:
        for name, g in golden_spmv.items():
            for dtype in ("float64", "float32"):
                a = make(b2, cuda, golden_data(b2, g), "coo", {}, dtype)
                x = b2.Dense(cuda, np.full(g["b"].shape, 7.0), value_dtype=dtype)
                a.apply(b2.Dense(cuda, g["b"], value_dtype=dtype), x)
                ref = g["x_csr"]
                if dtype == "float32":
                    n = int(g["n"])
                    rp = OS.csr_from_triples(n, g["rows"], g["cols"], g["vals"])
                    ref = OS.csr_spmv(rp, g["cols"], g["vals"].astype(np.float32).astype(np.float64),
                                      g["b"].astype(np.float32).astype(np.float64))
                assert OS.rel_error_inf(np.asarray(x.data), ref) <= TOL[dtype], (name, dtype)
        test_long_rows_straddling_tiles_and_chunks(cuda, "coo", {})
        test_fused_residual(cuda, golden_spmv, "coo", {})
        test_advanced_apply_matches_reference(cuda, golden_spmv, "coo", {})
    finally:
        _lib.set_tuning(knob, default)


@pytest.mark.parametrize("kind", ["27pt", "random", "odd"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_pipelined_host_apply_bitwise(cuda, host, kind, dtype):
    """Host operands on a large Csr take the streaming path (the chunked
    copy-engine pipeline); results are bitwise those of the device-resident
    apply."""
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import problems

    if kind == "27pt":
        a = problems.stencil(cuda, "27pt", 64, value_dtype=dtype)
    else:
        # "odd": a row count that is no multiple of the tile or the 16-byte store width
        n, rng = (70000 if kind == "random" else 65537 + 1024 * 3 + 1), np.random.default_rng(4)
        rows = np.repeat(np.arange(n), 8)
        cols = rng.integers(0, n, rows.size) if kind == "random" else (rows + rng.integers(-300, 300, rows.size)) % n
        data = b2.MatrixData((n, n), rows, cols, rng.standard_normal(rows.size))
        a = b2.matrix_from_data(cuda, data, "csr", value_dtype=dtype)
    a = b2.convert(a, "csr_classical")  # (fp32 long rows default to the stream strategy)
    n = a.size.rows
    assert a._pipeline_ok(b2.Dense(host, np.zeros((n, 1)), value_dtype=dtype),
                          b2.Dense(host, np.zeros((n, 1)), value_dtype=dtype))
    bv = np.random.default_rng(1).standard_normal((n, 1))
    xh = b2.Dense(host, np.full((n, 1), 3.0), value_dtype=dtype)
    a.apply(b2.Dense(host, bv, value_dtype=dtype), xh)
    xd = b2.Dense.zeros(cuda, n, 1, value_dtype=dtype)
    a.apply(b2.Dense(cuda, bv, value_dtype=dtype), xd)
    np.testing.assert_array_equal(np.asarray(xh.data), np.asarray(xd.data))
    for f in (2.0, 0.5, 4.0):  # plan, flags (epochs) and buffers reused; exact scalings
        a.apply(b2.Dense(host, f * bv, value_dtype=dtype), xh)
        np.testing.assert_array_equal(np.asarray(xh.data), f * np.asarray(xd.data))


def test_pipeline_refuses_pageable_memory(cuda, host):
    """The pipelined host apply issues asynchronous copies: it is taken only
    when both host operands are really page-locked (a Dense.wrap of a plain
    NumPy array on a pinned host executor is not); otherwise the plain
    migrate-apply-copy path runs -- same result."""
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import problems

    a = problems.stencil(cuda, "27pt", 64)
    n = a.size.rows
    bv = np.random.default_rng(2).standard_normal((n, 1))
    pageable = b2.Dense.wrap(host, bv.copy())
    xh = b2.Dense(host, np.zeros((n, 1)))
    assert not a._pipeline_ok(pageable, xh)
    a.apply(pageable, xh)
    xd = b2.Dense.zeros(cuda, n, 1)
    a.apply(b2.Dense(cuda, bv), xd)
    np.testing.assert_array_equal(np.asarray(xh.data), np.asarray(xd.data))


def test_clone_gets_its_own_pipeline_plan(cuda, host):
    """clone_to must not share the source's host-pipeline plan (device
    staging buffers, streams, CUDA graphs captured against the source's
    arrays): applying the clone after the source is freed stays correct."""
    import gc

    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import problems

    a = problems.stencil(cuda, "27pt", 48)
    n = a.size.rows
    bv = np.random.default_rng(3).standard_normal((n, 1))
    bh, xh = b2.Dense(host, bv), b2.Dense(host, np.zeros((n, 1)))
    a.apply(bh, xh)  # builds and caches the source's plan + graph
    ref = np.asarray(xh.data).copy()
    c = a.clone_to(cuda)
    assert getattr(c, "_pplan", None) is None
    del a
    gc.collect()
    xh2 = b2.Dense(host, np.zeros((n, 1)))
    c.apply(bh, xh2)
    np.testing.assert_array_equal(np.asarray(xh2.data), ref)


# ---------------------------------------------------------------------------
# row-loop variants of the classical kernel (predicated entry blocks, aligned
# pair loads) and Ell's predicated tail: every mode on odd / even entry counts
# and several row-length mixes, against the oracle; pair loads only with the
# even-count flag (no read past the arrays' end)
# ---------------------------------------------------------------------------
def _ragged(n, seed, max_len):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_len + 1, n)
    rows = np.repeat(np.arange(n), lens)
    cols = np.concatenate([np.sort(rng.choice(n, size=l, replace=False)) for l in lens]) if lens.sum() else np.zeros(0, int)
    vals = rng.standard_normal(rows.size)
    return rows, cols, vals


@pytest.mark.parametrize("kb", [0, 2, 3, 4, -1, -2, -4])
@pytest.mark.parametrize("sw", [1, 2, 4, 8])
@pytest.mark.parametrize("case", ["even", "odd", "ragged"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_classical_row_loop_variants(cuda, kb, sw, case, dtype):
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import _lib

    n = 777
    if case == "ragged":
        rows, cols, vals = _ragged(n, 5, 40)
    else:
        rows, cols, vals = _ragged(n, 6, 9)
        want_odd = case == "odd"
        if (rows.size % 2 == 1) != want_odd:  # drop the last entry to flip the parity
            rows, cols, vals = rows[:-1], cols[:-1], vals[:-1]
    data = b2.MatrixData((n, n), rows, cols, vals)
    rp, ci, v = P.to_csr(n, rows, cols, vals)
    bv = np.random.default_rng(1).standard_normal((n, 1))
    ref = OS.csr_spmv(rp, ci, v, bv)
    _lib.set_tuning("classical_kb", kb)
    try:
        a = b2.matrix_from_data(cuda, data, "csr", value_dtype=dtype, strategy="classical")
        a.set_strategy("classical", subwarp=sw)
        x = b2.Dense.zeros(cuda, n, 1, value_dtype=dtype)
        a.apply(b2.Dense(cuda, bv, value_dtype=dtype), x)
        assert OS.rel_error_inf(np.asarray(x.data, dtype=np.float64), ref) <= TOL[dtype]
        # alpha / beta path through the same kernel
        x0 = b2.Dense(cuda, np.ones((n, 1)), value_dtype=dtype)
        a.apply_advanced(0.5, b2.Dense(cuda, bv, value_dtype=dtype), -1.0, x0)
        assert OS.rel_error_inf(np.asarray(x0.data, dtype=np.float64), 0.5 * ref - 1.0) <= 4 * TOL[dtype]
    finally:
        _lib.reset_tuning("classical_kb")


@pytest.mark.parametrize("width_max", [1, 3, 4, 5, 8, 9, 27])
@pytest.mark.parametrize("fmt", ["ell", "sellp", "hybrid"])
def test_ell_predicated_tail_widths(cuda, width_max, fmt):
    import paper_2006_16852_b200 as b2

    n = 513
    rows, cols, vals = _ragged(n, width_max, width_max)
    data = b2.MatrixData((n, n), rows, cols, vals)
    rp, ci, v = P.to_csr(n, rows, cols, vals)
    bv = np.random.default_rng(2).standard_normal((n, 1))
    a = b2.matrix_from_data(cuda, data, fmt)
    x = b2.Dense.zeros(cuda, n, 1)
    a.apply(b2.Dense(cuda, bv), x)
    assert OS.rel_error_inf(np.asarray(x.data), OS.csr_spmv(rp, ci, v, bv)) <= 1e-14


@pytest.mark.parametrize("kind,g", [("7pt", 14), ("27pt", 9)])
def test_fused_solver_spmv_modes_bitwise(cuda, kind, g):
    """The fused SpMV + dot kernel's row-loop modes (loop, 4-entry blocks,
    aligned pairs) keep the loop's entry order: a CG solve gives bitwise the
    same iterate and iteration count in every mode."""
    import torch

    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import _lib, problems

    a = problems.stencil(cuda, kind, g)
    n = a.size.rows
    xs = {}
    try:
        for mode in (0, 1, 2):
            _lib.set_tuning("spmv_dot_mode", mode)
            _lib.set_tuning("coop_resident", 0)
            from paper_2006_16852_b200 import config

            old = config.CG_COOP_MAX_ROWS
            config.CG_COOP_MAX_ROWS = 0  # the batched (fused-SpMV) path
            try:
                s = b2.Cg(cuda, criteria=[b2.Iteration(500), b2.ResidualNormReduction(1e-10)]).generate(a)
                x = b2.Dense.wrap(cuda, torch.zeros((n, 1), dtype=torch.float64, device=cuda.device))
                s.apply(b2.Dense.wrap(cuda, torch.ones((n, 1), dtype=torch.float64, device=cuda.device)), x)
            finally:
                config.CG_COOP_MAX_ROWS = old
            xs[mode] = (s.last_status.iterations, x.values.cpu().numpy().copy())
    finally:
        _lib.reset_tuning("spmv_dot_mode")
        _lib.reset_tuning("coop_resident")
    assert xs[0][0] == xs[1][0] == xs[2][0]
    assert np.array_equal(xs[0][1], xs[1][1]) and np.array_equal(xs[0][1], xs[2][1])
