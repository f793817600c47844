"""Performance-profile harness: coverage curves pinned to
the reference's definition (src/bench.py:186-200) on hand-computed tables;
the GPU run over a directory of Matrix Market files and the automatic format
choice on a B200."""

import numpy as np
import pytest


def test_profile_curves_reference_semantics():
    from paper_2006_16852_b200.profile import profile_csv, profile_curves

    runtimes = {"csr": [1.0, 2.0, 4.0], "ell": [2.0, 2.0, 1.0], "coo": [4.0, 1.0, 8.0]}
    c = profile_curves(runtimes, [1.0, 2.0, 4.0])
    # best per matrix = (1, 1, 1); ties at tau = 1 credit every tied format
    assert c["csr"] == [(1.0, 1 / 3), (2.0, 2 / 3), (4.0, 1.0)]
    assert c["ell"] == [(1.0, 1 / 3), (2.0, 1.0), (4.0, 1.0)]
    assert c["coo"] == [(1.0, 1 / 3), (2.0, 1 / 3), (4.0, 2 / 3)]
    csv = profile_csv({"curves": c})
    assert csv.splitlines()[0] == "format,tau,fraction"
    assert "coo,1,0.333333" in csv and csv.endswith("\n")


@pytest.mark.gpu
def test_run_profile_and_choose_format(cuda, tmp_path):
    import paper_2006_16852_b200 as b2
    from oracle import problems as P
    from paper_2006_16852_b200 import mmio
    from paper_2006_16852_b200.profile import GPU_FORMATS, choose_format, run_profile

    for name, (n, r, c, v) in {"st7": P.stencil3d(12, "7pt"), "p2d": P.five_point(20)}.items():
        with open(tmp_path / f"{name}.mtx", "w") as f:
            mmio.write_matrix_market(f, b2.MatrixData((n, n), r, c, v))
    (tmp_path / "broken.mtx").write_text("%%MatrixMarket matrix coordinate complex general\n1 1 0\n")
    res = run_profile(str(tmp_path), reps=3)
    assert res["matrices"] == ["p2d.mtx", "st7.mtx"]
    assert [s["matrix"] for s in res["skipped"]] == ["broken.mtx"]
    assert set(res["runtimes_ns"]) == set(GPU_FORMATS)
    for f, curve in res["curves"].items():
        assert curve[-1][1] == 1.0 or max(t for t in res["runtimes_ns"][f]) > 0
    best_at_1 = sum(curve[0][1] for curve in res["curves"].values())
    assert best_at_1 >= 1.0  # every matrix has a best format
    n, r, c, v = P.stencil3d(16, "27pt")
    a = b2.matrix_from_data(cuda, b2.MatrixData((n, n), r, c, v), "csr")
    fmt, m, times = choose_format(a)
    assert fmt == min(times, key=times.get)
    x = b2.Dense.zeros(cuda, n, 1)
    bv = np.random.default_rng(0).standard_normal((n, 1))
    m.apply(b2.Dense(cuda, bv), x)
    rp, ci, vals = P.to_csr(n, r, c, v)
    from oracle import spmv as OS

    assert OS.rel_error_inf(np.asarray(x.data), OS.csr_spmv(rp, ci, vals, bv)) <= 1e-14
    assert choose_format(a)[0] == fmt  # cached
