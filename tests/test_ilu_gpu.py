"""ParILU(0) + sparse triangular solves + ILU-preconditioned Krylov solves
 against the reference's own runs (tests/golden/ilu.npz,
`python tests/golden/make_golden.py ilu`).

Factors: identical patterns (bit-exact row pointers / columns), values within
1e-13 relative per entry (the reference's per-entry sums are NumPy dot
products, the device sums them sequentially); triangular solves within
1e-12; preconditioned solves: iteration counts within +-1.
"""

import numpy as np
import pytest

from conftest import load_golden, random_sparse
from oracle import problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden_ilu():
    return load_golden("ilu.npz")


def mats():
    d = random_sparse(40, density=0.15, seed=7).canonicalize()
    return {"cd5": P.stencil3d(5, "convdiff"), "p2d8": P.five_point(8), "rand40": (40, d.rows, d.cols, d.vals)}


def csr(b2, exc, n, r, c, v):
    return b2.matrix_from_data(exc, b2.MatrixData((n, n), r, c, v), "csr")


@pytest.mark.parametrize("name", ["cd5", "p2d8", "rand40"])
def test_parilu_factors_match_reference(cuda, golden_ilu, name):
    import paper_2006_16852_b200 as b2

    n, r, c, v = mats()[name]
    a = csr(b2, cuda, n, r, c, v)
    for sw in (0, 1, 3, 2 * n):
        g = golden_ilu[f"parilu_{name}_s{sw}"]
        f = b2.ParIlu(cuda, sweeps=sw).generate(a)
        for fac, key in ((f.l, "l"), (f.u, "u")):
            np.testing.assert_array_equal(np.asarray(fac.row_ptrs), g[f"{key}_rp"])
            np.testing.assert_array_equal(np.asarray(fac.col_idxs), g[f"{key}_ci"])
            got, ref = np.asarray(fac.vals), g[f"{key}_v"]
            assert np.all(np.abs(got - ref) <= 1e-13 * np.maximum(np.abs(ref), 1.0)), (sw, key)
        assert abs(f.defect_on_pattern(a) - float(g["defect"])) <= 1e-10 * max(1.0, float(g["defect"]))


@pytest.mark.parametrize("name", ["cd5", "p2d8", "rand40"])
def test_triangular_solves_and_ilu_apply(cuda, golden_ilu, name):
    import paper_2006_16852_b200 as b2

    n, r, c, v = mats()[name]
    a = csr(b2, cuda, n, r, c, v)
    g = golden_ilu[f"trs_{name}"]
    f = b2.ParIlu(cuda, sweeps=2 * n).generate(a)
    b = b2.Dense(cuda, g["b"])
    for solver, key in ((b2.LowerTrs(cuda, unit_diagonal=True).generate(f.l), "xl"),
                        (b2.UpperTrs(cuda).generate(f.u), "xu"),
                        (b2.Ilu(cuda, sweeps=2 * n).generate(a), "xilu")):
        x = b2.Dense.zeros(cuda, n, 2)
        solver.apply(b, x)
        ref = g[key]
        assert np.linalg.norm(np.asarray(x.data) - ref) <= 1e-12 * np.linalg.norm(ref), key
        x2 = b2.Dense.zeros(cuda, n, 2)
        solver.apply(b, x2)  # repeatable (epoch flags)
        np.testing.assert_array_equal(np.asarray(x2.data), np.asarray(x.data))


def test_triangular_generate_errors(cuda):
    import paper_2006_16852_b200 as b2

    a = b2.matrix_from_data(cuda, b2.MatrixData((2, 2), [0, 1, 1], [0, 0, 1], [1.0, 2.0, 0.0]), "csr")
    with pytest.raises(b2.Singular):
        b2.LowerTrs(cuda).generate(a)
    b2.LowerTrs(cuda, unit_diagonal=True).generate(a)  # unit diagonal ignores the stored 0
    with pytest.raises(b2.Singular):
        b2.ParIlu(cuda).generate(a)
    with pytest.raises(b2.DimensionMismatch):
        b2.UpperTrs(cuda).generate(b2.matrix_from_data(cuda, b2.MatrixData((2, 3)), "csr"))


def test_large_lower_solve_sync_free(cuda):
    """A 7-point 64^3 lower triangle (262k rows, dependency chains of
    length ~190): sync-free substitution against scipy."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl

    import paper_2006_16852_b200 as b2

    n, r, c, v = P.stencil3d(64, "7pt")
    keep = c <= r
    a = b2.matrix_from_data(cuda, b2.MatrixData((n, n), r[keep], c[keep], v[keep]), "csr")
    bv = np.random.default_rng(2).standard_normal(n)
    x = b2.Dense.zeros(cuda, n, 1)
    b2.LowerTrs(cuda).generate(a).apply(b2.Dense(cuda, bv.reshape(n, 1)), x)
    m = sp.csr_matrix((v[keep], (r[keep], c[keep])), shape=(n, n))
    ref = spl.spsolve_triangular(m, bv, lower=True)
    assert np.linalg.norm(np.asarray(x.data)[:, 0] - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("name,kind,solver", [("cg_ilu_7pt_g8", "7pt", "cg"),
                                              ("bicgstab_ilu_cd_g8", "convdiff", "bicgstab"),
                                              ("gmres_ilu_cd_g8", "convdiff", "gmres")])
def test_ilu_preconditioned_solves_match_reference(cuda, golden_ilu, name, kind, solver):
    import paper_2006_16852_b200 as b2

    g = golden_ilu[name]
    n, r, c, v = P.stencil3d(8, kind)
    a = csr(b2, cuda, n, r, c, v)
    s = b2.SOLVER_FACTORIES[solver](cuda, criteria=[b2.Iteration(1000), b2.ResidualNormReduction(1e-10)],
                                    preconditioner=b2.Ilu(cuda)).generate(a)
    x = b2.Dense.zeros(cuda, n, 1)
    s.apply(b2.Dense(cuda, np.ones((n, 1))), x)
    st = s.last_status
    assert st.converged and abs(st.iterations - int(g["iterations"])) <= 1, (st.iterations, int(g["iterations"]))
    assert np.linalg.norm(np.asarray(x.data) - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])
