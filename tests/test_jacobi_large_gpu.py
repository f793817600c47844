"""Block-Jacobi with blocks over 32 rows (reference src/precond.py:28-208:
any block_size or explicit block_boundaries) against the reference's own
outputs (tests/golden/jacobi_large.npz, made by
`tests/golden/make_golden.py jacobi_large`): inverses, condition numbers and
the adaptive-precision decision bit-exact, the apply within rounding, and
preconditioned solves within +-1 iteration."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden
from oracle import problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    return load_golden("jacobi_large.npz")


def _matrix(b2, exc, g):
    n = int(g["n"])
    return b2.matrix_from_data(exc, b2.MatrixData((n, n), g["rows"], g["cols"], g["vals"]), "csr")


KW = {
    "bs64": {"block_size": 64},
    "bs100": {"block_size": 100},
    "bounds": {"block_boundaries": [0, 5, 37, 40, 240, 300, 301, 420]},
    "bs64_adapt": {"block_size": 64, "adaptive_precision": True, "condition_threshold": 1e2},
}


@pytest.mark.parametrize("name", list(KW))
def test_large_blocks_bitwise_and_apply(cuda, gold, name):
    import paper_2006_16852_b200 as b2

    g = gold[f"convdiff_g8_{name}"]
    a = _matrix(b2, cuda, g)
    jac = b2.Jacobi(cuda, **KW[name]).generate(a)
    assert not jac.fusable
    nb = g["starts"].size
    assert jac.num_blocks == nb
    assert np.array_equal(np.array(jac.block_conditions), g["cond"])
    assert np.array_equal(np.array([p == "reduced" for p in jac.block_precisions]), g["reduced"])
    flat = np.concatenate([jac.stored_inverse(i).astype(np.float64).reshape(-1) for i in range(nb)])
    assert np.array_equal(flat, g["inv_flat"])
    z = b2.Dense.zeros(cuda, int(g["n"]), 2)
    jac.apply(b2.Dense(cuda, g["r"]), z)
    # z = inv @ r: same inverse, summation order of the mat-vec differs
    np.testing.assert_allclose(np.asarray(z.data), g["z"], rtol=1e-12, atol=1e-13)


def test_pivoting_block_over_128_rows(cuda, gold):
    """150-row block: NumPy's recursive pairwise row sums in kappa and heavy
    partial pivoting (non-dominant random matrix)."""
    import paper_2006_16852_b200 as b2

    g = gold["rand200_b150"]
    a = _matrix(b2, cuda, g)
    jac = b2.Jacobi(cuda, block_boundaries=[0, 150]).generate(a)
    flat = np.concatenate([jac.stored_inverse(i).reshape(-1) for i in range(2)])
    assert np.array_equal(flat, g["inv_flat"])
    assert np.array_equal(np.array(jac.block_conditions), g["cond"])


def test_gauss_jordan_inverse_large(cuda, gold):
    import paper_2006_16852_b200 as b2

    g = gold["rand200_b150"]
    dense = np.zeros((200, 200))
    dense[g["rows"], g["cols"]] = g["vals"]
    inv = b2.gauss_jordan_inverse(dense[:150, :150], cuda)
    assert np.array_equal(inv.reshape(-1), g["inv_flat"][:150 * 150])


@pytest.mark.parametrize("name,kind,solver,bs,kw", [
    ("bicgstab_bj64_cd_g12", "convdiff", "bicgstab", 64, {}),
    ("gmres30_bj144_cd_g12", "convdiff", "gmres", 144, {"krylov_dim": 30}),
    ("cg_bj64_7pt_g12", "7pt", "cg", 64, {}),
])
def test_large_block_preconditioned_solves(cuda, gold, name, kind, solver, bs, kw):
    import paper_2006_16852_b200 as b2

    ref = gold[name]
    n, r, c, v = P.stencil3d(12, kind)
    a = b2.matrix_from_data(cuda, b2.MatrixData((n, n), r, c, v), "csr")
    fac = b2.SOLVER_FACTORIES[solver](cuda, criteria=[b2.Iteration(10000), b2.ResidualNormReduction(1e-8)],
                                      preconditioner=b2.Jacobi(cuda, block_size=bs), **kw)
    s = fac.generate(a)
    x = b2.Dense.zeros(cuda, n, 1)
    s.apply(b2.Dense(cuda, np.ones((n, 1))), x)
    st = s.last_status
    assert st.converged and st.stopping_id == int(ref["stopping_id"])
    assert abs(st.iterations - int(ref["iterations"])) <= 1, (st.iterations, int(ref["iterations"]))
    xr = ref["x"][:, 0]
    assert np.linalg.norm(np.asarray(x.data)[:, 0] - xr) <= 1e-6 * np.linalg.norm(xr)


def test_block_over_limit_raises(cuda):
    import paper_2006_16852_b200 as b2

    n = 5000
    d = b2.MatrixData((n, n), np.arange(n), np.arange(n), np.ones(n))
    a = b2.matrix_from_data(cuda, d, "csr")
    with pytest.raises(b2.Unsupported):
        b2.Jacobi(cuda, block_size=4097).generate(a)
