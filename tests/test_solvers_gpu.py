"""Solver + block-Jacobi parity on the B200 against the reference's own runs
(tests/golden/solvers.npz, jacobi.npz made by tests/golden/make_golden.py).

Contract (north_star): identical iteration counts within +-1 at the same
residual-reduction criterion; final residuals agree with the reference to the
stated tolerance. Block-Jacobi inverses and condition numbers bit-exact.
"""

import numpy as np
import pytest

from conftest import random_sparse, random_spd
from oracle import problems as P

pytestmark = pytest.mark.gpu


def system(b2, exc, n, r, c, v, fmt="csr"):
    return b2.matrix_from_data(exc, b2.MatrixData((n, n), r, c, v), fmt)


def solve(b2, exc, a, bvec, solver, precond=0, iters=10000, factor=1e-8, **kw):
    n = a.size.rows
    b = b2.Dense(exc, bvec.reshape(n, -1))
    x = b2.Dense.zeros(exc, n, b.size.cols)
    pre = b2.Jacobi(exc, block_size=precond) if precond else None
    fac = b2.SOLVER_FACTORIES[solver](exc, criteria=[b2.Iteration(iters), b2.ResidualNormReduction(factor)],
                                      preconditioner=pre, **kw)
    s = fac.generate(a)
    s.apply(b, x)
    return s.last_status, np.asarray(x.data)


def true_rel_residual(a_host, x, b):
    return np.linalg.norm(b - a_host @ x) / np.linalg.norm(b)


def csr_host(n, r, c, v):
    import scipy.sparse as sp

    return sp.csr_matrix((v, (r, c)), shape=(n, n))


CASES = [
    ("cg_c1", "5pt", 256, "cg", 0, {}),
    ("cg_7pt_g16", "7pt", 16, "cg", 0, {}),
    ("cg_bj32_7pt_g16", "7pt", 16, "cg", 32, {}),
    ("cg_7pt_g32", "7pt", 32, "cg", 0, {}),
    ("cg_7pt_g64", "7pt", 64, "cg", 0, {}),
    ("cg_7pt_g128", "7pt", 128, "cg", 0, {}),
    ("bicgstab_none_cd_g12", "convdiff", 12, "bicgstab", 0, {}),
    ("bicgstab_bj32_cd_g12", "convdiff", 12, "bicgstab", 32, {}),
    ("gmres30_none_cd_g12", "convdiff", 12, "gmres", 0, {"krylov_dim": 30}),
    ("gmres30_bj32_cd_g12", "convdiff", 12, "gmres", 32, {"krylov_dim": 30}),
    ("bicgstab_none_cd_g32", "convdiff", 32, "bicgstab", 0, {}),
    ("bicgstab_bj32_cd_g32", "convdiff", 32, "bicgstab", 32, {}),
    ("gmres30_none_cd_g32", "convdiff", 32, "gmres", 0, {"krylov_dim": 30}),
    ("gmres30_bj32_cd_g32", "convdiff", 32, "gmres", 32, {"krylov_dim": 30}),
]


@pytest.mark.parametrize("name,kind,g,solver,pre,kw", CASES, ids=[c[0] for c in CASES])
def test_iteration_count_and_residual_match_reference(cuda, golden_solvers, name, kind, g, solver, pre, kw):
    import paper_2006_16852_b200 as b2

    gold = golden_solvers[name]
    n, r, c, v = P.five_point(g) if kind == "5pt" else P.stencil3d(g, kind)
    a = system(b2, cuda, n, r, c, v)
    st, x = solve(b2, cuda, a, np.ones(n), solver, pre, **kw)
    ref_it = int(gold["iterations"])
    assert st.breakdown is None
    assert abs(st.iterations - ref_it) <= 1, (st.iterations, ref_it)
    assert st.converged and st.stopping_id == int(gold["stopping_id"])
    rel = true_rel_residual(csr_host(n, r, c, v), x[:, 0], np.ones(n))
    ref_rel = float(gold["true_res"][0]) / np.sqrt(n)
    assert rel <= max(ref_rel, 1e-8) * 2.0, (rel, ref_rel)
    if "x" in gold:
        xr = gold["x"][:, 0]
        assert np.linalg.norm(x[:, 0] - xr) <= 1e-6 * np.linalg.norm(xr)
    # residual history agrees while far from the floor
    hist = gold["history"][:, 0]
    assert hist.size == ref_it + 1


def test_c1_residual_history(cuda, golden_solvers):
    """C1: per-iteration residual norms reported through the logger match the
    reference's checks (relative 1e-6 while above 1e-6 of ||r0||)."""
    import paper_2006_16852_b200 as b2

    gold = golden_solvers["cg_c1"]
    n, r, c, v = P.five_point(256)
    a = system(b2, cuda, n, r, c, v)
    log = b2.RecordLogger(capacity=100000)
    b = b2.Dense(cuda, np.ones((n, 1)))
    x = b2.Dense.zeros(cuda, n, 1)
    s = b2.Cg(cuda, criteria=[b2.Iteration(10000), b2.ResidualNormReduction(1e-8)]).generate(a)
    s.attach(log)
    s.apply(b, x)
    checks = [e for e in log.query(b2.EventKind.CRITERION_CHECK_COMPLETED) if e[3]["relative_norms"]]
    rel = np.array([e[3]["relative_norms"][0] for e in checks])
    ref = gold["history"][:, 0] / gold["history"][0, 0]
    m = min(rel.size, ref.size)
    keep = ref[:m] > 1e-6
    np.testing.assert_allclose(rel[:m][keep], ref[:m][keep], rtol=1e-6)
    conv = b2.ConvergenceLogger()
    s.attach(conv)
    x2 = b2.Dense.zeros(cuda, n, 1)
    s.apply(b, x2)
    its, final = conv.result()
    assert abs(its - 470) <= 1 and final <= 1e-8


# ---------------------------------------------------------------------------
# reference test-suite behaviours (tests/test_solvers.py of the reference)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["cg", "bicgstab", "gmres"])
def test_identity_system_converges_first_iteration(cuda, name):
    import paper_2006_16852_b200 as b2

    data = b2.MatrixData((5, 5), range(5), range(5), [1.0] * 5)
    a = b2.matrix_from_data(cuda, data, "csr")
    bv = np.random.default_rng(1).standard_normal(5)
    b = b2.Dense.vector(cuda, bv)
    x = b2.Dense.zeros(cuda, 5, 1)
    s = b2.SOLVER_FACTORIES[name](cuda, criteria=[b2.Iteration(50), b2.ResidualNormReduction(1e-12)]).generate(a)
    s.apply(b, x)
    assert s.last_status.iterations == 1
    np.testing.assert_allclose(np.asarray(x.data)[:, 0], bv, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("name", ["cg", "bicgstab", "gmres"])
def test_zero_rhs_stops_at_iteration_zero(cuda, name):
    import paper_2006_16852_b200 as b2

    n, r, c, v = P.stencil3d(3, "7pt")
    a = system(b2, cuda, n, r, c, v)
    b = b2.Dense.zeros(cuda, n, 1)
    x = b2.Dense.zeros(cuda, n, 1)
    s = b2.SOLVER_FACTORIES[name](cuda, criteria=[b2.Iteration(50), b2.ResidualNormReduction(1e-8)]).generate(a)
    s.apply(b, x)
    assert s.last_status.iterations == 0
    assert np.array_equal(np.asarray(x.data), np.zeros((n, 1)))


def test_cg_breakdown_reported_on_indefinite(cuda):
    import paper_2006_16852_b200 as b2

    a = b2.matrix_from_data(cuda, b2.MatrixData((2, 2), [0, 1], [0, 1], [1.0, -1.0]), "csr")
    b = b2.Dense.vector(cuda, [0.0, 1.0])
    x = b2.Dense.zeros(cuda, 2, 1)
    s = b2.Cg(cuda, criteria=[b2.Iteration(10)]).generate(a)
    s.apply(b, x)
    assert s.last_status.breakdown is not None and s.last_status.breakdown.iteration == 1
    assert not s.last_status.converged


def test_bicgstab_breakdown_reported_on_skew(cuda):
    import paper_2006_16852_b200 as b2

    a = b2.matrix_from_data(cuda, b2.MatrixData((2, 2), [0, 1], [1, 0], [1.0, -1.0]), "csr")
    b = b2.Dense.vector(cuda, [1.0, 0.0])
    x = b2.Dense.zeros(cuda, 2, 1)
    s = b2.Bicgstab(cuda, criteria=[b2.Iteration(10)]).generate(a)
    s.apply(b, x)
    assert s.last_status.breakdown is not None


@pytest.mark.parametrize("name", ["cg", "bicgstab", "gmres"])
def test_nan_rhs_sustains_forced_iterations(cuda, name):
    import paper_2006_16852_b200 as b2

    a = b2.matrix_from_data(cuda, b2.MatrixData((1, 1), [0], [0], [1.0]), "coo")
    b = b2.Dense(cuda, [[float("nan")]])
    x = b2.Dense.zeros(cuda, 1, 1)
    kw = {"krylov_dim": 20} if name == "gmres" else {}
    s = b2.SOLVER_FACTORIES[name](cuda, criteria=[b2.Iteration(50)], **kw).generate(a)
    s.apply(b, x)
    assert s.last_status.iterations == 50


def test_identity_precond_bitwise_equals_unpreconditioned(cuda):
    import paper_2006_16852_b200 as b2

    data = random_spd(20, seed=10)
    bv = np.random.default_rng(10).standard_normal((20, 1))
    res = []
    for gen in (None, b2.Identity(cuda, 20)):
        a = b2.matrix_from_data(cuda, data, "csr")
        x = b2.Dense.zeros(cuda, 20, 1)
        s = b2.Cg(cuda, criteria=[b2.Iteration(30), b2.ResidualNormReduction(1e-10)],
                  generated_preconditioner=gen).generate(a)
        s.apply(b2.Dense(cuda, bv), x)
        res.append((s.last_status.iterations, np.asarray(x.data)))
    assert res[0][0] == res[1][0] and np.array_equal(res[0][1], res[1][1])


def test_gmres_restart_two_equals_full_on_2x2(cuda):
    import paper_2006_16852_b200 as b2

    data = b2.MatrixData((2, 2), [0, 0, 1, 1], [0, 1, 0, 1], [3.0, 1.0, -1.0, 2.0])
    bv = np.random.default_rng(5).standard_normal((2, 1))
    xs = []
    for k in (2, 50):
        a = b2.matrix_from_data(cuda, data, "csr")
        x = b2.Dense.zeros(cuda, 2, 1)
        b2.Gmres(cuda, criteria=[b2.Iteration(2)], krylov_dim=k).generate(a).apply(b2.Dense(cuda, bv), x)
        xs.append(np.asarray(x.data))
    assert np.array_equal(xs[0], xs[1])


def test_gmres_krylov_exactness_and_restarted(cuda, golden_solvers):
    import paper_2006_16852_b200 as b2

    data = random_sparse(24, density=0.3, seed=4)
    a = b2.matrix_from_data(cuda, data, "csr")
    bv = np.random.default_rng(4).standard_normal(24)
    st, x = solve(b2, cuda, a, bv, "gmres", iters=24, factor=1e-10, krylov_dim=30)
    assert st.iterations <= 24
    oracle = np.linalg.solve(data.to_dense_array(), bv)
    assert np.linalg.norm(x[:, 0] - oracle) <= 1e-10 * np.linalg.norm(oracle)
    gold = golden_solvers["gmres10_rand100"]
    data = random_sparse(100, density=0.1, seed=6)
    a = b2.matrix_from_data(cuda, data, "csr")
    st, x = solve(b2, cuda, a, gold["b"], "gmres", iters=3000, factor=1e-12, krylov_dim=10)
    assert abs(st.iterations - int(gold["iterations"])) <= 1
    assert np.linalg.norm(x[:, 0] - gold["x"][:, 0]) <= 1e-8 * np.linalg.norm(gold["x"])


def test_bicgstab_random_nonsymmetric(cuda, golden_solvers):
    import paper_2006_16852_b200 as b2

    gold = golden_solvers["bicgstab_rand100"]
    a = b2.matrix_from_data(cuda, random_sparse(100, density=0.1, seed=6), "csr")
    st, x = solve(b2, cuda, a, gold["b"], "bicgstab", iters=3000, factor=1e-12)
    assert abs(st.iterations - int(gold["iterations"])) <= 1
    assert np.linalg.norm(x[:, 0] - gold["x"][:, 0]) <= 1e-8 * np.linalg.norm(gold["x"])


def test_per_column_freeze_multi_rhs(cuda, golden_solvers):
    """Two right-hand sides (host-controlled loop): column 0 freezes bitwise
    once stopped; results match the reference run."""
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200.stop import Criterion, CriterionFactory

    gold = golden_solvers["cg_freeze"]
    data = random_spd(8, seed=11)
    a = b2.matrix_from_data(cuda, data, "csr")
    snaps = []

    class Freeze(Criterion):
        def check(self, stopping_id, set_finalized, status, updater):
            if status.data["stopped"][0] and not status.data["stopped"][1]:
                snaps.append(np.asarray(updater.solution.data)[:, 0].copy())
            return False, False

    class FreezeFactory(CriterionFactory):
        def generate(self, args):
            return Freeze()

    bd = b2.Dense(cuda, gold["b"])
    x = b2.Dense(cuda, np.zeros((8, 2)))
    s = b2.Cg(cuda, criteria=[b2.Iteration(60), b2.ResidualNormReduction(1e-10), FreezeFactory()]).generate(a)
    s.apply(bd, x)
    assert s.last_status.stopped["stopped"].all()
    assert s.last_status.iterations == int(gold["iterations"])
    for snap in snaps[1:]:
        assert np.array_equal(snap, snaps[0])
    np.testing.assert_allclose(np.asarray(x.data), gold["x"], rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("name", ["cg", "bicgstab", "gmres"])
def test_custom_criterion_host_loop_matches_device(cuda, name):
    """A user-defined criterion routes through the host-controlled loop; the
    iteration count equals the device-resident run."""
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200.stop import Criterion, CriterionFactory

    class Never(Criterion):
        def check(self, stopping_id, set_finalized, status, updater):
            return False, False

    class NeverFactory(CriterionFactory):
        def generate(self, args):
            return Never()

    n, r, c, v = P.stencil3d(10, "convdiff" if name != "cg" else "7pt")
    its = []
    for extra in ([], [NeverFactory()]):
        a = system(b2, cuda, n, r, c, v)
        b = b2.Dense(cuda, np.ones((n, 1)))
        x = b2.Dense.zeros(cuda, n, 1)
        kw = {"krylov_dim": 30} if name == "gmres" else {}
        s = b2.SOLVER_FACTORIES[name](cuda, criteria=[b2.Iteration(1000), b2.ResidualNormReduction(1e-8)] + extra,
                                      **kw).generate(a)
        s.apply(b, x)
        its.append(s.last_status.iterations)
    assert abs(its[0] - its[1]) <= 1, its


def test_solvers_on_every_format(cuda):
    import paper_2006_16852_b200 as b2

    n, r, c, v = P.stencil3d(12, "7pt")
    base = None
    for fmt in ("csr", "csr_classical", "csr_lb", "csr_stream", "coo", "ell", "sellp", "hybrid"):
        a = system(b2, cuda, n, r, c, v, fmt)
        st, x = solve(b2, cuda, a, np.ones(n), "cg")
        base = base or st.iterations
        assert abs(st.iterations - base) <= 1 and st.converged, fmt


def test_host_operands_end_to_end(cuda, host):
    import paper_2006_16852_b200 as b2

    n, r, c, v = P.stencil3d(16, "7pt")
    a = system(b2, cuda, n, r, c, v)
    b = b2.Dense(host, np.ones((n, 1)))
    x = b2.Dense(host, np.zeros((n, 1)))
    s = b2.Cg(cuda, criteria=[b2.Iteration(1000), b2.ResidualNormReduction(1e-8)]).generate(a)
    s.apply(b, x)
    assert abs(s.last_status.iterations - 39) <= 1
    assert true_rel_residual(csr_host(n, r, c, v), x.data[:, 0], np.ones(n)) <= 1.5e-8


# ---------------------------------------------------------------------------
# block-Jacobi
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("adaptive", [0, 1])
def test_jacobi_inverses_bitwise(cuda, golden_jacobi, adaptive):
    import paper_2006_16852_b200 as b2

    g = golden_jacobi[f"convdiff_g8_bs32_adapt{adaptive}"]
    n = int(g["n"])
    a = b2.matrix_from_data(cuda, b2.MatrixData((n, n), g["rows"], g["cols"], g["vals"]), "csr")
    jac = b2.Jacobi(cuda, block_size=32, adaptive_precision=bool(adaptive), condition_threshold=1e2).generate(a)
    assert np.array_equal(np.array(jac.block_conditions), g["cond"])
    assert np.array_equal(np.array([p == "reduced" for p in jac.block_precisions]), g["reduced"])
    for i in range(g["inv"].shape[0]):
        assert np.array_equal(jac.stored_inverse(i).astype(np.float64), g["inv"][i]), i


def test_jacobi_pivoting_blocks_and_apply(cuda, golden_jacobi):
    import paper_2006_16852_b200 as b2

    g = golden_jacobi["rand60_bs16"]
    a = b2.matrix_from_data(cuda, b2.MatrixData((60, 60), g["rows"], g["cols"], g["vals"]), "csr")
    jac = b2.Jacobi(cuda, block_size=16).generate(a)
    flat = np.concatenate([jac.stored_inverse(i).reshape(-1) for i in range(4)])
    assert np.array_equal(flat, g["inv_flat"])
    assert np.array_equal(np.array(jac.block_conditions), g["cond"])
    z = b2.Dense.zeros(cuda, 60, 1)
    jac.apply(b2.Dense(cuda, g["r"]), z)
    np.testing.assert_allclose(np.asarray(z.data), g["z"], rtol=1e-13, atol=1e-14)


def test_jacobi_single_block_is_exact_solve(cuda):
    import paper_2006_16852_b200 as b2

    data = random_spd(12, seed=7)
    a = b2.matrix_from_data(cuda, data, "csr")
    jac = b2.Jacobi(cuda, block_size=12).generate(a)
    bv = np.random.default_rng(7).standard_normal((12, 1))
    z = b2.Dense.zeros(cuda, 12, 1)
    jac.apply(b2.Dense(cuda, bv), z)
    np.testing.assert_allclose(np.asarray(z.data)[:, 0], np.linalg.solve(data.to_dense_array(), bv[:, 0]),
                               rtol=1e-10)


def test_jacobi_singular_block_raises(cuda):
    import paper_2006_16852_b200 as b2

    data = b2.MatrixData((4, 4), [0, 1, 2, 3], [0, 0, 2, 3], [1.0, 2.0, 1.0, 1.0])
    a = b2.matrix_from_data(cuda, data, "csr")
    with pytest.raises(b2.Singular):
        b2.Jacobi(cuda, block_size=2).generate(a)


def test_concurrent_applies_of_one_solver(cuda):
    """concurrent applies of one operator to disjoint outputs
    are safe: two host threads share one generated CG."""
    import threading

    import paper_2006_16852_b200 as b2

    n, r, c, v = P.stencil3d(16, "7pt")
    a = system(b2, cuda, n, r, c, v)
    s = b2.Cg(cuda, criteria=[b2.Iteration(1000), b2.ResidualNormReduction(1e-10)]).generate(a)
    rhs = [np.random.default_rng(k).standard_normal((n, 1)) for k in range(4)]
    out = [None] * 4

    def work(k):
        x = b2.Dense.zeros(cuda, n, 1)
        s.apply(b2.Dense(cuda, rhs[k]), x)
        out[k] = np.asarray(x.data)

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    m = csr_host(n, r, c, v)
    for k in range(4):
        assert true_rel_residual(m, out[k][:, 0], rhs[k][:, 0]) <= 1e-9


class _ResidualAgreement:
    """Recurrence vs true residual norms at consistent checks (the
    reference's tests/test_solvers.py:251-279 probe)."""

    def __init__(self, dense, b, even_only=False):
        self.dense, self.b, self.even_only = dense, b, even_only
        self.rows = []

    def check(self, stopping_id, set_finalized, status, updater):
        if self.even_only and updater.num_iterations % 2 == 1:
            return False, False
        true_r = None
        if updater.solution is not None:
            true_r = np.linalg.norm(self.b - self.dense @ np.asarray(updater.solution.data)[:, 0])
        if updater.residual is not None:
            rec = float(np.linalg.norm(np.asarray(updater.residual.data)))
        elif updater.residual_norm is not None:
            rec = float(updater.residual_norm[0])
        else:
            return False, False
        self.rows.append((rec, true_r))
        return False, False


def _probe_factory(b2, probe):
    class ProbeCrit(b2.stop.Criterion):
        def check(self, stopping_id, set_finalized, status, updater):
            return probe.check(stopping_id, set_finalized, status, updater)

    class ProbeFactory(b2.stop.CriterionFactory):
        def generate(self, args):
            return ProbeCrit()

    return ProbeFactory()


@pytest.mark.parametrize("name,tol", [("cg", 1e-6), ("fcg", 1e-6), ("cgs", 1e-6), ("bicgstab", 1e-6)])
def test_recurrence_residual_tracks_true_residual(cuda, name, tol):
    """Reference tests/test_solvers.py:282-306 (user-defined criterion: the
    host-controlled loop over device kernels)."""
    import paper_2006_16852_b200 as b2

    data = random_spd(40, seed=12) if name in ("cg", "fcg") else random_sparse(40, density=0.2, seed=12)
    dense = data.to_dense_array()
    a = b2.matrix_from_data(cuda, data, "csr")
    bv = np.random.default_rng(12).standard_normal(40)
    b = b2.Dense.vector(cuda, bv)
    x = b2.Dense.zeros(cuda, 40, 1)
    probe = _ResidualAgreement(dense, bv.copy(), even_only=(name == "bicgstab"))
    s = b2.SOLVER_FACTORIES[name](cuda, criteria=[b2.Iteration(25), _probe_factory(b2, probe)]).generate(a)
    s.apply(b, x)
    assert probe.rows
    bn = np.linalg.norm(bv)
    for rec, true_r in probe.rows:
        if true_r is None or true_r <= 1e-8 * bn:
            continue
        assert abs(rec - true_r) <= tol * max(true_r, 1e-300)


def test_gmres_rotation_residual_matches_true_residual(cuda):
    """Reference tests/test_solvers.py:309-333: the Givens estimate equals the
    true residual of the iterate committed at the stop."""
    import paper_2006_16852_b200 as b2

    data = random_sparse(40, density=0.2, seed=12)
    dense = data.to_dense_array()
    bv = np.random.default_rng(12).standard_normal(40)
    for j in (1, 3, 7, 12, 20):
        a = b2.matrix_from_data(cuda, data, "csr")
        x = b2.Dense.zeros(cuda, 40, 1)
        est = {}

        class Probe:
            def check(self, stopping_id, set_finalized, status, updater):
                est[updater.num_iterations] = float(updater.residual_norm[0])
                return False, False

        s = b2.Gmres(cuda, criteria=[b2.Iteration(j), _probe_factory(b2, Probe())], krylov_dim=50).generate(a)
        s.apply(b2.Dense.vector(cuda, bv), x)
        true_r = np.linalg.norm(bv - dense @ np.asarray(x.data)[:, 0])
        if true_r > 1e-10 * np.linalg.norm(bv):
            # + 1e-14 ||b||: near 1e-8 ||b|| the evaluation of b - A x itself
            # carries ~eps ||A|| ||x|| of rounding (j = 20 differs by 4.6e-16)
            assert abs(est[j] - true_r) <= 1e-8 * true_r + 1e-14 * np.linalg.norm(bv), j


@pytest.mark.parametrize("name", ["Bicgstab", "Cgs", "Fcg"])
def test_cooperative_small_system_path(cuda, monkeypatch, name):
    """Small unpreconditioned systems run BiCGSTAB / CGS / FCG as one
    persistent cooperative launch; it must agree with the batched kernels
    (same iteration count +-1, same solution to 1e-10)."""
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import _lib, config, problems

    kind = "7pt" if name == "Fcg" else "convdiff"
    a = problems.stencil(cuda, kind, 16)
    n = a.size.rows
    res = {}
    for coop in (True, False):
        monkeypatch.setattr(config, "BICGSTAB_COOP", coop)
        s = getattr(b2, name)(cuda, criteria=[b2.Iteration(2000), b2.ResidualNormReduction(1e-10)]).generate(a)
        x = b2.Dense.zeros(cuda, n, 1)
        l0 = _lib.launch_count()
        s.apply(b2.Dense(cuda, np.ones((n, 1))), x)
        res[coop] = (s.last_status.iterations, np.asarray(x.data).copy(), _lib.launch_count() - l0)
    assert res[True][0] > 0 and abs(res[True][0] - res[False][0]) <= 1
    assert res[True][2] < res[False][2]  # one solve launch vs batches of step kernels
    np.testing.assert_allclose(res[True][1], res[False][1], rtol=0, atol=1e-10 * np.abs(res[False][1]).max())


def test_cg_cooperative_variants_and_counter_reuse(cuda):
    """C1-style CG through the persistent cooperative kernels: the
    global-memory kernel and the register-resident one give bitwise the same
    iterate at the same CTA shape; the register-resident one with its fenced
    or flag-in-data sigma exchange and 256 / 512-thread CTAs stays within the
    reference's iteration count; and the grid-exchange counter (reset by the
    last CTA out) survives back-to-back solves of different sizes."""
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import _lib, problems

    def solve(a):
        n = a.size.rows
        s = b2.Cg(cuda, criteria=[b2.Iteration(10000), b2.ResidualNormReduction(1e-8)]).generate(a)
        x = b2.Dense.zeros(cuda, n, 1)
        s.apply(b2.Dense(cuda, np.ones((n, 1))), x)
        return s.last_status.iterations, np.asarray(x.data).copy()

    a = problems.stencil(cuda, "5pt", 128)
    small = problems.stencil(cuda, "5pt", 20)
    knobs = ("coop_resident", "coop_res_block", "coop_nofence")
    try:
        _lib.set_tuning("coop_res_block", 256)
        _lib.set_tuning("coop_nofence", 0)
        _lib.set_tuning("coop_resident", 0)
        it0, x0 = solve(a)
        _lib.set_tuning("coop_resident", 1)
        it1, x1 = solve(a)
        assert it0 == it1 and np.array_equal(x0, x1)
        for bs in (256, 512):
            for nofence in (0, 1):
                _lib.set_tuning("coop_res_block", bs)
                _lib.set_tuning("coop_nofence", nofence)
                runs = [solve(a), solve(small), solve(a)]
                assert runs[0][0] == runs[2][0] and np.array_equal(runs[0][1], runs[2][1])  # counter reset
                assert abs(runs[0][0] - it0) <= 1
                np.testing.assert_allclose(runs[0][1], x0, rtol=0, atol=1e-9 * np.abs(x0).max())
    finally:
        for k in knobs:
            _lib.reset_tuning(k)
