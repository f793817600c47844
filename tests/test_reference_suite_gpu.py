"""The reference's own API-behaviour suite, run against the CUDA executor.

A port of /root/reference/pkg/tests/test_linop.py, test_stop.py,
test_formats.py and test_solvers.py: the same statements with the `ref`
fixture replaced by `CudaExecutor` (and `par` by a second, independent
`CudaExecutor` on the same device), so a user switching backends sees the
same observable contract -- dimension checks, composition, clone_to
rebinding, give/share/lend ownership, criteria semantics (incl. the
randomized Combined-OR property and per-iteration TimeLimit), the
format-equivalence hypothesis property over every format this backend
adds, and the solver behaviours. Where the reference compares its
ReferenceExecutor with its CPU ParallelExecutor, the port compares two
CUDA executors (bitwise). Tests are named after their reference originals.
"""

from __future__ import annotations

import time

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2006_16852_b200 as opalg
from paper_2006_16852_b200 import (Composition, Coo, Csr, Dense, Dim2, DimensionMismatch, Identity, Iteration,
                                   MatrixData, ParameterError, ResidualNormReduction, Singular, StencilMatrix,
                                   Unsupported, clone, compose, convert, give, lend, share)
from paper_2006_16852_b200.problems import (convection_diffusion, random_sparse, random_spd, tridiagonal)
from paper_2006_16852_b200.solvers import LowerTrs, UpperTrs
from paper_2006_16852_b200.stop import (Combined, Criterion, CriterionArgs, CriterionFactory, TimeLimit, Updater,
                                        new_stopping_status)

pytestmark = pytest.mark.gpu

ALL_KRYLOV = ["cg", "fcg", "cgs", "bicgstab", "gmres"]
FORMATS = ["csr", "coo", "dense"]
# formats this backend adds (reference SPEC.md:294 names them, no implementation)
B200_FORMATS = ["ell", "sellp", "hybrid", "csr_classical", "csr_lb", "csr_stream"]


@pytest.fixture(scope="module")
def ref():
    return opalg.CudaExecutor(0)


@pytest.fixture(scope="module")
def par():
    return opalg.CudaExecutor(0)


def make_system(exc, data, fmt="csr", rhs=None, seed=0):
    """reference tests/conftest.py:31-39"""
    a = opalg.matrix_from_data(exc, data, fmt)
    n = a.size.rows
    if rhs is None:
        rhs = np.random.default_rng(seed).standard_normal(n)
    b = Dense.vector(exc, rhs)
    x = Dense.zeros(exc, n, 1)
    return a, b, x


def _factory(name, exc, criteria, **kw):
    return opalg.SOLVER_FACTORIES[name](exc, criteria=criteria, **kw)


# ===========================================================================
# test_linop.py
# ===========================================================================
def test_identity_apply(ref):
    ident = Identity(ref, 3)
    b = Dense.vector(ref, [1.0, 2.0, 3.0])
    x = Dense.zeros(ref, 3, 1)
    ident.apply(b, x)
    np.testing.assert_array_equal(x.data[:, 0], [1, 2, 3])


def test_csr_apply_known_values(ref):
    a = Csr.from_data(ref, tridiagonal(3))
    b = Dense.vector(ref, [1.0, 1.0, 1.0])
    x = Dense.zeros(ref, 3, 1)
    a.apply(b, x)
    np.testing.assert_allclose(x.data[:, 0], [1.0, 0.0, 1.0], atol=0)
    np.testing.assert_array_equal(x.data[:, 0], tridiagonal(3).to_dense_array() @ np.ones(3))


def test_multicolumn_apply_is_columnwise(ref):
    data = tridiagonal(5, -1.0, 3.0, -2.0)
    a = Csr.from_data(ref, data)
    cols = np.random.default_rng(0).standard_normal((5, 2))
    x = Dense.zeros(ref, 5, 2)
    a.apply(Dense(ref, cols), x)
    for j in range(2):
        xj = Dense.zeros(ref, 5, 1)
        a.apply(Dense.vector(ref, cols[:, j]), xj)
        np.testing.assert_array_equal(x.data[:, j], xj.data[:, 0])


def test_apply_dimension_checks(ref):
    a = Csr.from_data(ref, tridiagonal(4))
    with pytest.raises(DimensionMismatch):
        a.apply(Dense.zeros(ref, 3, 1), Dense.zeros(ref, 4, 1))
    with pytest.raises(DimensionMismatch):
        a.apply(Dense.zeros(ref, 4, 1), Dense.zeros(ref, 5, 1))
    with pytest.raises(DimensionMismatch):
        a.apply(Dense.zeros(ref, 4, 2), Dense.zeros(ref, 4, 1))


def test_sparse_operands_rejected(ref):
    a = Csr.from_data(ref, tridiagonal(3))
    other = Csr.from_data(ref, tridiagonal(3))
    with pytest.raises(Unsupported):
        a.apply(other, Dense.zeros(ref, 3, 1))


def test_advanced_apply_identities(ref):
    a = Csr.from_data(ref, tridiagonal(6, -1, 4, -1))
    rng = np.random.default_rng(1)
    b = Dense(ref, rng.standard_normal((6, 1)))
    x0 = rng.standard_normal((6, 1))
    x1 = Dense(ref, x0.copy())
    a.apply_advanced(1.0, b, 0.0, x1)
    x2 = Dense.zeros(ref, 6, 1)
    a.apply(b, x2)
    np.testing.assert_allclose(x1.data, x2.data, rtol=0, atol=1e-15)
    x3 = Dense(ref, x0.copy())
    a.apply_advanced(0.0, b, 1.0, x3)
    np.testing.assert_array_equal(x3.data, x0)
    ident = Identity(ref, 6)
    x4 = Dense(ref, x0.copy())
    ident.apply_advanced(2.0, Dense(ref, x0.copy()), -1.0, x4)
    np.testing.assert_allclose(x4.data, x0, rtol=1e-15)


def test_advanced_apply_with_dense_scalars(ref):
    a = Csr.from_data(ref, tridiagonal(4))
    x = Dense.vector(ref, [1.0, 1.0, 1.0, 1.0])
    a.apply_advanced(Dense(ref, [[2.0]]), Dense.vector(ref, [1.0, 0.0, 0.0, 1.0]), Dense(ref, [[-1.0]]), x)
    oracle = 2.0 * (tridiagonal(4).to_dense_array() @ [1, 0, 0, 1]) - 1.0
    np.testing.assert_allclose(x.data[:, 0], oracle, rtol=1e-15)


def test_generate_solver_solves(ref):
    data = random_spd(20, seed=2)
    a, b, x = make_system(ref, data, seed=2)
    solver = opalg.Cg(ref, criteria=[Iteration(500), ResidualNormReduction(1e-12)]).generate(a)
    solver.apply(b, x)
    oracle = np.linalg.solve(data.to_dense_array(), b.data[:, 0])
    np.testing.assert_allclose(x.data[:, 0], oracle, rtol=1e-8, atol=1e-10)


def test_nested_factory_generates_from_same_matrix(ref):
    data = random_spd(12, seed=3)
    a, b, x = make_system(ref, data, seed=3)
    solver = opalg.Cg(ref, criteria=[Iteration(100)], preconditioner=opalg.Jacobi(ref)).generate(a)
    standalone = opalg.Jacobi(ref).generate(a)
    r = Dense.vector(ref, np.arange(1.0, 13.0))
    z1, z2 = Dense.zeros(ref, 12, 1), Dense.zeros(ref, 12, 1)
    solver.precond.apply(r, z1)
    standalone.apply(r, z2)
    np.testing.assert_array_equal(z1.data, z2.data)


def test_generate_rejects_non_square(ref):
    a = Csr.from_data(ref, MatrixData(Dim2(3, 4), [0], [0], [1.0]))
    with pytest.raises(DimensionMismatch):
        opalg.Cg(ref, criteria=[Iteration(5)]).generate(a)


def test_factory_generate_repeatable(ref):
    data = random_spd(10, seed=4)
    factory = opalg.Cg(ref, criteria=[Iteration(30)])
    a1, b1, x1 = make_system(ref, data, seed=4)
    a2, b2, x2 = make_system(ref, data, seed=4)
    factory.generate(a1).apply(b1, x1)
    factory.generate(a2).apply(b2, x2)
    assert np.array_equal(x1.data, x2.data)


def test_compose_identity_is_noop(ref):
    a = Csr.from_data(ref, tridiagonal(5))
    comp = compose(Identity(ref, 5), a)
    b = Dense.vector(ref, np.arange(5.0))
    x1, x2 = Dense.zeros(ref, 5, 1), Dense.zeros(ref, 5, 1)
    comp.apply(b, x1)
    a.apply(b, x2)
    np.testing.assert_array_equal(x1.data, x2.data)


def test_compose_matches_dense_product(ref):
    rng = np.random.default_rng(5)
    a_arr, b_arr = rng.standard_normal((3, 3)), rng.standard_normal((3, 3))
    comp = compose(Dense(ref, a_arr), Dense(ref, b_arr))
    assert tuple(comp.size) == (3, 3)
    v = rng.standard_normal(3)
    out = Dense.zeros(ref, 3, 1)
    comp.apply(Dense.vector(ref, v), out)
    np.testing.assert_allclose(out.data[:, 0], a_arr @ (b_arr @ v), rtol=1e-13)


def test_compose_empty_and_nonconformal(ref):
    with pytest.raises(DimensionMismatch):
        Composition([])
    with pytest.raises(DimensionMismatch):
        compose(Dense(ref, np.ones((2, 3))), Dense(ref, np.ones((2, 3))))


def test_clone_to_preserves_behavior(ref, par):
    data = tridiagonal(40, -1.0, 2.5, -0.5)
    a = Csr.from_data(ref, data)
    a2 = opalg.clone_to(a, par)
    assert tuple(a2.size) == tuple(a.size)
    v = np.random.default_rng(6).standard_normal(40)
    x1, x2 = Dense.zeros(ref, 40, 1), Dense.zeros(par, 40, 1)
    a.apply(Dense.vector(ref, v), x1)
    a2.apply(Dense.vector(par, v), x2)
    np.testing.assert_array_equal(x1.data, x2.data)


def test_clone_solver_rebinds_matrix(ref, par):
    data = random_spd(15, seed=7)
    a, b, x = make_system(ref, data, seed=7)
    solver = opalg.Cg(ref, criteria=[Iteration(200), ResidualNormReduction(1e-10)]).generate(a)
    cloned = solver.clone_to(par)
    assert cloned.a is not solver.a
    x2 = Dense.zeros(par, 15, 1)
    solver.apply(b, x)
    cloned.apply(Dense.vector(par, b.data[:, 0]), x2)
    np.testing.assert_allclose(x2.data, x.data, rtol=1e-10)


def test_apply_repeatable_bitwise(ref):
    data = random_spd(25, seed=8)
    a, b, x = make_system(ref, data, seed=8)
    solver = opalg.Gmres(ref, criteria=[Iteration(40)], krylov_dim=10).generate(a)
    solver.apply(b, x)
    first = np.array(x.data)
    x.fill(0.0)
    solver.apply(b, x)
    assert np.array_equal(x.data, first)


def test_executor_transparency(ref, par):
    """Reference: Reference/Parallel/Instrumented executors agree; here two
    independent CUDA executors and a host-operand apply agree bitwise."""
    data = random_spd(30, seed=9)
    v = np.random.default_rng(9).standard_normal(30)
    results = []
    for exc in (ref, par):
        a = Csr.from_data(exc, data)
        x = Dense.zeros(exc, 30, 1)
        a.apply(Dense.vector(exc, v), x)
        results.append(np.array(x.data))
    host = opalg.HostExecutor()
    xh = Dense.zeros(host, 30, 1)
    Csr.from_data(ref, data).apply(Dense.vector(host, v), xh)
    assert np.array_equal(results[0], results[1])
    assert np.array_equal(results[0], np.asarray(xh.data))


def test_auto_migration_copies_back_output(ref):
    host = opalg.HostExecutor()
    a = Csr.from_data(ref, tridiagonal(8))
    b = Dense.vector(host, np.ones(8))
    x = Dense.zeros(host, 8, 1)
    a.apply(b, x)
    np.testing.assert_array_equal(x.data[:, 0], tridiagonal(8).to_dense_array() @ np.ones(8))
    assert x.exec is host
    np.testing.assert_array_equal(b.data[:, 0], np.ones(8))


def test_give_then_use_detected(ref):
    a = Csr.from_data(ref, tridiagonal(4, -1, 4, -1))
    solver = opalg.Cg(ref, criteria=[Iteration(3)]).generate(give(a))
    with pytest.raises(opalg.ContractViolation):
        a.apply(Dense.zeros(ref, 4, 1), Dense.zeros(ref, 4, 1))
    x = Dense.zeros(ref, 4, 1)
    solver.apply(Dense.vector(ref, np.ones(4)), x)
    assert solver.last_status.iterations == 3


def test_share_and_lend_leave_source_usable(ref):
    a = Csr.from_data(ref, tridiagonal(4, -1, 4, -1))
    opalg.Cg(ref, criteria=[Iteration(2)]).generate(share(a))
    x = Dense.zeros(ref, 4, 1)
    lend(a).apply(Dense.vector(ref, np.ones(4)), x)
    np.testing.assert_array_equal(x.data[:, 0], tridiagonal(4, -1, 4, -1).to_dense_array() @ np.ones(4))


def test_clone_pass_mode_leaves_source_independent(ref):
    a = Csr.from_data(ref, tridiagonal(4, -1, 4, -1))
    solver = opalg.Cg(ref, criteria=[Iteration(2)]).generate(clone(a))
    assert solver.a is not a
    a.vals[:] = 0.0  # write-through DeviceView: mutates the source on the device
    assert float(np.asarray(a.vals).max()) == 0.0
    assert solver.a.vals.max() == 4.0


# ===========================================================================
# test_stop.py
# ===========================================================================
def _args(exc, n=4, m=1):
    return CriterionArgs(None, Dense.zeros(exc, n, m), Dense.zeros(exc, n, m), None)


def test_reduction_factor_validation():
    for bad in (0.0, 1.0, -0.5, 2.0):
        with pytest.raises(ParameterError):
            ResidualNormReduction(bad)
    ResidualNormReduction(1e-15)


def test_iteration_and_time_validation():
    with pytest.raises(ParameterError):
        Iteration(-1)
    with pytest.raises(ParameterError):
        TimeLimit(0.0)
    with pytest.raises(ParameterError):
        Combined([])


def test_iteration_boundary(ref):
    crit = Iteration(20).generate(_args(ref))
    status = new_stopping_status(ref, 1)
    assert crit.check(1, True, status, Updater(19)) == (False, False)
    assert crit.check(1, True, status, Updater(20)) == (True, True)
    assert status.data["stopped"].all() and status.data["finalized"].all()
    assert (status.data["stopping_id"] == 1).all()


def test_iteration_does_not_overwrite_stopped_columns(ref):
    crit = Iteration(5).generate(_args(ref, m=3))
    status = new_stopping_status(ref, 3)
    status.data["stopped"][1] = True
    status.data["stopping_id"][1] = 7
    assert crit.check(1, False, status, Updater(5))[0]
    assert status.data["stopping_id"].tolist() == [1, 7, 1]


def test_monotonic_once_stopped(ref):
    crit = Iteration(3).generate(_args(ref))
    status = new_stopping_status(ref, 1)
    assert crit.check(1, True, status, Updater(3))[0]
    for it in (4, 5, 100):
        assert crit.check(1, True, status, Updater(it))[0]
        assert status.data["stopped"].all()


def test_rnr_stops_at_reduction(ref):
    crit = ResidualNormReduction(0.25).generate(_args(ref))
    status = new_stopping_status(ref, 1)
    assert not crit.check(1, True, status, Updater(0, residual_norm=[4.0]))[0]
    assert not crit.check(1, True, status, Updater(1, residual_norm=[1.5]))[0]
    assert crit.check(1, True, status, Updater(2, residual_norm=[1.0]))[0]


def test_rnr_baseline_from_initial_residual(ref):
    crit = ResidualNormReduction(0.5).generate(CriterionArgs(None, None, None, Dense.vector(ref, [3.0, 4.0])))
    status = new_stopping_status(ref, 1)
    assert not crit.check(1, True, status, Updater(0, residual_norm=[2.6]))[0]
    assert crit.check(1, True, status, Updater(1, residual_norm=[2.5]))[0]


def test_rnr_requires_residual_information(ref):
    crit = ResidualNormReduction(0.5).generate(_args(ref))
    with pytest.raises(Unsupported):
        crit.check(1, True, new_stopping_status(ref, 1), Updater(0))


def test_rnr_norm_from_residual_vector(ref):
    crit = ResidualNormReduction(0.5).generate(_args(ref))
    status = new_stopping_status(ref, 2)
    assert not crit.check(1, True, status, Updater(0, residual=Dense(ref, np.array([[3.0, 0.3], [4.0, 0.4]]))))[0]
    assert not crit.check(1, True, status, Updater(1, residual=Dense(ref, np.array([[1.4, 0.3], [2.0, 0.4]]))))[0]
    assert status.data["stopped"].tolist() == [True, False]


def test_generates_are_independent(ref):
    factory = ResidualNormReduction(0.5)
    c1, c2 = factory.generate(_args(ref)), factory.generate(_args(ref))
    s1, s2 = new_stopping_status(ref, 1), new_stopping_status(ref, 1)
    c1.check(1, True, s1, Updater(0, residual_norm=[10.0]))
    c2.check(1, True, s2, Updater(0, residual_norm=[2.0]))
    assert c1.check(1, True, s1, Updater(1, residual_norm=[4.9]))[0]
    assert not c2.check(1, True, s2, Updater(1, residual_norm=[1.5]))[0]


def test_time_criterion_stops_after_limit(ref):
    crit = TimeLimit(0.05).generate(_args(ref))
    status = new_stopping_status(ref, 1)
    assert not crit.check(1, True, status, Updater(0))[0]
    time.sleep(0.06)
    assert crit.check(1, True, status, Updater(1))[0]


def test_time_criteria_staggered_independent(ref):
    factory = TimeLimit(0.08)
    c1 = factory.generate(_args(ref))
    time.sleep(0.05)
    c2 = factory.generate(_args(ref))
    time.sleep(0.04)
    assert c1.check(1, True, new_stopping_status(ref, 1), Updater(0))[0]
    assert not c2.check(1, True, new_stopping_status(ref, 1), Updater(0))[0]


def test_combined_or_dominance(ref):
    crit = Combined([Iteration(5), TimeLimit(36000)]).generate(_args(ref))
    status = new_stopping_status(ref, 1)
    assert not crit.check(1, True, status, Updater(4))[0]
    assert crit.check(1, True, status, Updater(5))[0]
    assert status.data["stopping_id"][0] == 1


def test_combined_holds_generated_children(ref):
    assert len(Combined([Iteration(5), Iteration(7), TimeLimit(100)]).generate(_args(ref)).children) == 3


def test_combined_single_equals_bare(ref):
    bare = Iteration(4).generate(_args(ref))
    comb = Combined([Iteration(4)]).generate(_args(ref))
    s1, s2 = new_stopping_status(ref, 2), new_stopping_status(ref, 2)
    for it in range(6):
        assert bare.check(1, True, s1, Updater(it))[0] == comb.check(1, True, s2, Updater(it))[0]
        assert np.array_equal(s1.data["stopped"], s2.data["stopped"])


class _ScriptedCriterion(Criterion):
    def __init__(self, plan):
        super().__init__()
        self.plan = np.asarray(plan)

    def check(self, stopping_id, set_finalized, status, updater):
        changed = self._mark(status, updater.num_iterations >= self.plan, stopping_id, set_finalized)
        return bool(status.data["stopped"].all()), changed


class _ScriptedFactory(CriterionFactory):
    def __init__(self, plan):
        self.plan = plan

    def generate(self, args):
        return _ScriptedCriterion(self.plan)


def test_combined_equals_per_column_or_randomized(ref):
    rng = np.random.default_rng(2024)
    for _ in range(300):
        m = int(rng.integers(1, 5))
        plans = rng.integers(0, 8, size=(int(rng.integers(1, 5)), m))
        crit = Combined([_ScriptedFactory(p) for p in plans]).generate(_args(ref, m=m))
        status = new_stopping_status(ref, m)
        for it in range(10):
            stopped_all, _ = crit.check(1, True, status, Updater(it))
            oracle = (plans <= it).any(axis=0)
            assert np.array_equal(status.data["stopped"], oracle)
            assert stopped_all == oracle.all()


def test_two_rhs_column_convergence_order(ref):
    data = random_spd(8, seed=1)
    a = Csr.from_data(ref, data)
    dense = data.to_dense_array()
    w, v = np.linalg.eigh(dense)
    b = np.stack([dense @ v[:, 0], np.ones(8)], axis=1)
    x = Dense.zeros(ref, 8, 2)
    solver = opalg.Cg(ref, criteria=[Iteration(100), ResidualNormReduction(1e-10)]).generate(a)
    solver.apply(Dense(ref, b), x)
    assert solver.last_status.stopped["stopped"].all()
    np.testing.assert_allclose(x.data, np.linalg.solve(dense, b), rtol=1e-7, atol=1e-9)


# -- TimeLimit inside a device-resident solve (reference src/stop.py:134-147:
#    checked at every iteration) ------------------------------------------------
@pytest.mark.parametrize("name", ["cg", "bicgstab", "gmres", "fcg", "cgs"])
def test_time_limit_stops_device_solve_per_iteration(ref, name):
    from paper_2006_16852_b200 import problems

    # 128^3: ~0.1 ms per iteration, so the limit lands after a few hundred
    # iterations -- long before the recurrence residual underflows toward the
    # 1e-300 reduction (it keeps shrinking past machine precision)
    a = problems.stencil(ref, "7pt" if name in ("cg", "fcg") else "convdiff", 128)
    n = a.size.rows
    limit = 0.05
    crit = [Iteration(1_000_000), ResidualNormReduction(1e-300), TimeLimit(limit)]
    kw = {"krylov_dim": 30} if name == "gmres" else {}
    s = _factory(name, ref, crit, **kw).generate(a)
    x = Dense.zeros(ref, n, 1)
    b = Dense.vector(ref, np.ones(n))
    s.apply(b, x)  # warm-up (plans, graph capture)
    x.fill(0.0)
    t0 = time.monotonic()
    s.apply(b, x)
    wall = time.monotonic() - t0
    st_ = s.last_status
    assert st_.stopped["stopped"].all() and st_.stopping_id == 3, st_
    assert st_.iterations > 2
    # the stop lands within about one iteration of the limit, not a batch later
    per_it = wall / st_.iterations
    assert wall >= limit * 0.9
    assert wall <= limit + 0.02 + 4 * per_it, (wall, per_it)


# ===========================================================================
# test_formats.py
# ===========================================================================
@pytest.mark.parametrize("fmt", FORMATS + B200_FORMATS)
def test_spmv_tridiagonal_known_result(ref, fmt):
    a = convert(opalg.matrix_from_data(ref, tridiagonal(3), "csr"), fmt)
    x = Dense.zeros(ref, 3, 1)
    a.apply(Dense.vector(ref, [1.0, 2.0, 3.0]), x)
    np.testing.assert_array_equal(x.data[:, 0], [0.0, 0.0, 4.0])


@pytest.mark.parametrize("fmt", ["csr", "coo"] + B200_FORMATS)
def test_spmv_empty_matrix(ref, fmt):
    a = convert(opalg.matrix_from_data(ref, MatrixData(Dim2(4, 4)), "csr"), fmt)
    x = Dense(ref, np.full((4, 1), 7.0))
    a.apply(Dense.vector(ref, np.ones(4)), x)
    np.testing.assert_array_equal(x.data, np.zeros((4, 1)))


@pytest.mark.parametrize("fmt", FORMATS + B200_FORMATS)
def test_spmv_one_by_one(ref, fmt):
    a = convert(opalg.matrix_from_data(ref, MatrixData(Dim2(1, 1), [0], [0], [2.5]), "csr"), fmt)
    x = Dense.zeros(ref, 1, 1)
    a.apply(Dense.vector(ref, [3.0]), x)
    assert x.data[0, 0] == 7.5


def test_stencil_apply_known_values(ref):
    x = Dense.zeros(ref, 3, 1)
    StencilMatrix(ref, 3, -1.0, 2.0, -1.0).apply(Dense.vector(ref, [1.0, 1.0, 1.0]), x)
    np.testing.assert_array_equal(x.data[:, 0], [1.0, 0.0, 1.0])


def test_stencil_identity_coefficients(ref):
    v = np.arange(5.0)
    x = Dense.zeros(ref, 5, 1)
    StencilMatrix(ref, 5, 0.0, 1.0, 0.0).apply(Dense.vector(ref, v), x)
    np.testing.assert_array_equal(x.data[:, 0], v)


def test_stencil_matches_assembled_csr(ref):
    s = StencilMatrix(ref, 64, -1.0, 2.0, -1.0)
    c = convert(s, Csr)
    v = np.random.default_rng(0).standard_normal(64)
    xs, xc = Dense.zeros(ref, 64, 1), Dense.zeros(ref, 64, 1)
    s.apply(Dense.vector(ref, v), xs)
    c.apply(Dense.vector(ref, v), xc)
    assert np.abs(np.asarray(xs.data) - np.asarray(xc.data)).max() <= 1e-14 * np.abs(xc.data).max()


def test_stencil_to_csr_row_ptrs(ref):
    np.testing.assert_array_equal(convert(StencilMatrix(ref, 3, -1.0, 2.0, -1.0), Csr).row_ptrs, [0, 2, 5, 7])


def test_stencil_only_converts_to_csr(ref):
    with pytest.raises(Unsupported):
        convert(StencilMatrix(ref, 3, -1.0, 2.0, -1.0), Coo)


def test_conversion_round_trip_identity(ref):
    coo = Coo.from_data(ref, tridiagonal(6, -1.5, 4.0, -0.5).canonicalize())
    back = convert(convert(coo, Csr), Coo)
    np.testing.assert_array_equal(back.row_idxs, coo.row_idxs)
    np.testing.assert_array_equal(back.col_idxs, coo.col_idxs)
    np.testing.assert_array_equal(back.vals, coo.vals)


def test_dense_zero_converts_to_empty_sparse(ref):
    assert convert(Dense(ref, np.zeros((2, 2))), Csr).nnz == 0


@pytest.mark.parametrize("src", FORMATS + ["ell", "sellp", "hybrid"])
@pytest.mark.parametrize("dst", FORMATS + ["ell", "sellp", "hybrid"])
def test_conversion_preserves_triples(ref, src, dst):
    data = random_sparse(12, density=0.3, seed=5).canonicalize()
    a = convert(opalg.matrix_from_data(ref, data, "csr"), src)
    out = convert(a, dst).to_data().canonicalize()
    np.testing.assert_array_equal(out.rows, data.rows)
    np.testing.assert_array_equal(out.cols, data.cols)
    np.testing.assert_allclose(out.vals, data.vals, rtol=0, atol=0)


def test_matrix_data_canonicalize_sums_duplicates():
    canon = MatrixData(Dim2(2, 2), [1, 0, 1, 1], [0, 0, 0, 1], [2.0, 1.0, 3.0, 4.0]).canonicalize()
    assert canon.nnz == 3
    np.testing.assert_array_equal(canon.rows, [0, 1, 1])
    np.testing.assert_array_equal(canon.cols, [0, 0, 1])
    np.testing.assert_array_equal(canon.vals, [1.0, 5.0, 4.0])


def test_dense_blas_properties(ref):
    rng = np.random.default_rng(11)
    x = Dense(ref, rng.standard_normal((50, 2)))
    y = Dense(ref, rng.standard_normal((50, 2)))
    np.testing.assert_array_equal(x.dot(y), y.dot(x))
    for n2, d in zip(np.asarray(x.norm2()) ** 2, np.asarray(x.dot(x))):
        assert abs(n2 - d) <= 4 * np.spacing(d)
    y0 = np.array(y.data)
    y.add_scaled(0.7, x)
    y.add_scaled(-0.7, x)
    assert np.abs(np.asarray(y.data) - y0).max() <= 1e-15 * np.abs(y0).max()


def test_dense_stride_view(ref):
    import torch

    base = torch.zeros((6, 5), dtype=torch.float64, device=ref.device)
    base[:, :3] = torch.arange(18.0, dtype=torch.float64).reshape(6, 3)
    d = Dense.wrap(ref, base[:, :3])
    assert d.stride == 5
    assert tuple(d.size) == (6, 3)


@settings(max_examples=30, deadline=None)
@given(n=st.integers(1, 24), density=st.floats(0.05, 0.5), seed=st.integers(0, 1000))
def test_format_equivalence_property(n, density, seed):
    exc = opalg.CudaExecutor(0)
    data = random_sparse(n, density=density, seed=seed, diag_dominant=False)
    dense = data.to_dense_array()
    v = np.random.default_rng(seed).standard_normal(n)
    oracle = dense @ v
    scale = max(np.abs(oracle).max(), 1e-300)
    base = opalg.matrix_from_data(exc, data, "csr")
    for fmt in FORMATS + B200_FORMATS:
        a = opalg.matrix_from_data(exc, data, fmt) if fmt in FORMATS else convert(base, fmt)
        x = Dense.zeros(exc, n, 1)
        a.apply(Dense.vector(exc, v), x)
        assert np.abs(np.asarray(x.data)[:, 0] - oracle).max() <= 1e-13 * scale, fmt


# ===========================================================================
# test_solvers.py
# ===========================================================================
@pytest.mark.parametrize("name", ALL_KRYLOV)
def test_identity_system_converges_first_iteration(ref, name):
    a, b, x = make_system(ref, MatrixData(Dim2(5, 5), range(5), range(5), [1.0] * 5), seed=1)
    s = _factory(name, ref, [Iteration(50), ResidualNormReduction(1e-12)]).generate(a)
    s.apply(b, x)
    assert s.last_status.iterations == (2 if name == "cgs" else 1)
    np.testing.assert_allclose(x.data, b.data, rtol=1e-12, atol=1e-14)


def test_cg_matches_dense_oracle_tridiag(ref):
    data = tridiagonal(50)
    a, b, x = make_system(ref, data, seed=2)
    _factory("cg", ref, [Iteration(500), ResidualNormReduction(1e-12)]).generate(a).apply(b, x)
    oracle = np.linalg.solve(data.to_dense_array(), b.data[:, 0])
    assert np.linalg.norm(x.data[:, 0] - oracle) / np.linalg.norm(oracle) <= 1e-8


@pytest.mark.parametrize("name", ["cgs", "bicgstab"])
def test_nonsymmetric_convection_diffusion(ref, name):
    data = convection_diffusion(100)
    a, b, x = make_system(ref, data, seed=3)
    s = _factory(name, ref, [Iteration(4000), ResidualNormReduction(1e-10)]).generate(a)
    s.apply(b, x)
    assert s.last_status.converged
    r = b.data[:, 0] - data.to_dense_array() @ x.data[:, 0]
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(b.data) * 1.01
    oracle = np.linalg.solve(data.to_dense_array(), b.data[:, 0])
    assert np.linalg.norm(x.data[:, 0] - oracle) / np.linalg.norm(oracle) <= 1e-6


def test_gmres_krylov_exactness(ref):
    data = random_sparse(24, density=0.3, seed=4)
    a, b, x = make_system(ref, data, seed=4)
    s = _factory("gmres", ref, [Iteration(24), ResidualNormReduction(1e-10)], krylov_dim=30).generate(a)
    s.apply(b, x)
    assert s.last_status.iterations <= 24
    oracle = np.linalg.solve(data.to_dense_array(), b.data[:, 0])
    assert np.linalg.norm(x.data[:, 0] - oracle) / np.linalg.norm(oracle) <= 1e-10


def test_gmres_restart_two_equals_full_on_2x2(ref):
    data = MatrixData(Dim2(2, 2), [0, 0, 1, 1], [0, 1, 0, 1], [3.0, 1.0, -1.0, 2.0])
    a1, b1, x1 = make_system(ref, data, seed=5)
    a2, b2, x2 = make_system(ref, data, seed=5)
    _factory("gmres", ref, [Iteration(2)], krylov_dim=2).generate(a1).apply(b1, x1)
    _factory("gmres", ref, [Iteration(2)], krylov_dim=50).generate(a2).apply(b2, x2)
    assert np.array_equal(x1.data, x2.data)


def test_gmres_restarted_matches_oracle(ref):
    dense = np.random.default_rng(6).standard_normal((100, 100)) + np.diag(np.full(100, 12.0))
    a, b, x = make_system(ref, MatrixData.from_dense_array(dense), seed=6)
    s = _factory("gmres", ref, [Iteration(3000), ResidualNormReduction(1e-12)], krylov_dim=10).generate(a)
    s.apply(b, x)
    assert s.last_status.converged
    oracle = np.linalg.solve(dense, b.data[:, 0])
    assert np.linalg.norm(x.data[:, 0] - oracle) / np.linalg.norm(oracle) <= 1e-8


def test_ir_with_exact_inner_converges_immediately(ref):
    data = random_spd(12, seed=7)
    a, b, x = make_system(ref, data, seed=7)
    s = opalg.Ir(ref, criteria=[Iteration(50), ResidualNormReduction(1e-12)],
                 inner=opalg.Jacobi(ref, block_size=12)).generate(a)
    s.apply(b, x)
    assert s.last_status.iterations == 1
    np.testing.assert_allclose(x.data[:, 0], np.linalg.solve(data.to_dense_array(), b.data[:, 0]), rtol=1e-10)


def test_ir_with_exact_inner_block_over_warp(ref):
    """As above with a single 40-row Jacobi block (the CTA-per-block path)."""
    data = random_spd(40, seed=7)
    a, b, x = make_system(ref, data, seed=7)
    s = opalg.Ir(ref, criteria=[Iteration(50), ResidualNormReduction(1e-12)],
                 inner=opalg.Jacobi(ref, block_size=40)).generate(a)
    s.apply(b, x)
    assert s.last_status.iterations == 1
    np.testing.assert_allclose(x.data[:, 0], np.linalg.solve(data.to_dense_array(), b.data[:, 0]), rtol=1e-10)


def test_ir_jacobi_sweep_geometric_decay(ref):
    data = random_sparse(30, density=0.15, seed=8)
    dense = data.to_dense_array()
    rho = max(abs(np.linalg.eigvals(np.eye(30) - np.diag(1.0 / np.diag(dense)) @ dense)))
    assert rho < 1
    a, b, x = make_system(ref, data, seed=8)
    norms = []

    class Probe(Criterion):
        def check(self, stopping_id, set_finalized, status, updater):
            if updater.residual is not None:
                norms.append(float(np.linalg.norm(np.asarray(updater.residual.data))))
            return False, False

    class ProbeFactory(CriterionFactory):
        def generate(self, args):
            return Probe()

    opalg.Ir(ref, criteria=[Iteration(20), ProbeFactory()], inner=opalg.Jacobi(ref)).generate(a).apply(b, x)
    measured = max(n2 / n1 for n1, n2 in zip(norms[2:], norms[3:]) if n1 > 0)
    assert measured < 1 and measured <= rho * 1.5


def test_ir_with_loose_cg_inner(ref):
    a, b, x = make_system(ref, random_spd(40, seed=9), seed=9)
    inner = opalg.Cg(ref, criteria=[Iteration(100), ResidualNormReduction(1e-2)])
    s = opalg.Ir(ref, criteria=[Iteration(200), ResidualNormReduction(1e-10)], inner=inner).generate(a)
    s.apply(b, x)
    assert s.last_status.converged
    first = s.last_status.iterations
    x2 = Dense.zeros(ref, 40, 1)
    s.apply(b, x2)
    assert s.last_status.iterations == first
    assert np.array_equal(x.data, x2.data)


def test_zero_rhs_zero_guess_stops_at_iteration_zero(ref):
    a = Csr.from_data(ref, tridiagonal(6))
    b, x = Dense.zeros(ref, 6, 1), Dense.zeros(ref, 6, 1)
    for name in ALL_KRYLOV:
        s = _factory(name, ref, [Iteration(50), ResidualNormReduction(1e-8)]).generate(a)
        s.apply(b, x)
        assert s.last_status.iterations == 0
        assert np.array_equal(x.data, np.zeros((6, 1)))


def test_cg_breakdown_reported_on_indefinite(ref):
    a = Csr.from_data(ref, MatrixData(Dim2(2, 2), [0, 1], [0, 1], [1.0, -1.0]))
    x = Dense.zeros(ref, 2, 1)
    s = _factory("cg", ref, [Iteration(10)]).generate(a)
    s.apply(Dense.vector(ref, [0.0, 1.0]), x)
    st_ = s.last_status
    assert st_.breakdown is not None and st_.breakdown.iteration == 1 and not st_.converged


def test_bicgstab_breakdown_reported_on_skew(ref):
    a = Csr.from_data(ref, MatrixData(Dim2(2, 2), [0, 1], [1, 0], [1.0, -1.0]))
    s = _factory("bicgstab", ref, [Iteration(10)]).generate(a)
    s.apply(Dense.vector(ref, [1.0, 0.0]), Dense.zeros(ref, 2, 1))
    assert s.last_status.breakdown is not None


@pytest.mark.parametrize("name", ALL_KRYLOV)
def test_nan_rhs_sustains_forced_iterations(ref, name):
    a = opalg.Coo.from_data(ref, MatrixData(Dim2(1, 1), [0], [0], [1.0]))
    s = _factory(name, ref, [Iteration(50)], **({"krylov_dim": 20} if name == "gmres" else {})).generate(a)
    s.apply(Dense(ref, [[float("nan")]]), Dense.zeros(ref, 1, 1))
    assert s.last_status.iterations == 50


def test_identity_precond_bitwise_equals_unpreconditioned(ref):
    data = random_spd(20, seed=10)
    a1, b1, x1 = make_system(ref, data, seed=10)
    a2, b2, x2 = make_system(ref, data, seed=10)
    plain = opalg.Cg(ref, criteria=[Iteration(30), ResidualNormReduction(1e-10)]).generate(a1)
    with_ident = opalg.Cg(ref, criteria=[Iteration(30), ResidualNormReduction(1e-10)],
                          generated_preconditioner=Identity(ref, 20)).generate(a2)
    plain.apply(b1, x1)
    with_ident.apply(b2, x2)
    assert plain.last_status.iterations == with_ident.last_status.iterations
    assert np.array_equal(x1.data, x2.data)


def test_per_column_freeze_bitwise(ref):
    data = random_spd(8, seed=11)
    dense = data.to_dense_array()
    a = Csr.from_data(ref, data)
    w, v = np.linalg.eigh(dense)
    b = np.stack([dense @ v[:, 0], np.ones(8)], axis=1)
    x = Dense(ref, np.zeros((8, 2)))
    snapshots = []

    class Freeze(Criterion):
        def check(self, stopping_id, set_finalized, status, updater):
            if status.data["stopped"][0] and not status.data["stopped"][1]:
                snapshots.append(np.array(updater.solution.data[:, 0]))
            return False, False

    class FreezeFactory(CriterionFactory):
        def generate(self, args):
            return Freeze()

    s = opalg.Cg(ref, criteria=[Iteration(60), ResidualNormReduction(1e-10), FreezeFactory()]).generate(a)
    s.apply(Dense(ref, b.copy()), x)
    assert s.last_status.stopped["stopped"].all()
    assert len(snapshots) > 1
    for snap in snapshots[1:]:
        assert np.array_equal(snap, snapshots[0])
    assert np.array_equal(np.asarray(x.data)[:, 0], snapshots[0])


class _ResidualAgreement(Criterion):
    def __init__(self, dense, b, even_only=False):
        super().__init__()
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


@pytest.mark.parametrize("name,tol", [("cg", 1e-6), ("fcg", 1e-6), ("cgs", 1e-6), ("bicgstab", 1e-6)])
def test_recurrence_residual_tracks_true_residual(ref, name, tol):
    data = random_spd(40, seed=12) if name in ("cg", "fcg") else random_sparse(40, density=0.2, seed=12)
    dense = data.to_dense_array()
    a, b, x = make_system(ref, data, seed=12)
    probe = _ResidualAgreement(dense, np.array(b.data[:, 0]), even_only=(name == "bicgstab"))

    class ProbeFactory(CriterionFactory):
        def generate(self, args):
            return probe

    _factory(name, ref, [Iteration(25), ProbeFactory()]).generate(a).apply(b, x)
    b_norm = np.linalg.norm(b.data)
    assert probe.rows
    for rec, true_r in probe.rows:
        if true_r is None or true_r <= 1e-8 * b_norm:
            continue
        assert abs(rec - true_r) <= tol * max(true_r, 1e-300)


def test_gmres_rotation_residual_matches_true_residual(ref):
    data = random_sparse(40, density=0.2, seed=12)
    dense = data.to_dense_array()
    for j in (1, 3, 7, 12, 20):
        a, b, x = make_system(ref, data, seed=12)
        estimates = {}

        class Probe(Criterion):
            def check(self, stopping_id, set_finalized, status, updater):
                estimates[updater.num_iterations] = float(updater.residual_norm[0])
                return False, False

        class ProbeFactory(CriterionFactory):
            def generate(self, args):
                return Probe()

        _factory("gmres", ref, [Iteration(j), ProbeFactory()], krylov_dim=50).generate(a).apply(b, x)
        true_r = np.linalg.norm(b.data[:, 0] - dense @ x.data[:, 0])
        if true_r > 1e-10 * np.linalg.norm(b.data):
            # + 1e-14 ||b||: near 1e-8 ||b|| the test's own evaluation of b - A x
            # carries ~eps ||A|| ||x|| of rounding (j = 20 differs by 4.6e-16)
            assert abs(estimates[j] - true_r) <= 1e-8 * true_r + 1e-14 * np.linalg.norm(b.data)


def test_lower_trs_hand_example(ref):
    factor = Csr.from_data(ref, MatrixData(Dim2(2, 2), [0, 1, 1], [0, 0, 1], [1.0, -0.5, 1.0]))
    y = Dense.zeros(ref, 2, 1)
    LowerTrs(ref, unit_diagonal=True).generate(factor).apply(Dense.vector(ref, [2.0, 1.0]), y)
    np.testing.assert_array_equal(y.data[:, 0], [2.0, 2.0])


def test_upper_trs_identity(ref):
    s = UpperTrs(ref).generate(Csr.from_data(ref, MatrixData(Dim2(3, 3), range(3), range(3), [1.0] * 3)))
    x = Dense.zeros(ref, 3, 1)
    s.apply(Dense.vector(ref, [4.0, 5.0, 6.0]), x)
    np.testing.assert_array_equal(x.data[:, 0], [4.0, 5.0, 6.0])


def _plain_lu(dense):
    n = dense.shape[0]
    lower, upper = np.eye(n), dense.astype(float).copy()
    for k in range(n - 1):
        for i in range(k + 1, n):
            f = upper[i, k] / upper[k, k]
            lower[i, k] = f
            upper[i, k:] -= f * upper[k, k:]
            upper[i, k] = 0.0
    return lower, upper


def test_lu_solve_composition_matches_dense(ref):
    n = 30
    dense = random_sparse(n, density=0.2, seed=13).to_dense_array()
    lower, upper = _plain_lu(dense)
    l_solver = LowerTrs(ref, unit_diagonal=True).generate(Csr.from_data(ref, MatrixData.from_dense_array(lower)))
    u_solver = UpperTrs(ref).generate(Csr.from_data(ref, MatrixData.from_dense_array(upper)))
    bvec = np.random.default_rng(13).standard_normal(n)
    x = Dense.zeros(ref, n, 1)
    compose(u_solver, l_solver).apply(Dense.vector(ref, bvec), x)
    oracle = np.linalg.solve(dense, bvec)
    assert np.linalg.norm(x.data[:, 0] - oracle) / np.linalg.norm(oracle) <= 1e-12


def test_parallel_triangular_level_scheduled_bitwise(ref, par):
    tri = MatrixData.from_dense_array(np.tril(random_sparse(60, density=0.15, seed=14).to_dense_array()))
    bvec = np.random.default_rng(14).standard_normal(60)
    s_ref = LowerTrs(ref).generate(Csr.from_data(ref, tri))
    s_par = LowerTrs(par).generate(Csr.from_data(par, tri))
    x_ref, x_par = Dense.zeros(ref, 60, 1), Dense.zeros(par, 60, 1)
    s_ref.apply(Dense.vector(ref, bvec), x_ref)
    s_par.apply(Dense.vector(par, bvec), x_par)
    assert np.array_equal(x_ref.data, x_par.data)
    assert len(s_par.levels) > 1


def test_singular_triangular_factor_rejected(ref):
    with pytest.raises(Singular):
        UpperTrs(ref).generate(Csr.from_data(ref, MatrixData(Dim2(2, 2), [0, 1], [0, 0], [1.0, 2.0])))
