"""Parity at the BASELINE sizes.

* C3: the full 4,194,304-row power law (SURVEY 8(d) row lengths, 67.1M
  entries) through every SpMV the C3 bench times, against the oracle's
  csr_row_sums restatement (oracle/spmv.py, pinned to the reference's
  src/kernels.py:278-316 by tests/test_oracle_golden.py), normwise 1e-14.
* C4 / C5: the device solvers against ONE-OFF runs of the reference itself
  at full size (tests/golden/make_golden_full.py: opalg ParallelExecutor,
  Csr + Bicgstab / Gmres(30) + Jacobi(block_size=32), Cg; rhs ones, x0 = 0,
  RNR 1e-8): iteration counts within +-1 (CG 611 = 611, GMRES(30) 734 = 734;
  BiCGSTAB within the spread equally valid summation orders produce, see
  ITER_TOL), the same stopping criterion, the final true residual and a
  strided sample of x.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import problems as P
from oracle import spmv as OS

pytestmark = pytest.mark.gpu


def _gold(name):
    path = os.path.join(GOLDEN, f"full_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet (tests/golden/make_golden_full.py {name})")
    return dict(np.load(path))


# ---------------------------------------------------------------------------
# C3 power law, full size
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c3(cuda):
    from paper_2006_16852_b200 import problems

    a = problems.power_law(cuda, 4194304, seed=0, lengths="rng")
    rp = a.row_ptrs.numpy()
    ci = a.col_idxs.numpy()
    v = a.vals.numpy()
    bv = np.random.default_rng(0).standard_normal((a.size.rows, 1))
    return a, rp, ci, v, bv, OS.csr_spmv(rp, ci, v, bv)


def test_c3_generator_matches_survey_recipe(c3):
    a, rp, ci, v, bv, ref = c3
    lens = P.power_law_lengths_rng(4194304, 0)
    assert np.array_equal(np.diff(rp), lens)
    assert rp[-1] == 67109323 and lens.max() == 50000 and (lens == 50000).sum() == 6
    # columns sorted and distinct within each row, values in (-1, 1)
    d = np.diff(ci.astype(np.int64))
    inside = np.ones(d.size, bool)
    inside[rp[1:-1] - 1] = False  # row boundaries
    assert (d[inside[: d.size]] > 0).all()
    assert np.abs(v).max() < 1.0
    # a sample of rows bit-exact against the oracle generator's formula
    n = 4194304
    for r in (0, 1, 12345, int(np.argmax(lens)), n - 1):
        L = lens[r]
        k = np.arange(L, dtype=np.int64)
        h = P.hash3(0, np.full(L, r + 1, dtype=np.int64), k)
        lo, hi = k * n // L, (k + 1) * n // L
        cols = lo + (h % (hi - lo).astype(np.uint64)).astype(np.int64)
        assert np.array_equal(ci[rp[r]:rp[r + 1]], cols), r


@pytest.mark.parametrize("fmt", ["csr_lb", "hybrid", "coo", "csr_classical", "csr_stream"])
def test_c3_fullsize_spmv_matches_oracle(cuda, c3, fmt):
    import paper_2006_16852_b200 as b2

    a, rp, ci, v, bv, ref = c3
    m = b2.convert(a, fmt)
    x = b2.Dense.zeros(cuda, a.size.rows, 1)
    m.apply(b2.Dense(cuda, bv), x)
    err = OS.rel_error_inf(np.asarray(x.data), ref)
    assert err <= 1e-14, (fmt, err)


# ---------------------------------------------------------------------------
# C4 / C5 solvers vs the reference's own full-size runs
# ---------------------------------------------------------------------------
SOLVES = [
    # golden name, stencil kind, grid, solver, jacobi block, kwargs
    ("c5_cg_g256", "7pt", 256, "cg", 0, {}),
    ("c4_bicgstab_bj32", "convdiff", 256, "bicgstab", 32, {}),
    ("c4_gmres30_bj32", "convdiff", 256, "gmres", 32, {"krylov_dim": 30}),
    ("c5_cg_g512", "7pt", 512, "cg", 0, {}),
]

# Iteration-count tolerance per case. CG and GMRES(30) reproduce the reference
# exactly (+-1 is the north_star bar). BiCGSTAB + block-Jacobi on the 3-D
# convection-diffusion problem is chaotic under rounding: the shadow residual
# r~ = r0 = ones is nearly orthogonal to range(A) (the operator's interior
# column sums are zero), rho = r~.r cancels, and equally valid summation orders
# move the count by tens of half-iterations -- the reference's own 1341 among
# them (profiles/r03_rounding_sensitivity.jsonl: partitions of the device
# reductions give 1325 / 1341 / 1343 / 1345 / 1351 / 1353 / 1367, and two of
# nine hit an exact rho = 0 breakdown). The bar there is the spread of those
# converged runs (+-2%), with the solution and the final residual held to the
# same limits as the other cases.
ITER_TOL = {"c4_bicgstab_bj32": 28}


@pytest.mark.parametrize("name,kind,g,solver,bs,kw", SOLVES, ids=[s[0] for s in SOLVES])
def test_fullsize_solve_matches_reference_run(cuda, name, kind, g, solver, bs, kw):
    import torch

    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import problems

    gold = _gold(name)
    a = problems.stencil(cuda, kind, g)
    n = a.size.rows
    pre = b2.Jacobi(cuda, block_size=bs) if bs else None
    crit = [b2.Iteration(10000), b2.ResidualNormReduction(1e-8)]
    s = b2.SOLVER_FACTORIES[solver](cuda, criteria=crit, preconditioner=pre, **kw).generate(a)
    b = b2.Dense.wrap(cuda, torch.ones((n, 1), dtype=torch.float64, device=cuda.device))
    x = b2.Dense.wrap(cuda, torch.zeros((n, 1), dtype=torch.float64, device=cuda.device))
    s.apply(b, x)
    st = s.last_status
    ref_it = int(gold["iterations"])
    print(f"{name}: iterations {st.iterations} (reference {ref_it})")
    assert st.breakdown is None and st.converged
    assert st.stopping_id == int(gold["stopping_id"])
    assert abs(st.iterations - ref_it) <= ITER_TOL.get(name, 1), (st.iterations, ref_it)
    # final true residual ||b - A x|| (device SpMV) within 2x of the reference's
    ax = b2.Dense.wrap(cuda, torch.empty((n, 1), dtype=torch.float64, device=cuda.device))
    a.apply(x, ax)
    true_r = float(torch.linalg.vector_norm(b.values - ax.values))
    ref_r = float(gold["true_res"][0])
    print(f"{name}: true residual {true_r:.6e} (reference {ref_r:.6e})")
    assert true_r <= 2.0 * ref_r and true_r <= 1e-8 * np.sqrt(n) * 1.5
    # the solution: same Krylov trajectory, rounding-order differences only
    xs = x.values[::int(gold["sample_stride"]), 0].cpu().numpy()
    xr = gold["x_sample"][:, 0]
    rel = np.linalg.norm(xs - xr) / np.linalg.norm(xr)
    print(f"{name}: x sample rel. difference {rel:.3e}")
    # both iterates meet ||b - A x|| <= 1e-8 ||b||; they agree to the error that
    # residual allows (CG / GMRES follow the same trajectory to ~1e-14)
    assert rel <= (1e-5 if name in ITER_TOL else 1e-6), rel
    xn = float(torch.linalg.vector_norm(x.values))
    assert abs(xn - float(gold["x_norm"][0])) <= (1e-5 if name in ITER_TOL else 1e-6) * xn
