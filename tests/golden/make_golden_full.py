"""One-off REFERENCE runs at the BASELINE sizes (C4 256^3, C5 256^3 / 512^3).

Run in the build container (where /root/reference exists), one case per call
so the cases can run side by side:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_full.py c4_bicgstab_bj32
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_full.py c4_gmres30_bj32
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_full.py c5_cg_g256
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_full.py c5_cg_g512

Each writes tests/golden/full_<case>.npz: iteration count, stopping id, the
residual-norm history the reference's criteria saw, the final true residual
norm, ||x|| and a strided sample of x (the full x is 134 MB / 1 GB and does not
belong in the repo).

The reference (`opalg`, pure Python + NumPy) is imported read-only from
/root/reference/pkg/src and driven through its public API only:
`Csr.from_data` -> `Bicgstab/Gmres/Cg(exc, criteria=[Iteration, RNR],
preconditioner=Jacobi(exc, block_size=32))` -> `apply` (reference
src/solvers/krylov.py:36-77, :190-271, src/solvers/gmres.py:183-340,
src/precond.py:155-208). Executor: `ParallelExecutor` (src/executor.py:166-215),
the reference's multi-threaded CPU path; its SpMV is bitwise the
ReferenceExecutor's (rows are independent) and its dots are blocked partial
sums combined in block order. The matrices are the oracle generators'
(oracle/problems.py, bit-exact with the device generators) because the
reference has no 3-D generator; rhs = ones, x0 = 0 (src/bench.py:105-107).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import opalg  # noqa: E402  (the reference)
from opalg import (Bicgstab, Cg, Csr, Dense, Dim2, Gmres, Iteration, Jacobi,  # noqa: E402
                   MatrixData, ResidualNormReduction)
from opalg.stop import Criterion, CriterionFactory  # noqa: E402

from oracle import problems as P  # noqa: E402

SAMPLE_STRIDE = 4099

CASES = {
    # name: (grid, stencil kind, solver, jacobi block size, solver kwargs)
    "c4_bicgstab_bj32": (256, "convdiff", "bicgstab", 32, {}),
    "c4_gmres30_bj32": (256, "convdiff", "gmres", 32, {"krylov_dim": 30}),
    "c5_cg_g256": (256, "7pt", "cg", 0, {}),
    "c5_cg_g512": (512, "7pt", "cg", 0, {}),
}


class _History(Criterion):
    def __init__(self, sink, t0):
        super().__init__()
        self.sink = sink
        self.t0 = t0

    def check(self, stopping_id, set_finalized, status, updater):
        if updater.residual_norm is not None:
            self.sink.append(np.asarray(updater.residual_norm, dtype=float).copy())
        elif updater.residual is not None:
            r = updater.residual.data
            self.sink.append(np.sqrt(np.einsum("ij,ij->j", r, r)))
        k = len(self.sink)
        if k % 25 == 0:
            print(f"    check {k}: |r| = {self.sink[-1][0]:.6e}  "
                  f"({time.time() - self.t0:.0f} s)", flush=True)
        return False, False


class _HistoryFactory(CriterionFactory):
    def __init__(self, t0):
        self.rows = []
        self.t0 = t0

    def generate(self, args):
        self.rows = []
        return _History(self.rows, self.t0)


def csr_7pt(g):
    """The 7-point Poisson CSR (canonical order, int32 indices) built plane by
    plane -- the same matrix as oracle/problems.stencil3d(g, "7pt") without the
    22.5 GB of int64 triples MatrixData would hold at 512^3."""
    n = g ** 3
    p2 = g * g
    jj, kk = np.divmod(np.arange(p2, dtype=np.int64), g)
    rp = np.zeros(n + 1, dtype=np.int64)
    for i in range(g):
        lens = (1 + (i > 0) + (i < g - 1) + (jj > 0) + (jj < g - 1) + (kk > 0) + (kk < g - 1)).astype(np.int64)
        np.cumsum(lens, out=rp[i * p2 + 1:(i + 1) * p2 + 1])
        rp[i * p2 + 1:(i + 1) * p2 + 1] += rp[i * p2]
    nnz = int(rp[-1])
    ci = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64)
    offs = np.array([-p2, -g, -1, 0, 1, g, p2], dtype=np.int64)
    cvals = np.array([-1.0, -1.0, -1.0, 6.0, -1.0, -1.0, -1.0])
    for i in range(g):
        rows = i * p2 + np.arange(p2, dtype=np.int64)
        keep = np.stack([np.full(p2, i > 0), jj > 0, kk > 0, np.ones(p2, bool), kk < g - 1, jj < g - 1,
                         np.full(p2, i < g - 1)], axis=1)
        cols = rows[:, None] + offs[None, :]
        lo, hi = rp[i * p2], rp[(i + 1) * p2]
        ci[lo:hi] = cols[keep]
        vals[lo:hi] = np.broadcast_to(cvals, (p2, 7))[keep]
    return rp.astype(np.int32), ci, vals


def run(name):
    g, kind, solver, bs, kw = CASES[name]
    t0 = time.time()
    exc = opalg.ParallelExecutor(int(os.environ.get("GOLDEN_WORKERS", os.cpu_count())))
    if kind == "7pt" and g >= 512:  # lean build (the reference's own Csr constructor)
        rp8, ci8, v8 = csr_7pt(8)
        n8, r8, c8, vv8 = P.stencil3d(8, "7pt")
        rpo, cio, vo = P.to_csr(n8, r8, c8, vv8)
        assert np.array_equal(rp8, rpo) and np.array_equal(ci8, cio) and np.array_equal(v8, vo)
        rp, ci, vals = csr_7pt(g)
        n = g ** 3
        a = Csr(exc, Dim2(n, n), rp, ci, vals)
        del rp, ci, vals
    else:
        n, r, c, v = P.stencil3d(g, kind)
        data = MatrixData(Dim2(n, n), r, c, v)
        del r, c, v
        a = Csr.from_data(exc, data)
        del data
    print(f"{name}: n={n} nnz={a.col_idxs.size} matrix ready ({time.time() - t0:.0f} s)", flush=True)
    hist = _HistoryFactory(t0)
    crits = [Iteration(10000), ResidualNormReduction(1e-8), hist]
    fac = {"cg": Cg, "bicgstab": Bicgstab, "gmres": Gmres}[solver]
    if bs:
        kw = dict(kw, preconditioner=Jacobi(exc, block_size=bs))
    s = fac(exc, criteria=crits, **kw).generate(a)
    print(f"{name}: solver generated ({time.time() - t0:.0f} s)", flush=True)
    b = Dense(exc, np.ones((n, 1)))
    x = Dense.zeros(exc, n, 1)
    s.apply(b, x)
    st = s.last_status
    ax = Dense.zeros(exc, n, 1)
    a.apply(x, ax)
    true_r = np.linalg.norm(b.data - ax.data, axis=0)
    rec = {
        "n": np.array(n),
        "iterations": np.array(st.iterations),
        "stopping_id": np.array(st.stopping_id),
        "breakdown": np.array(st.breakdown is not None),
        "history": np.array(hist.rows),
        "true_res": true_r,
        "x_norm": np.linalg.norm(x.data, axis=0),
        "x_sample": x.data[::SAMPLE_STRIDE].copy(),
        "sample_stride": np.array(SAMPLE_STRIDE),
        "seconds": np.array(time.time() - t0),
        "executor": np.array(repr(exc)),
    }
    print(f"{name}: iterations={st.iterations} stop_id={st.stopping_id} "
          f"breakdown={st.breakdown} true_res={true_r} ({time.time() - t0:.0f} s)", flush=True)
    path = os.path.join(HERE, f"full_{name}.npz")
    np.savez_compressed(path, **rec)
    print(f"wrote {path}", flush=True)


if __name__ == "__main__":
    for case in sys.argv[1:]:
        run(case)
