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


def run(name):
    g, kind, solver, bs, kw = CASES[name]
    t0 = time.time()
    exc = opalg.ParallelExecutor(int(os.environ.get("GOLDEN_WORKERS", os.cpu_count())))
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
