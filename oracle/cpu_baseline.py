"""CPU baseline = the reference's CPU path restated (TEST/BENCH INFRASTRUCTURE).

The reference's fastest CPU execution of Csr SpMV is ParallelExecutor
(src/executor.py:166-215): contiguous row blocks (np.linspace partition,
:181-184) over a thread pool, each block running csr_row_sums
(src/kernels.py:304-316). This module restates that with the oracle's
csr_spmv per block; bench.py times it on the GPU box's host cores as the
`cpu_baseline` and as the `--impl reference` arm. It is never used by the
product package.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np



def csr_row_sums(vals, col_idxs, row_ptrs, b, lo, hi):
    """src/kernels.py:304-316 restated statement by statement (the same NumPy
    calls on the same dtypes: int32 row pointers and indices)."""
    e0, e1 = int(row_ptrs[lo]), int(row_ptrs[hi])
    out = np.zeros((hi - lo, b.shape[1]), dtype=b.dtype)
    if e0 == e1:
        return out
    prod = vals[e0:e1, None] * b[col_idxs[e0:e1]]
    counts = np.diff(row_ptrs[lo:hi + 1])
    nonempty = np.flatnonzero(counts > 0)
    starts = row_ptrs[lo + nonempty] - e0
    out[nonempty] = np.add.reduceat(prod, starts.astype(np.intp), axis=0)
    return out


class ParallelCsr:
    """ParallelExecutor.map_blocks (src/executor.py:181-200) around
    CsrSpmvKernel._run (src/kernels.py:285-293): `x[lo:hi] = csr_row_sums(...)`
    per contiguous row block on a thread pool of os.cpu_count() workers."""

    def __init__(self, rp, ci, vals, workers=None):
        self.rp = np.asarray(rp, dtype=np.int32)  # config.DEFAULT_INDEX_DTYPE
        self.ci = np.asarray(ci, dtype=np.int32)
        self.vals = np.asarray(vals)
        self.n = self.rp.size - 1
        self.workers = workers or os.cpu_count() or 1
        w = min(self.workers, max(self.n, 1))
        b = np.linspace(0, self.n, w + 1).astype(np.int64)
        self.blocks = [(int(b[i]), int(b[i + 1])) for i in range(w) if b[i] < b[i + 1]]
        self.pool = ThreadPoolExecutor(max_workers=len(self.blocks)) if len(self.blocks) > 1 else None

    def _block(self, lo, hi, b, out):
        out[lo:hi] = csr_row_sums(self.vals, self.ci, self.rp, b, lo, hi)

    def apply(self, b, out):
        if self.pool is None:
            self._block(0, self.n, b, out)
        else:
            list(self.pool.map(lambda blk: self._block(blk[0], blk[1], b, out), self.blocks))
        return out

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


def time_csr_spmv(rp, ci, vals, b, reps=5, warmup=1, workers=None):
    """Median seconds per SpMV (run_profile style: warm-up then median,
    src/bench.py:222-228)."""
    op = ParallelCsr(rp, ci, vals, workers)
    out = np.empty((op.n, b.shape[1]), dtype=b.dtype)
    for _ in range(warmup):
        op.apply(b, out)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        op.apply(b, out)
        ts.append(time.perf_counter() - t0)
    op.close()
    return float(np.median(ts)), len(op.blocks), ts
