"""SpMV oracles (NumPy). TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates, on plain arrays:
  csr_spmv   -- CsrSpmvKernel + csr_row_sums, reference src/kernels.py:278-316:
                per row, products vals[k]*b[col[k]] (separate multiply), summed
                with np.add.reduceat over each row's segment (first element then
                NumPy's pairwise tail); empty rows are 0.
  coo_spmv   -- CooSpmvKernel, src/kernels.py:163-199: x = 0, then unbuffered
                scatter-add (np.add.at) in entry order.
  coo_adv    -- CooAdvSpmvKernel, src/kernels.py:202-240: x = beta x, then
                np.add.at of alpha * (vals * b[cols]).
  residual   -- CooResidualKernel, src/kernels.py:243-275: r = b, then
                np.subtract.at of the products.
  dense_spmv -- DenseSpmvKernel, src/kernels.py:319-332 (np.matmul).
Formats without a reference kernel (Ell/Sellp/Hybrid) are checked through the
format-independent result of csr_spmv (north_star tolerance 1e-14 / 1e-6).
"""

from __future__ import annotations

import numpy as np


def csr_spmv(row_ptrs, col_idxs, vals, b):
    """x = A b for (n, m) b; reduceat summation order of src/kernels.py:304-316."""
    rp = np.asarray(row_ptrs, dtype=np.int64)
    n = rp.size - 1
    b = np.asarray(b)
    if b.ndim == 1:
        b = b[:, None]
    out = np.zeros((n, b.shape[1]), dtype=b.dtype)
    if rp[-1] == 0:
        return out
    prod = np.asarray(vals)[:, None] * b[np.asarray(col_idxs)]
    lens = np.diff(rp)
    rows = np.flatnonzero(lens > 0)
    out[rows] = np.add.reduceat(prod, rp[rows].astype(np.intp), axis=0)
    return out


def coo_spmv(row_idxs, col_idxs, vals, b, n):
    b = np.asarray(b)
    if b.ndim == 1:
        b = b[:, None]
    out = np.zeros((n, b.shape[1]), dtype=b.dtype)
    if len(vals):
        prod = np.asarray(vals)[:, None] * b[np.asarray(col_idxs)]
        np.add.at(out, np.asarray(row_idxs, dtype=np.intp), prod)
    return out


def coo_adv(row_idxs, col_idxs, vals, alpha, b, beta, x):
    out = np.multiply(x, beta)
    if len(vals):
        prod = alpha * (np.asarray(vals)[:, None] * b[np.asarray(col_idxs)])
        np.add.at(out, np.asarray(row_idxs, dtype=np.intp), prod)
    return out


def residual(row_idxs, col_idxs, vals, x, b):
    r = np.array(b, copy=True)
    if len(vals):
        prod = np.asarray(vals)[:, None] * x[np.asarray(col_idxs)]
        np.subtract.at(r, np.asarray(row_idxs, dtype=np.intp), prod)
    return r


def dense_spmv(a, b):
    return np.matmul(a, b)


def csr_from_triples(n, rows, cols, vals):
    """Row pointers of canonical triples (src/formats.py:196-203 builds them
    with np.add.at(rows + 1) and cumsum)."""
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, np.asarray(rows, dtype=np.int64) + 1, 1)
    np.cumsum(rp, out=rp)
    return rp


def rel_error_inf(x, ref):
    """Normwise infinity relative error (tests/test_formats.py:164-169)."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = max(float(np.abs(ref).max(initial=0.0)), 1e-300)
    return float(np.abs(x - ref).max(initial=0.0)) / scale
