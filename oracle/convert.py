"""Format-conversion oracles (NumPy). TEST INFRASTRUCTURE ONLY.

The reference has no Ell/Sellp/Hybrid and converts its own
formats through canonical MatrixData (src/formats.py:301-322); these
functions are the specification of the device layouts (see
paper_2006_16852_b200/csrc/convert.cu) and are compared bit-for-bit with the
device conversions. Inputs are canonical Csr arrays (sorted columns).
"""

from __future__ import annotations

import math

import numpy as np


def row_lengths(rp):
    return np.diff(np.asarray(rp, dtype=np.int64))


def ell_stride(n):
    return max(1, (n + 31) // 32 * 32)


def csr_to_ell(rp, ci, v, width=None, stride=None):
    """Column-major ELL; element (row, k) at k*stride + row; pad col -1, val 0."""
    rp = np.asarray(rp, dtype=np.int64)
    n = rp.size - 1
    lens = row_lengths(rp)
    w = int(lens.max(initial=0)) if width is None else int(width)
    st = ell_stride(n) if stride is None else int(stride)
    eci = np.full(w * st, -1, dtype=np.int32)
    ev = np.zeros(w * st, dtype=np.asarray(v).dtype)
    rows = np.repeat(np.arange(n), lens)
    k = np.arange(rp[-1]) - np.repeat(rp[:-1], lens)
    keep = k < w
    slot = k[keep] * st + rows[keep]
    eci[slot] = np.asarray(ci)[keep]
    ev[slot] = np.asarray(v)[keep]
    return eci, ev, w, st


def csr_to_sellp(rp, ci, v, slice_size=64, stride_factor=1):
    rp = np.asarray(rp, dtype=np.int64)
    n = rp.size - 1
    lens = row_lengths(rp)
    ns = math.ceil(n / slice_size)
    padded = np.zeros(ns * slice_size, dtype=np.int64)
    padded[:n] = lens
    sl = padded.reshape(ns, slice_size).max(axis=1) if ns else np.zeros(0, np.int64)
    sl = (sl + stride_factor - 1) // stride_factor * stride_factor
    ss = np.zeros(ns + 1, dtype=np.int64)
    np.cumsum(sl, out=ss[1:])
    total = int(ss[-1])
    sci = np.full(total * slice_size, -1, dtype=np.int32)
    sv = np.zeros(total * slice_size, dtype=np.asarray(v).dtype)
    rows = np.repeat(np.arange(n), lens)
    k = np.arange(rp[-1]) - np.repeat(rp[:-1], lens)
    s = rows // slice_size
    slot = (ss[s] + k) * slice_size + rows % slice_size
    sci[slot] = np.asarray(ci)
    sv[slot] = np.asarray(v)
    return sl.astype(np.int32), ss.astype(np.int32), sci, sv


def csr_to_hybrid(rp, ci, v, width):
    """First `width` entries of each row in Ell, the rest (row-major) in Coo."""
    rp = np.asarray(rp, dtype=np.int64)
    n = rp.size - 1
    eci, ev, w, st = csr_to_ell(rp, ci, v, width=width)
    lens = row_lengths(rp)
    rows = np.repeat(np.arange(n), lens)
    k = np.arange(rp[-1]) - np.repeat(rp[:-1], lens)
    over = k >= width
    return (eci, ev, w, st), (rows[over].astype(np.int32), np.asarray(ci)[over].astype(np.int32),
                              np.asarray(v)[over])


def length_histogram(rp, nbins):
    lens = np.minimum(row_lengths(rp), nbins - 1)
    return np.bincount(lens, minlength=nbins).astype(np.float64)


def hybrid_width_imbalance(rp, percent=0.8):
    lens = np.sort(row_lengths(rp))
    if lens.size == 0:
        return 0
    return int(lens[min(lens.size - 1, int(math.floor(percent * lens.size)))])


def hybrid_width_minimal_storage(rp, vt_bytes):
    lens = row_lengths(rp)
    n = lens.size
    if n == 0:
        return 0
    best_w, best = 0, None
    for w in range(int(lens.max(initial=0)) + 1):
        cost = n * w * (vt_bytes + 4) + float(np.maximum(lens - w, 0).sum()) * (vt_bytes + 8)
        if best is None or cost < best:
            best, best_w = cost, w
    return best_w
