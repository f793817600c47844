"""Benchmark-system generators (NumPy). TEST INFRASTRUCTURE ONLY.

Vectorised restatements producing canonical (row, col)-sorted triples:
  five_point(g)       == reference five_point_poisson(g) after canonicalize
                         (src/problems.py:22-39); pinned by tests/golden.
  stencil3d(g, kind)  3-D 7-point Poisson (centre 6, neighbours -1), 27-point
                      (centre 26, neighbours -1), 7-point convection-diffusion
                      (neighbour at offset -1 / +1 along an axis: -1-c / -1+c,
                      the 3-D extension of convection_diffusion,
                      src/problems.py:42-45; pinned at g=1-D analogue).
  power_law(n, ...)   hash-based generator (no reference counterpart): row
                      length from thresholds t_k=(c/k)^1.5, stratified distinct
                      sorted columns, values U(-1,1). Same formulas as
                      paper_2006_16852_b200/csrc/generate.cu.
Grid index is idx = (i*g + j)*g + k with Dirichlet truncation.
"""

from __future__ import annotations

import numpy as np

_U = np.uint64


def _mix64(z):
    z = (z + _U(0x9E3779B97F4A7C15))
    z = (z ^ (z >> _U(30))) * _U(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> _U(27))) * _U(0x94D049BB133111EB)
    return z ^ (z >> _U(31))


def hash3(seed, a, b):
    with np.errstate(over="ignore"):
        s = _mix64(np.asarray(seed, dtype=_U))
        return _mix64(_mix64(s ^ (np.asarray(a, dtype=_U) * _U(0xD1B54A32D192ED03)))
                      + np.asarray(b, dtype=_U))


def unit(h):
    return (np.asarray(h, dtype=_U) >> _U(11)).astype(np.float64) * 2.0 ** -53


def five_point(g):
    """Canonical triples of the 2-D 5-point Laplacian on a g x g grid."""
    n = g * g
    idx = np.arange(n, dtype=np.int64)
    i, j = idx // g, idx % g
    parts = []  # (mask, col offset, value) in canonical column order
    for m, off, val in ((i > 0, -g, -1.0), (j > 0, -1, -1.0), (np.ones(n, bool), 0, 4.0),
                        (j < g - 1, 1, -1.0), (i < g - 1, g, -1.0)):
        parts.append((idx[m], idx[m] + off, np.full(int(m.sum()), val)))
    return _merge(n, parts)


def stencil3d(g, kind, conv=0.4, nz=None):
    """kind: '7pt' | '27pt' | 'convdiff'; nz planes of g x g along the
    slowest axis (default g: the cube)."""
    nz = g if nz is None else nz
    n = g * g * nz
    idx = np.arange(n, dtype=np.int64)
    i, j, k = idx // (g * g), (idx // g) % g, idx % g
    parts = []
    if kind == "27pt":
        for di in (-1, 0, 1):
            for dj in (-1, 0, 1):
                for dk in (-1, 0, 1):
                    m = ((i + di >= 0) & (i + di < nz) & (j + dj >= 0) & (j + dj < g)
                         & (k + dk >= 0) & (k + dk < g))
                    val = 26.0 if (di, dj, dk) == (0, 0, 0) else -1.0
                    parts.append((idx[m], idx[m] + (di * g + dj) * g + dk, np.full(int(m.sum()), val)))
        return _merge(n, parts)
    lo = -1.0 - conv if kind == "convdiff" else -1.0
    hi = -1.0 + conv if kind == "convdiff" else -1.0
    for m, off, val in ((i > 0, -g * g, lo), (j > 0, -g, lo), (k > 0, -1, lo),
                        (np.ones(n, bool), 0, 6.0),
                        (k < g - 1, 1, hi), (j < g - 1, g, hi), (i < nz - 1, g * g, hi)):
        parts.append((idx[m], idx[m] + off, np.full(int(m.sum()), val)))
    return _merge(n, parts)


def _merge(n, parts):
    """Interleave per-offset parts into canonical row-major order (parts are
    given in increasing column-offset order, so a stable sort by row keeps the
    columns sorted)."""
    rows = np.concatenate([p[0] for p in parts])
    cols = np.concatenate([p[1] for p in parts])
    vals = np.concatenate([p[2] for p in parts])
    order = np.argsort(rows, kind="stable")
    return n, rows[order], cols[order], vals[order]


def power_law_thresholds(max_len=50000, c=5.5154):
    return (c / np.arange(1, max_len + 1, dtype=np.float64)) ** 1.5


def power_law_lengths(n, seed=0, max_len=50000, c=5.5154):
    t = power_law_thresholds(max_len, c)
    u = 1.0 - unit(hash3(seed, 0, np.arange(n, dtype=np.int64)))
    lens = np.searchsorted(-t, -u, side="right")  # count of t_k >= u (t decreasing)
    return np.clip(lens, 1, n).astype(np.int64)


def power_law_lengths_rng(n, seed=0, max_len=50000, c=5.5154):
    """SURVEY.md 8(d) C3 row lengths verbatim: u = 1 - default_rng(seed).random(n),
    L = max(1, min(max_len, floor(c * u^(-1/1.5)))). At n = 4,194,304, seed 0:
    nnz 67,109,323, mean 16.0001, median 8, max 50,000 (6 rows at the cap)."""
    u = 1.0 - np.random.default_rng(seed).random(n)
    return np.maximum(1, np.minimum(min(max_len, n), np.floor(c * u ** (-1.0 / 1.5)))).astype(np.int64)


def power_law(n, seed=0, max_len=50000, c=5.5154, lengths="hash"):
    """lengths: 'hash' (counter-hash u, this repo's original generator) or
    'rng' (numpy default_rng(seed)). Columns: row i's L entries
    are distinct and sorted, entry k uniform in its own stratum
    [k n / L, (k+1) n / L); values U(-1, 1) from the same counter hash."""
    lens = (power_law_lengths_rng if lengths == "rng" else power_law_lengths)(n, seed, max_len, c)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    rows = np.repeat(np.arange(n, dtype=np.int64), lens)
    k = np.arange(rp[-1], dtype=np.int64) - np.repeat(rp[:-1], lens)
    L = lens[rows]
    lo = k * n // L
    hi = (k + 1) * n // L
    h = hash3(seed, rows + 1, k)
    cols = lo + (h % (hi - lo).astype(_U)).astype(np.int64)
    with np.errstate(over="ignore"):
        vals = 2.0 * unit(_mix64(h ^ _U(0x5851F42D4C957F2D))) - 1.0
    return n, rows, cols, vals


def to_csr(n, rows, cols, vals):
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    return rp, np.asarray(cols, dtype=np.int64), np.asarray(vals, dtype=np.float64)
