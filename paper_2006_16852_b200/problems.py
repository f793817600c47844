"""Benchmark systems generated directly in HBM as canonical Csr.

Replaces the reference's host generators (src/problems.py:11-45) at device
scale: the C2/C5 systems (56M / 938M entries) never exist as host triples.
Formulas are documented in csrc/generate.cu and restated in
oracle/problems.py (the parity check).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .base import Dim2
from .executor import ptr
from .formats import Csr, _scan

STENCILS = {"5pt": 0, "7pt": 1, "27pt": 2, "convdiff": 3}


def stencil(exc, kind, grid, value_dtype="float64", convection=0.4, strategy="automatic"):
    """2-D 5-point (kind='5pt', grid^2 rows) or 3-D 7pt / 27pt / convdiff
    (grid^3 rows) stencil matrix as Csr on ``exc``."""
    code = STENCILS[kind]
    n = grid * grid if code == 0 else grid ** 3
    lens = torch.empty(max(n, 1), dtype=torch.int32, device=exc.device)
    _lib.call("stencil_lengths", code, grid, grid, 0, n, ptr(lens), exc.stream)
    rp = _scan(exc, lens[:n])
    nnz = int(rp[-1].item())
    vt = torch.float64 if np.dtype(value_dtype) == np.float64 else torch.float32
    ci = torch.empty(nnz, dtype=torch.int32, device=exc.device)
    v = torch.empty(nnz, dtype=vt, device=exc.device)
    _lib.call("stencil_fill_" + _lib.suffix(vt), code, grid, grid, float(convection), 0, n, ptr(rp), ptr(ci),
              ptr(v), exc.stream)
    return Csr._from_device(exc, Dim2(n, n), rp, ci, v, strategy=strategy)


# ---------------------------------------------------------------------------
# the reference's host generators (src/problems.py:11-58), same triples in the
# same (non-canonical) order, vectorised
# ---------------------------------------------------------------------------
def tridiagonal(n, lower=-1.0, diag=2.0, upper=-1.0):
    """MatrixData of tridiag(lower, diag, upper); per row: lower, diagonal,
    upper, zero off-diagonals omitted (src/problems.py:11-19)."""
    from .formats import MatrixData

    i = np.arange(n, dtype=np.int64)
    cols = np.stack([i - 1, i, i + 1], axis=1)
    vals = np.broadcast_to(np.array([lower, diag, upper], dtype=np.float64), (n, 3))
    keep = np.stack([(i > 0) & (lower != 0.0), np.ones(n, bool), (i < n - 1) & (upper != 0.0)], axis=1)
    rows = np.repeat(i, 3).reshape(n, 3)
    return MatrixData(Dim2(n, n), rows[keep], cols[keep], vals[keep])


def five_point_poisson(grid):
    """MatrixData of the 5-point Laplacian on a grid x grid mesh (diagonal 4,
    neighbours -1); per row: diagonal, then (-1,0), (1,0), (0,-1), (0,1)
    (src/problems.py:22-39)."""
    from .formats import MatrixData

    n = grid * grid
    me = np.arange(n, dtype=np.int64)
    i, j = me // grid, me % grid
    cols = np.stack([me, me - grid, me + grid, me - 1, me + 1], axis=1)
    vals = np.broadcast_to(np.array([4.0, -1.0, -1.0, -1.0, -1.0]), (n, 5))
    keep = np.stack([np.ones(n, bool), i > 0, i < grid - 1, j > 0, j < grid - 1], axis=1)
    rows = np.repeat(me, 5).reshape(n, 5)
    return MatrixData(Dim2(n, n), rows[keep], cols[keep], vals[keep])


def convection_diffusion(n, convection=0.4):
    """1-D convection-diffusion: tridiag(-1 - c, 2, -1 + c) (src/problems.py:42-45)."""
    return tridiagonal(n, lower=-1.0 - convection, diag=2.0, upper=-1.0 + convection)


def random_sparse(n, density=0.1, seed=0, diag_dominant=True):
    """Seeded random matrix with a full diagonal, optionally strictly
    diagonally dominant (src/problems.py:48-58)."""
    from .formats import MatrixData

    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, True)
    dense = np.where(mask, rng.uniform(-1.0, 1.0, (n, n)), 0.0)
    if diag_dominant:
        off = np.abs(dense).sum(axis=1) - np.abs(np.diag(dense))
        np.fill_diagonal(dense, off + 1.0)
    return MatrixData.from_dense_array(dense)


def random_spd(n, density=0.2, seed=0):
    """Seeded random sparse SPD matrix: symmetric pattern, diagonal made
    strictly dominant (src/problems.py:61-69)."""
    from .formats import MatrixData

    rng = np.random.default_rng(seed)
    mask = np.triu(rng.random((n, n)) < density / 2)
    dense = np.where(mask, rng.uniform(-1.0, 1.0, (n, n)), 0.0)
    dense = dense + dense.T
    off = np.abs(dense).sum(axis=1) - np.abs(np.diag(dense))
    np.fill_diagonal(dense, off + 1.0)
    return MatrixData.from_dense_array(dense)


def power_law(exc, n, seed=0, max_len=50000, c=5.5154, value_dtype="float64", strategy="automatic",
              lengths="hash"):
    """Synthetic power-law matrix (mean row length ~16 for c=5.5154, longest
    rows capped at max_len), columns and values generated on the device.

    Row lengths L = floor(c u^(-1/1.5)) clipped to [1, max_len]; ``lengths``
    picks u: "hash" (a counter hash, computed on the device) or "rng"
    (SURVEY.md 8(d)'s C3 recipe: u = 1 - numpy default_rng(seed).random(n),
    drawn on the host and uploaded, 4 bytes per row)."""
    if lengths == "rng":
        u = 1.0 - np.random.default_rng(seed).random(n)
        host = np.maximum(1, np.minimum(min(max_len, n), np.floor(c * u ** (-1.0 / 1.5)))).astype(np.int32)
        lens = torch.from_numpy(host).to(exc.device) if n else torch.empty(1, dtype=torch.int32, device=exc.device)
    else:
        thresholds = torch.from_numpy((c / np.arange(1, max_len + 1, dtype=np.float64)) ** 1.5).to(exc.device)
        lens = torch.empty(max(n, 1), dtype=torch.int32, device=exc.device)
        _lib.call("powerlaw_lengths", n, seed, ptr(thresholds), max_len, ptr(lens), exc.stream)
    rp = _scan(exc, lens[:n])
    nnz = int(rp[-1].item())
    vt = torch.float64 if np.dtype(value_dtype) == np.float64 else torch.float32
    ci = torch.empty(nnz, dtype=torch.int32, device=exc.device)
    v = torch.empty(nnz, dtype=vt, device=exc.device)
    _lib.call("powerlaw_fill_" + _lib.suffix(vt), n, seed, ptr(rp), ptr(ci), ptr(v), exc.stream)
    return Csr._from_device(exc, Dim2(n, n), rp, ci, v, strategy=strategy)
