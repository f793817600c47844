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
    _lib.call("stencil_lengths", code, grid, 0, n, ptr(lens), exc.stream)
    rp = _scan(exc, lens[:n])
    nnz = int(rp[-1].item())
    vt = torch.float64 if np.dtype(value_dtype) == np.float64 else torch.float32
    ci = torch.empty(nnz, dtype=torch.int32, device=exc.device)
    v = torch.empty(nnz, dtype=vt, device=exc.device)
    _lib.call("stencil_fill_" + _lib.suffix(vt), code, grid, float(convection), 0, n, ptr(rp), ptr(ci),
              ptr(v), exc.stream)
    return Csr._from_device(exc, Dim2(n, n), rp, ci, v, strategy=strategy)


def five_point_poisson(exc, grid, **kw):
    return stencil(exc, "5pt", grid, **kw)


def power_law(exc, n, seed=0, max_len=50000, c=5.5154, value_dtype="float64", strategy="automatic"):
    """Synthetic power-law matrix (mean row length ~16 for c=5.5154, longest
    rows capped at max_len), generated on the device."""
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
