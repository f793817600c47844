"""Direct sparse triangular solvers (reference src/solvers/triangular.py:18-155).

The reference substitutes row by row (or level by level across workers).
Here a synchronisation-free kernel (csrc/ilu.cu: trs_kernel) solves every
column in one launch: warps claim rows through an atomic ticket in the order
of their dependency levels (computed on the device at generation: claiming
in plain row order serialised a stencil factor along its x-neighbour chain,
143 ms vs 4.3 ms per ILU apply at 128^3), wait on the rows they depend on
with acquire loads of per-row flags, and publish their x_i with a release
store. Generation extracts the diagonal
on the device and raises Singular on a zero (or missing) one, like the
reference; ``levels`` (the reference's dependency levels) is computed on
demand for inspection only.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _lib
from ..base import LinOp, LinOpFactory
from ..errors import DimensionMismatch, Singular
from ..executor import ptr
from ..formats import Csr, _require_cuda, _scan

INT_MAX = 2 ** 31 - 1


def extract_diagonal(factor):
    """Device diagonal of a Csr; Singular names the first zero/missing row."""
    exc = factor.exec
    n = factor.size.rows
    diag = torch.empty(max(n, 1), dtype=factor._v.dtype, device=exc.device)
    zero = torch.full((1,), INT_MAX, dtype=torch.int32, device=exc.device)
    _lib.call("diag_" + _lib.suffix(factor._v.dtype), n, ptr(factor._rp), ptr(factor._ci), ptr(factor._v),
              ptr(diag), ptr(zero), exc.stream)
    return diag[:n], int(zero.item())


class TriangularSolver(LinOp):
    """Exact substitution with a (unit-)triangular Csr factor."""

    #: level-synchronous cooperative substitution instead of the sync-free
    #: kernel (measured slower: a grid barrier costs ~7 us per level vs
    #: ~5.6 us of flag latency; profiles/r02_trs_sweep.txt)
    LEVEL_SYNC = False

    def __init__(self, factor: Csr, lower: bool, unit_diagonal=False):
        _require_cuda(factor.exec)
        super().__init__(factor.exec, factor.size)
        self.factor = factor
        self.lower = lower
        self.unit_diagonal = unit_diagonal
        self.diag = None
        if not unit_diagonal:
            diag, bad = extract_diagonal(factor)
            if bad != INT_MAX:
                raise Singular(f"zero diagonal entry in row {bad}")
            self.diag = diag
        dev = factor.exec.device
        self._ready = torch.zeros(max(factor.size.rows, 1), dtype=torch.int32, device=dev)
        self._ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        self._epoch = 0
        self._levels = None
        self._order, self._nlevels = self._level_order()

    def _level_order(self):
        """Rows grouped by dependency level, computed on the device by
        relaxation sweeps (one host check per sweep; depth + 1 sweeps)."""
        f, exc = self.factor, self.exec
        n = f.size.rows
        if n == 0:
            return None, 0
        dev = exc.device
        level = torch.zeros(n, dtype=torch.int32, device=dev)
        changed = torch.zeros(1, dtype=torch.int32, device=dev)
        while True:
            changed.zero_()
            _lib.call("trs_levels", n, ptr(f._rp), ptr(f._ci), int(self.lower), ptr(level), ptr(changed),
                      exc.stream)
            if not int(changed.item()):
                break
        nlev = int(level.max().item()) + 1
        count = torch.zeros(nlev, dtype=torch.int32, device=dev)
        _lib.call("trs_level_hist", n, ptr(level), ptr(count), exc.stream)
        offs = _scan(exc, count)
        cursor = torch.zeros(nlev, dtype=torch.int32, device=dev)
        order = torch.empty(n, dtype=torch.int32, device=dev)
        _lib.call("trs_order", n, ptr(level), ptr(offs), ptr(cursor), ptr(order), exc.stream)
        self._level_of = level
        self._level_offs = offs
        return order, nlev

    @property
    def levels(self):
        """Rows grouped by dependency level (reference attribute; host)."""
        if self._levels is None:
            f = self.factor
            n = f.size.rows
            rp, ci = np.asarray(f.row_ptrs), np.asarray(f.col_idxs)
            level = np.zeros(n, dtype=np.int64)
            for i in (range(n) if self.lower else range(n - 1, -1, -1)):
                deps = ci[rp[i]:rp[i + 1]]
                deps = deps[deps != i]
                if deps.size:
                    level[i] = level[deps].max() + 1
            self._levels = [np.flatnonzero(level == lv) for lv in range(int(level.max()) + 1 if n else 0)]
        return self._levels

    def _apply_impl(self, b, x):
        f = self.factor
        n = f.size.rows
        bv, xv = b.values, x.values
        suf = _lib.suffix(xv.dtype)
        isz = xv.element_size()
        for j in range(xv.shape[1]):
            if self.LEVEL_SYNC and self._order is not None:
                _lib.call("trs_coop_" + suf, n, ptr(f._rp), ptr(f._ci), ptr(f._v),
                          ptr(self.diag) if self.diag is not None else 0,
                          bv.data_ptr() + j * bv.stride(1) * isz, bv.stride(0),
                          xv.data_ptr() + j * xv.stride(1) * isz, xv.stride(0),
                          ptr(self._order), ptr(self._level_offs), self._nlevels, self.exec.stream)
                continue
            self._epoch += 1
            _lib.call("trs_" + suf, n, ptr(f._rp), ptr(f._ci), ptr(f._v),
                      ptr(self.diag) if self.diag is not None else 0, int(self.lower),
                      bv.data_ptr() + j * bv.stride(1) * isz, bv.stride(0),
                      xv.data_ptr() + j * xv.stride(1) * isz, xv.stride(0),
                      ptr(self._ready), self._epoch, ptr(self._ticket), ptr(self._order), self.exec.stream)

    def clone_to(self, target):
        return TriangularSolver(self.factor.clone_to(target), self.lower, self.unit_diagonal)


def _as_csr(a):
    return a if isinstance(a, Csr) else a.convert_to(Csr)


class LowerTrs(LinOpFactory):
    """Forward substitution with a lower-triangular factor."""

    def __init__(self, exc, unit_diagonal=False):
        super().__init__(exc)
        self.unit_diagonal = unit_diagonal

    def _validate(self, a):
        if not a.size.square:
            raise DimensionMismatch("triangular factor must be square")

    def _generate(self, a):
        return TriangularSolver(_as_csr(a), lower=True, unit_diagonal=self.unit_diagonal)


class UpperTrs(LinOpFactory):
    """Backward substitution with an upper-triangular factor."""

    def __init__(self, exc, unit_diagonal=False):
        super().__init__(exc)
        self.unit_diagonal = unit_diagonal

    def _validate(self, a):
        if not a.size.square:
            raise DimensionMismatch("triangular factor must be square")

    def _generate(self, a):
        return TriangularSolver(_as_csr(a), lower=False, unit_diagonal=self.unit_diagonal)
