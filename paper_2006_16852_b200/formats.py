"""Matrix formats on the device: Dense, Csr, Coo, Ell, Sellp, Hybrid.

API mirror of the reference's src/formats.py:21-329 (MatrixData interchange,
Dense doubling as the vector type, Csr/Coo with from_data / to_data /
convert_to / clone_to, ``convert`` and ``matrix_from_data``) extended with the
formats the paper names but the reference omits: Ell, Sellp,
Hybrid, and the Csr strategies ``classical`` / ``load_balance``.

Storage lives in HBM as torch tensors; every numeric operation is an
sm_100a kernel of libb200sp. Conversions use Csr as the hub and run on the
device (two-phase: size query, fill). ``MatrixData`` is the host interchange
form (file I/O, assembly) exactly as in the reference.
"""

from __future__ import annotations

import copy
import math
import threading

import numpy as np

from . import _lib, config
from .loggers import EventKind
from .base import Dim2, LinOp
from .errors import DimensionMismatch, Unsupported
from .executor import CudaExecutor, DeviceView, HostExecutor, ptr
from .kernels import AddScaledOp, CopyOp, DotOp, FillOp, ScaleOp, SpmvOp

try:
    import torch
except Exception:  # pragma: no cover
    torch = None


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def _np_vt(value_dtype):
    dt = np.dtype(value_dtype or config.DEFAULT_VALUE_DTYPE)
    if dt not in (np.dtype("float64"), np.dtype("float32")):
        raise Unsupported(f"value type {dt} (supported: float64, float32)")
    return dt


def _torch_vt(np_dt):
    return torch.float64 if np.dtype(np_dt) == np.float64 else torch.float32


def _check_index_dtype(index_dtype):
    if index_dtype is not None and np.dtype(index_dtype) != np.dtype("int32"):
        raise Unsupported("this backend stores 32-bit indices (DEFAULT_INDEX_DTYPE)")


def _to_device(exc, arr, torch_dtype):
    if torch is not None and isinstance(arr, torch.Tensor):
        return arr.to(device=exc.device, dtype=torch_dtype).contiguous()
    if isinstance(arr, DeviceView):
        return arr.tensor.to(dtype=torch_dtype).contiguous()
    a = np.ascontiguousarray(np.asarray(arr))
    t = torch.from_numpy(a).to(torch_dtype) if a.size else torch.empty(a.shape, dtype=torch_dtype)
    return t.to(exc.device)


def _scan(exc, counts):
    """Exclusive scan of int32 counts -> int32 tensor of len+1 (total last)."""
    n = counts.numel()
    out = torch.empty(n + 1, dtype=torch.int32, device=exc.device)
    ws = torch.empty(max(1, int(_lib.query("scan_workspace_elems", n))), dtype=torch.int64,
                     device=exc.device)
    _lib.call("exclusive_scan_i32", n, ptr(counts), ptr(out), ptr(ws), exc.stream)
    return out


def _max_i32(exc, t):
    out = torch.empty(1, dtype=torch.int32, device=exc.device)
    _lib.call("reduce_max_i32", t.numel(), ptr(t), ptr(out), exc.stream)
    return int(out.item())


def _require_cuda(exc):
    if not isinstance(exc, CudaExecutor):
        raise Unsupported("sparse matrices live on a CudaExecutor "
                          "(the host arena runs no numeric kernels)")


# ---------------------------------------------------------------------------
# MatrixData (host interchange; src/formats.py:21-64)
# ---------------------------------------------------------------------------
class MatrixData:
    """Size plus coordinate triples; canonical order is (row, col) with
    duplicates summed in their original order (src/formats.py:40-53)."""

    def __init__(self, size, rows=(), cols=(), vals=()):
        self.size = size if isinstance(size, Dim2) else Dim2(*size)
        self.rows = np.asarray(rows, dtype=np.int64).reshape(-1)
        self.cols = np.asarray(cols, dtype=np.int64).reshape(-1)
        self.vals = np.asarray(vals, dtype=np.float64).reshape(-1)
        if not (self.rows.size == self.cols.size == self.vals.size):
            raise DimensionMismatch("triple arrays must have equal length")

    @property
    def nnz(self):
        return int(self.vals.size)

    def is_canonical(self):
        if self.nnz < 2:
            return True
        key_ok = (self.rows[1:] > self.rows[:-1]) | (
            (self.rows[1:] == self.rows[:-1]) & (self.cols[1:] > self.cols[:-1]))
        return bool(key_ok.all())

    def canonicalize(self):
        if self.nnz == 0:
            return MatrixData(self.size)
        if self.is_canonical():
            return MatrixData(self.size, self.rows, self.cols, self.vals)
        order = np.lexsort((self.cols, self.rows))
        r, c, v = self.rows[order], self.cols[order], self.vals[order]
        first = np.ones(r.size, dtype=bool)
        first[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        if not first.all():
            grp = np.cumsum(first) - 1
            acc = np.zeros(int(grp[-1]) + 1, dtype=np.float64)
            np.add.at(acc, grp, v)
            r, c, v = r[first], c[first], acc
        return MatrixData(self.size, r, c, v)

    def to_dense_array(self):
        out = np.zeros(tuple(self.size), dtype=np.float64)
        np.add.at(out, (self.rows, self.cols), self.vals)
        return out

    @classmethod
    def from_dense_array(cls, arr, drop_zeros=True):
        arr = np.asarray(arr, dtype=np.float64)
        if drop_zeros:
            r, c = np.nonzero(arr)
        else:
            r, c = np.indices(arr.shape).reshape(2, -1)
        return cls(Dim2(*arr.shape), r, c, arr[r, c])


# ---------------------------------------------------------------------------
# Dense (src/formats.py:67-158)
# ---------------------------------------------------------------------------
class Dense(LinOp):
    """Row-major (rows, cols) block; doubles as the multi-column vector type.

    ``values`` is the storage (torch tensor on a CudaExecutor, numpy array on
    the host arena); ``data`` is numpy-compatible in both cases (a
    synchronising DeviceView for device storage)."""

    is_dense = True

    def __init__(self, exc, data=None, size=None, value_dtype=None):
        if data is not None:
            if torch is not None and isinstance(data, torch.Tensor):
                vt = _np_vt(value_dtype or str(data.dtype).replace("torch.", ""))
                t = data if data.dim() == 2 else data.reshape(1, -1)
                vals = self._adopt(exc, t, vt)
            else:
                vt = _np_vt(value_dtype)
                arr = np.array(data, dtype=vt, ndmin=2)
                vals = self._adopt(exc, arr, vt)
        else:
            vt = _np_vt(value_dtype)
            vals = exc.alloc(tuple(int(s) for s in size), vt.name)
        super().__init__(exc, Dim2(*vals.shape))
        self.values = vals

    @staticmethod
    def _adopt(exc, arr, vt):
        if isinstance(exc, CudaExecutor):
            return _to_device(exc, arr, _torch_vt(vt))
        if torch is not None and isinstance(arr, torch.Tensor):
            arr = arr.detach().cpu().numpy()
        out = exc.alloc(arr.shape, vt.name)
        out[...] = arr
        return out

    # -- storage views -----------------------------------------------------
    @property
    def on_device(self):
        return isinstance(self.exec, CudaExecutor)

    @property
    def data(self):
        return DeviceView(self.values) if self.on_device else self.values

    @property
    def dtype(self):
        return np.dtype(str(self.values.dtype).replace("torch.", ""))

    @property
    def stride(self):
        if self.on_device:
            return self.values.stride(0)
        return self.values.strides[0] // self.values.itemsize

    # -- constructors --------------------------------------------------------
    @classmethod
    def zeros(cls, exc, rows, cols=1, value_dtype=None):
        out = cls(exc, size=(rows, cols), value_dtype=value_dtype)
        out.fill(0.0)
        return out

    @classmethod
    def vector(cls, exc, values, value_dtype=None):
        if torch is not None and isinstance(values, torch.Tensor):
            return cls(exc, values.reshape(-1, 1), value_dtype=value_dtype)
        arr = np.asarray(values, dtype=_np_vt(value_dtype))
        return cls(exc, arr.reshape(-1, 1), value_dtype=value_dtype)

    @classmethod
    def wrap(cls, exc, arr):
        """Dense view over existing storage (no copy); arr is a 2-D tensor
        (device) or ndarray (host)."""
        obj = cls.__new__(cls)
        LinOp.__init__(obj, exc, Dim2(*arr.shape))
        obj.values = arr
        return obj

    def like(self, rows, cols):
        return Dense(self.exec, size=(rows, cols), value_dtype=self.dtype)

    def empty_like_on(self, target):
        return Dense(target, size=tuple(self.size), value_dtype=self.dtype)

    def column(self, j):
        """(n, 1) view of column j (no copy)."""
        return Dense.wrap(self.exec, self.values[:, j:j + 1])

    def clone_to(self, target):
        out = Dense(target, size=tuple(self.size), value_dtype=self.dtype)
        out.copy_from(self)
        return out

    def to_numpy(self):
        return np.asarray(self.data).copy()

    # -- BLAS-1 (kernels; src/formats.py:121-147) ----------------------------
    def fill(self, value=0.0):
        self.exec.run(FillOp(self, value))

    def copy_from(self, other):
        """self <- other (same shape); handles host<->device migration."""
        if other.exec is self.exec:
            self.exec.run(CopyOp(other, self))
            return
        src, dst = other.values, self.values
        if self.on_device and other.on_device:
            dst.copy_(src)
        elif self.on_device:  # H2D (pinned source -> async on the current stream)
            dst.copy_(torch.from_numpy(np.asarray(src)), non_blocking=True)
        elif other.on_device:  # D2H into the host arena; synchronous on return
            host = torch.from_numpy(dst) if dst.flags.c_contiguous else None
            if host is not None:
                host.copy_(src, non_blocking=True)
                torch.cuda.current_stream(src.device).synchronize()
            else:
                dst[...] = src.detach().cpu().numpy()
        else:
            dst[...] = src

    def scale(self, alpha):
        self.exec.run(ScaleOp(alpha, self))

    def add_scaled(self, alpha, x):
        self.exec.run(AddScaledOp(alpha, x, self))

    def compute_dot(self, other, out):
        self.exec.run(DotOp(self, other, out))

    def compute_norm2(self, out):
        self.exec.run(DotOp(self, self, out, norm=True))

    def dot(self, other):
        out = self.like(1, self.size.cols)
        self.compute_dot(other, out)
        return np.asarray(out.data)[0].copy()

    def norm2(self):
        out = self.like(1, self.size.cols)
        self.compute_norm2(out)
        return np.asarray(out.data)[0].copy()

    # -- operator interface ------------------------------------------------------
    def _apply_impl(self, b, x):
        self.exec.run(SpmvOp(self, b, x))

    def _launch_column(self, exc, suf, bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins):
        a = self.values
        if a_p or xin or a_h != 1.0:
            raise Unsupported("Dense advanced apply goes through the generic path")
        _lib.call("dense_spmv_" + suf, a.shape[0], a.shape[1], ptr(a), a.stride(0), bp, bs, xp, xs,
                  exc.stream)

    def convert_to(self, kind):
        return convert(self, kind)

    def to_data(self):
        return MatrixData.from_dense_array(np.asarray(self.data))

    def _to_csr(self, **kw):
        _require_cuda(self.exec)
        exc, a = self.exec, self.values
        n, k = a.shape
        suf = _lib.suffix(a.dtype)
        lens = torch.empty(n, dtype=torch.int32, device=exc.device)
        _lib.call("dense_row_nnz_" + suf, n, k, ptr(a), a.stride(0), ptr(lens), exc.stream)
        rp = _scan(exc, lens)
        nnz = int(rp[-1].item())
        ci = torch.empty(nnz, dtype=torch.int32, device=exc.device)
        v = torch.empty(nnz, dtype=a.dtype, device=exc.device)
        _lib.call("dense_to_csr_fill_" + suf, n, k, ptr(a), a.stride(0), ptr(rp), ptr(ci), ptr(v),
                  exc.stream)
        return Csr._from_device(exc, Dim2(n, k), rp, ci, v, **kw)

    @classmethod
    def _from_csr(cls, csr, **_):
        exc = csr.exec
        out = cls.zeros(exc, csr.size.rows, csr.size.cols, value_dtype=csr.value_dtype)
        a = out.values
        _lib.call("csr_to_dense_" + _lib.suffix(a.dtype), csr.size.rows, ptr(csr._rp), ptr(csr._ci),
                  ptr(csr._v), ptr(a), a.stride(0), exc.stream)
        return out


# ---------------------------------------------------------------------------
# sparse base
# ---------------------------------------------------------------------------
class _Sparse(LinOp):
    def __init__(self, exc, size):
        _require_cuda(exc)
        super().__init__(exc, size)

    @property
    def value_dtype(self):
        return np.dtype(str(self._v.dtype).replace("torch.", ""))

    def _apply_impl(self, b, x):
        self.exec.run(SpmvOp(self, b, x))

    def _apply_advanced_impl(self, alpha, b, beta, x):
        self.exec.run(SpmvOp(self, b, x, alpha=alpha, beta=beta, x_in=x))

    def residual(self, x, b, r):
        """r <- b - A x in one fused launch per column (CooResidualKernel,
        src/kernels.py:243-275, generalised to every format)."""
        self.exec.run(SpmvOp(self, x, r, alpha=-1.0, beta=1.0, x_in=b))

    def convert_to(self, kind, **kw):
        return convert(self, kind, **kw)

    @classmethod
    def from_data(cls, exc, data, **kw):
        csr = Csr._from_host_data(exc, data, kw.pop("value_dtype", None),
                                  kw.pop("index_dtype", None))
        return csr if cls is Csr and not kw else cls._from_csr(csr, **kw)

    def to_data(self):
        return self._to_csr().to_data()

    def clone_to(self, target):
        """Deep copy with identical apply behaviour on ``target``."""
        _require_cuda(target)
        obj = copy.copy(self)
        LinOp.__init__(obj, target, self.size)
        for name, val in vars(self).items():
            if torch is not None and isinstance(val, torch.Tensor):
                setattr(obj, name, val.clone().to(target.device))
            elif isinstance(val, _Sparse):
                setattr(obj, name, val.clone_to(target))
        # per-instance caches hold device buffers, streams and CUDA graphs
        # captured against the SOURCE's pointers: the clone rebuilds its own
        for cache in _INSTANCE_CACHES:
            if hasattr(obj, cache):
                setattr(obj, cache, None)
        return obj


#: lazily built per-instance state that must never be shared by clones
_INSTANCE_CACHES = ("_plan", "_ws", "_pplan")


# ---------------------------------------------------------------------------
# Csr (src/formats.py:168-221) + strategies
# ---------------------------------------------------------------------------
CSR_STRATEGIES = ("classical", "load_balance", "stream", "automatic")


_PIPELINE_LOCK = threading.Lock()


def assemble_device(exc, data, vt):
    """MatrixData -> canonical (row, col)-sorted int32 rows / cols and values
    on the device (csrc/assemble.cu): the reference's canonicalize
    (src/formats.py:40-53) bit for bit -- stable sort by (row, col),
    duplicates summed in input order -- so Csr.from_data never sorts on the
    host. Index ranges are validated first (the reference's Csr/Coo checks)."""
    n, m = data.size
    k = data.nnz
    if k:
        if int(data.rows.min()) < 0 or int(data.rows.max()) >= n:
            raise DimensionMismatch("row index out of range")
        if int(data.cols.min()) < 0 or int(data.cols.max()) >= m:
            raise DimensionMismatch("column index out of range")
    if k >= 2 ** 31 - 1:
        raise Unsupported("more than 2^31-1 stored entries need 64-bit indices")
    dev = exc.device
    tv = _torch_vt(vt)
    rows_o = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    cols_o = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    vals_o = torch.empty(max(k, 1), dtype=tv, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    if k:
        r = torch.from_numpy(np.ascontiguousarray(data.rows, dtype=np.int64)).to(dev)
        c = torch.from_numpy(np.ascontiguousarray(data.cols, dtype=np.int64)).to(dev)
        v = torch.from_numpy(np.ascontiguousarray(data.vals, dtype=np.float64)).to(dev)
        ws = torch.empty(int(_lib.query("assemble_workspace_bytes", k)), dtype=torch.uint8, device=dev)
        _lib.call("assemble_coo_" + _lib.suffix(tv), k, ptr(r), ptr(c), ptr(v), n, m, ptr(rows_o), ptr(cols_o),
                  ptr(vals_o), ptr(cnt), ptr(ws), exc.stream)
    nnz = int(cnt.item())
    return rows_o[:nnz], cols_o[:nnz], vals_o[:nnz]


class Csr(_Sparse):
    """Compressed sparse row with an SpMV strategy:

    * ``classical``    -- sub-warp per row, several rows in flight per
                          sub-warp (sub-warp = next power of two of
                          mean row length / 8, capped at 32);
    * ``load_balance`` -- merge-path tiles of equal (rows + nonzeros) work
                          with a deterministic carry fix-up;
    * ``stream``       -- row blocks whose nonzeros are staged through shared
                          memory with 128-bit loads, thread-per-row reduction;
    * ``automatic``    -- classical unless the row lengths are skewed
                          (max > 4 x mean + 64), then load_balance.
    """

    def __init__(self, exc, size, row_ptrs, col_idxs, vals, index_dtype=None, value_dtype=None,
                 strategy="automatic"):
        super().__init__(exc, size)
        _check_index_dtype(index_dtype)
        vt = _np_vt(value_dtype or (getattr(vals, "dtype", None) if not isinstance(vals, (list, tuple))
                                    else None) or config.DEFAULT_VALUE_DTYPE)
        host_check = not (torch is not None and isinstance(row_ptrs, torch.Tensor))
        if host_check:
            rp_h = np.asarray(row_ptrs, dtype=np.int64).reshape(-1)
            ci_h = np.asarray(col_idxs, dtype=np.int64).reshape(-1)
            nv = np.asarray(vals).size
            self._check_structure(rp_h, ci_h, nv)
        self._rp = _to_device(exc, row_ptrs, torch.int32)
        self._ci = _to_device(exc, col_idxs, torch.int32)
        self._v = _to_device(exc, vals, _torch_vt(vt))
        self._set_strategy(strategy)

    def _check_structure(self, rp, ci, nvals):
        rows, cols = self.size
        if rp.size != rows + 1 or rp[0] != 0 or rp[-1] != nvals:
            raise DimensionMismatch("bad row_ptrs")
        if np.any(np.diff(rp) < 0):
            raise DimensionMismatch("row_ptrs must be non-decreasing")
        if ci.size and (ci.min() < 0 or ci.max() >= cols):
            raise DimensionMismatch("column index out of range")
        if rp[-1] >= 2 ** 31:
            raise Unsupported("more than 2^31-1 stored entries need 64-bit indices")

    @classmethod
    def _from_device(cls, exc, size, rp, ci, v, strategy="automatic"):
        obj = cls.__new__(cls)
        _Sparse.__init__(obj, exc, size)
        obj._rp, obj._ci, obj._v = rp, ci, v
        obj._set_strategy(strategy)
        return obj

    @classmethod
    def _from_host_data(cls, exc, data, value_dtype=None, index_dtype=None):
        """Device assembly: raw triples go to the GPU once, where they are
        canonicalised bit-exactly (assemble_device) and compressed."""
        _require_cuda(exc)
        _check_index_dtype(index_dtype)
        n = data.size.rows
        vt = _np_vt(value_dtype or config.DEFAULT_VALUE_DTYPE)
        ri, ci, v = assemble_device(exc, data, vt)
        rp = torch.empty(n + 1, dtype=torch.int32, device=exc.device)
        _lib.call("coo_to_csr_ptrs", int(v.numel()), n, ptr(ri), ptr(rp), exc.stream)
        return cls._from_device(exc, data.size, rp, ci, v)

    # -- strategy ----------------------------------------------------------------
    def _set_strategy(self, strategy):
        if strategy not in CSR_STRATEGIES:
            raise Unsupported(f"csr strategy {strategy!r} (known: {CSR_STRATEGIES})")
        self._requested = strategy
        self._plan = None      # (coords, carry_row, carry_val) for load_balance
        self._subwarp = None
        self._max_row = None

    @property
    def strategy(self):
        return self._resolved_strategy()

    def set_strategy(self, strategy, subwarp=None, stream_shape=None, stream_cap=None, stream_impl=None,
                     gather_in_reduce=None, stream_stages=None, stream_consumers=None, lb_mode=None):
        """Switch SpMV strategy; ``subwarp`` pins the classical sub-warp size,
        ``stream_shape`` = (threads per row, rows per thread), ``stream_cap``
        (entries per staging chunk), ``stream_impl`` ("tma": bulk-copy
        staging, "ld": 128-bit load staging) and ``gather_in_reduce`` (gather
        x row-coherently in the reduction) the stream one."""
        self._set_strategy(strategy)
        self._stream_shape = tuple(stream_shape) if stream_shape is not None else None
        self._stream_cap = int(stream_cap) if stream_cap else None
        self._stream_stages = int(stream_stages) if stream_stages else None
        self._stream_consumers = int(stream_consumers) if stream_consumers else None
        if lb_mode is not None:
            if lb_mode not in (2, 3):
                raise Unsupported("lb_mode must be 2 (row-parallel tiles) or 3 (nnz split)")
            self._lb_mode = int(lb_mode)
        if stream_impl is not None:
            self._stream_impl = stream_impl
        if gather_in_reduce is not None:
            self._stream_gr = bool(gather_in_reduce)
        if subwarp is not None:
            if subwarp not in (1, 2, 4, 8, 16, 32):
                raise Unsupported("subwarp must be a power of two <= 32")
            self._subwarp = int(subwarp)

    def _row_stats(self):
        if self._max_row is None:
            n = self.size.rows
            if n == 0:
                self._max_row = 0
            else:
                lens = torch.empty(n, dtype=torch.int32, device=self.exec.device)
                _lib.call("csr_row_lengths", n, ptr(self._rp), ptr(lens), self.exec.stream)
                self._max_row = _max_i32(self.exec, lens)
        return self._max_row

    def _resolved_strategy(self):
        """automatic: load_balance for skewed row lengths (max > 4 x mean +
        64), else classical -- with L1-allocating matrix loads the sub-warp
        kernel is the fastest Csr SpMV measured on B200 for every stencil
        (C2 fp64 0.82, fp32 0.79-0.81, 7-point 0.87 of the HBM roofline;
        profiles/r03_classical_kb.txt) ahead of the staged stream kernels."""
        if self._requested != "automatic":
            return self._requested
        n = self.size.rows
        if n == 0:
            return "classical"
        mean = self.nnz / n
        if self._row_stats() > 4 * mean + 64:
            return "load_balance"
        # (fp32 with long rows took the TMA pipeline, 0.759 vs 0.72, until the
        # classical kernel's aligned pair loads: 0.79-0.81 vs 0.75 on C2,
        # profiles/r03_classical_kb.txt)
        return "classical"

    def _stream_ok(self):
        return self._rp.data_ptr() % 16 == 0 and self._ci.data_ptr() % 16 == 0 and self._v.data_ptr() % 16 == 0

    def subwarp(self):
        if self._subwarp is None:
            n = self.size.rows
            per_lane = max(1, math.ceil(self.nnz / max(n, 1) / 8))
            self._subwarp = min(32, 1 << (per_lane - 1).bit_length())
        return self._subwarp

    def stream_impl(self):
        """"tma" (persistent bulk-copy pipeline) or "ld" (register-staged CTA
        blocks). Measured on B200 (profiles/r02_pipe_sweep.txt, clean-L2
        timing): 27-point fp64 tma 0.728 vs ld 0.573 of the HBM roofline;
        27-point fp32 ld 0.728 vs tma 0.673; 7-point fp64 ld 0.758 vs tma
        0.378 -- short rows leave too few rows in flight per stage to hide the
        x-gather latency behind 16 consumer warps."""
        impl = getattr(self, "_stream_impl", None)
        if impl is not None:
            return impl
        mean = self.nnz / max(1, self.size.rows)
        return "tma" if mean >= 12 else "ld"

    def tma_config(self):
        """(entries per stage, rows per thread, stages, consumer threads,
        threads per row) of the persistent TMA pipeline. Default (measured
        best for 27-point fp64): 512 consumers, two threads per row, two rows
        per thread group (tiles of 512 rows), stages as large as two fit."""
        vb = self._v.element_size()
        shape = getattr(self, "_stream_shape", None)
        mean = self.nnz / max(1, self.size.rows)
        if shape is None:
            # fp64 long rows: 512 consumers, 2 threads x 2 rows (0.727); fp32
            # long rows: 256 consumers, thread per row, whole-tile stages, two
            # CTAs per SM (0.759)
            shape = ((2, 2) if vb == 8 else (1, 1)) if mean >= 12 else (1, 4 if mean < 6 else 2)
        tpr, rpt = shape
        nt = int(getattr(self, "_stream_consumers", None) or (512 if tpr > 1 else 256))
        rows = nt // tpr * rpt
        budget = 220 * 1024 - 256
        rp_bytes = ((rows + 1 + 3) // 4 * 4) * 4
        need = (rows * max(1, self._row_stats()) + 4 + 3) // 4 * 4
        cap_fit2 = ((budget // 2 - rp_bytes) // (4 + vb)) // 4 * 4
        cap = int(getattr(self, "_stream_cap", None) or min(need, cap_fit2))
        stage = rp_bytes + cap * (4 + vb)
        # two stages per CTA: three measured slower everywhere (the ring only
        # has to cover one tile of latency); two CTAs per SM when they fit
        stages = int(getattr(self, "_stream_stages", None) or 2)
        return cap, rpt, stages, nt, tpr

    def stream_config(self):
        """(chunk entries, threads per row, rows per thread) of the stream
        kernel: long rows share 2 threads (fp64), short rows give each thread
        several rows so a CTA still stages thousands of nonzeros; the chunk
        holds a whole row block when it fits."""
        vb = self._v.element_size()
        longest = max(1, self._row_stats())
        shape = getattr(self, "_stream_shape", None)
        if shape is None:
            # measured on C2 / 7-pt / 5-pt (tools/spmv_sweep.py): fp64 27-pt 1x2,
            # 7-pt 1x2, 5-pt 1x4; fp32 27-pt 1x1
            mean = self.nnz / max(1, self.size.rows)
            if vb == 4 and mean >= 16:
                shape = (1, 1)
            elif mean < 12:
                shape = (1, 4)
            else:
                shape = (1, 2)
        tpr, rpt = shape
        # gather-in-reduce pays off for long fp64 rows only (27-pt: 62% vs 60%;
        # 7-pt and fp32 lose; profiles/r01_stream_sweep.txt)
        gr_default = vb == 8 and self.nnz / max(1, self.size.rows) >= 12
        gr = int(getattr(self, "_stream_gr", gr_default))
        # 32 KB of staging per CTA measured best (64 KB halves the CTAs per SM;
        # profiles/r01_stream_sweep.txt); GR stages (col, val) = 4 + VT bytes
        per = vb + (4 if gr else 0)
        cap = int(getattr(self, "_stream_cap", None) or (32768 // per) // 4 * 4)
        rows = (256 // tpr) * rpt
        need = (rows * longest + 4 + 3) // 4 * 4
        return min(cap, need), tpr, rpt, gr

    def lb_mode(self):
        """2 = row-parallel merge-path tiles (stencils: C2 fp64 0.70, 7-point
        0.85), 3 = nnz split with Coo-style warp chunks (skewed rows: C3 power
        law 404 us vs 617 us row-parallel; profiles/r03_c3_seg.txt). Chosen
        automatically from the longest row."""
        mode = getattr(self, "_lb_mode", None)
        if mode is None:
            n = self.size.rows
            mean = self.nnz / max(n, 1)
            mode = 3 if n and self._row_stats() > 4 * mean + 64 else 2
        return mode

    def lb_plan(self):
        if self._plan is None:
            exc = self.exec
            n, nnz = self.size.rows, self.nnz
            vb = self._v.element_size()
            mode = self.lb_mode()
            tile = int(_lib.query("csr_lb_tile", vb, mode))
            if mode == 3:  # nnz split: chunk start rows, chunk tail rows, head + tail carries
                nt = (nnz + tile - 1) // tile
                coords = torch.empty(nt + 1, dtype=torch.int32, device=exc.device)
                _lib.call("csr_seg_plan", n, nnz, ptr(self._rp), ptr(coords), exc.stream)
                carry_row = torch.empty(max(nt, 1), dtype=torch.int32, device=exc.device)
                carry_val = torch.empty(max(2 * nt, 1), dtype=self._v.dtype, device=exc.device)
                self._plan = (coords, carry_row, carry_val, tile, mode)
                return self._plan
            nt = int(_lib.query("csr_lb_num_tiles", n, nnz, tile))
            coords = torch.empty(2 * (nt + 1), dtype=torch.int32, device=exc.device)
            _lib.call("csr_lb_plan", n, nnz, ptr(self._rp), tile, ptr(coords), exc.stream)
            carry_row = torch.empty(max(nt, 1), dtype=torch.int32, device=exc.device)
            carry_val = torch.empty(max(nt, 1), dtype=self._v.dtype, device=exc.device)
            self._plan = (coords, carry_row, carry_val, tile, mode)
        return self._plan

    # -- attributes (reference names) --------------------------------------------
    @property
    def nnz(self):
        return int(self._v.numel())

    @property
    def row_ptrs(self):
        return DeviceView(self._rp)

    @property
    def col_idxs(self):
        return DeviceView(self._ci)

    @property
    def vals(self):
        return DeviceView(self._v)

    # -- host operands: pipelined transfers -----------------------------------------
    #: row chunks of the pipelined host apply (0 disables it)
    HOST_PIPELINE_CHUNKS = 8  # 4 / 8 / 16 measured 0.626 / 0.568 / 0.649 ms on C2 (link ceiling 0.38)

    def apply(self, b, x):
        """x <- A b. With both operands in host (pinned) memory, a single column
        and the row-parallel classical strategy, the transfers are pipelined
        with the SpMV: b goes up in chunks on one copy stream, each row chunk
        starts as soon as every b entry its columns reach has arrived (column
        range per chunk, planned once), and x comes down chunk by chunk on a
        second copy stream -- H2D and D2H overlap each other and the kernels
        instead of running back to back (same results: rows are independent)."""
        if not self._pipeline_ok(b, x):
            return super().apply(b, x)
        self._check_usable()
        self._check_conformal(b, x)
        self._log(EventKind.LINOP_APPLY_STARTED, {"op": type(self).__name__, "uid": self.uid})
        with _PIPELINE_LOCK:  # the plan's device buffers / graphs are shared
            self._pipelined_apply(b, x)
        self._log(EventKind.LINOP_APPLY_COMPLETED, {"op": type(self).__name__, "uid": self.uid})

    def _pipeline_ok(self, b, x):
        from .executor import HostExecutor

        if not (self.HOST_PIPELINE_CHUNKS > 0 and isinstance(getattr(b, "exec", None), HostExecutor)
                and isinstance(getattr(x, "exec", None), HostExecutor) and b.exec.pinned and x.exec.pinned
                and getattr(b, "is_dense", False) and getattr(x, "is_dense", False)
                and b.size.cols == 1 and x.size.cols == 1 and self.size.rows >= (1 << 16)
                and self._resolved_strategy() == "classical"
                and np.asarray(b.values).flags.c_contiguous and np.asarray(x.values).flags.c_contiguous
                and np.dtype(b.dtype) == self.value_dtype and np.dtype(x.dtype) == self.value_dtype):
            return False
        # the graph issues non_blocking copies: both buffers must really be
        # page-locked (a Dense.wrap of a user ndarray on a pinned executor is not)
        return all(torch.from_numpy(np.asarray(v.values).reshape(-1)).is_pinned() for v in (b, x))

    # (a cooperative kernel streaming b from / x to host memory over PCIe --
    # SM loads / stores to host memory -- measured slower than the copy
    # engines: C2 0.54 vs 0.50 ms, profiles/r02_e2e_probe.txt; archived as
    # tools/hoststream_probe.cu)

    def _pipeline_plan(self):
        plan = getattr(self, "_pplan", None)
        if plan is None:
            n = self.size.rows
            k = self.HOST_PIPELINE_CHUNKS
            bounds = [n * j // k for j in range(k + 1)]
            rp = self._rp.cpu().numpy()
            ci = self._ci
            need = []  # highest column each row chunk reads
            for j in range(k):
                lo, hi = int(rp[bounds[j]]), int(rp[bounds[j + 1]])
                need.append(int(ci[lo:hi].max().item()) if hi > lo else -1)
            m = self.size.cols
            # b chunk i ends right after the highest column row chunk i reads
            # (running max), so row chunk j waits only for b chunks 0..j --
            # not for the next one, as equal b chunks would for a band
            cb, hi = [0], 0
            for j in range(k - 1):
                hi = min(m, max(hi, need[j] + 1, cb[-1]))
                cb.append(hi)
            cb.append(m)
            # b chunk index whose arrival completes columns [0, need]
            wait = [next(i for i in range(k) if cb[i + 1] > nd) if nd >= 0 else -1 for nd in need]
            dev = self.exec.device
            plan = {"rows": bounds, "cols": cb, "wait": wait,
                    "s_in": torch.cuda.Stream(dev), "s_out": torch.cuda.Stream(dev),
                    "b": torch.empty(m, dtype=self._v.dtype, device=dev),
                    "x": torch.empty(n, dtype=self._v.dtype, device=dev)}
            self._pplan = plan
        return plan

    def _pipelined_apply(self, b, x):
        """Replays a CUDA graph of the whole chunked pipeline (captured once per
        pair of host buffers: one launch instead of ~4 per chunk)."""
        P = self._pipeline_plan()
        bh = torch.from_numpy(np.asarray(b.values).reshape(-1))
        xh = torch.from_numpy(np.asarray(x.values).reshape(-1))
        key = (bh.data_ptr(), xh.data_ptr())
        graphs = P.setdefault("graphs", {})
        g = graphs.get(key)
        if g is None:
            if len(graphs) >= 4:
                graphs.clear()
            torch.cuda.synchronize(self.exec.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._pipeline_issue(P, bh, xh)
            graphs[key] = g
        g.replay()
        torch.cuda.current_stream(self.exec.device).synchronize()

    def _pipeline_issue(self, P, bh, xh):
        exc = self.exec
        k = len(P["wait"])
        bd, xd = P["b"], P["x"]
        cur = torch.cuda.current_stream(exc.device)
        s_in, s_out = P["s_in"], P["s_out"]
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        ev_in = []
        with torch.cuda.stream(s_in):
            for i in range(k):
                lo, hi = P["cols"][i], P["cols"][i + 1]
                bd[lo:hi].copy_(bh[lo:hi], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_in)
                ev_in.append(e)
        suf = _lib.suffix(self._v.dtype)
        isz = self._v.element_size()
        sw = self._subwarp_arg()
        for j in range(k):
            r0, r1 = P["rows"][j], P["rows"][j + 1]
            if P["wait"][j] >= 0:
                cur.wait_event(ev_in[P["wait"][j]])
            _lib.call("csr_spmv_classical_" + suf, r1 - r0, self._rp.data_ptr() + 4 * r0, ptr(self._ci), ptr(self._v),
                      ptr(bd), 1, xd.data_ptr() + isz * r0, 1, 1.0, 0, 0.0, 0, 0, 0, sw, cur.cuda_stream)
            e = torch.cuda.Event()
            e.record(cur)
            s_out.wait_event(e)
            with torch.cuda.stream(s_out):
                xh[r0:r1].copy_(xd[r0:r1], non_blocking=True)
        cur.wait_stream(s_in)
        cur.wait_stream(s_out)

    # -- kernels -------------------------------------------------------------------
    def _launch_column(self, exc, suf, bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins):
        n = self.size.rows
        strategy = self._resolved_strategy()
        if strategy == "load_balance":
            coords, crow, cval, tile, mode = self.lb_plan()
            _lib.call("csr_spmv_lb_" + suf, n, self.nnz, ptr(self._rp), ptr(self._ci), ptr(self._v),
                      bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins, ptr(coords), ptr(crow),
                      ptr(cval), tile, mode, exc.stream)
        elif strategy == "stream" and self._stream_ok():
            if self.stream_impl() == "tma":
                _lib.call("csr_spmv_tma_" + suf, n, self.nnz, ptr(self._rp), ptr(self._ci), ptr(self._v),
                          bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins, *self.tma_config(), exc.stream)
            else:
                _lib.call("csr_spmv_stream_" + suf, n, self.nnz, ptr(self._rp), ptr(self._ci), ptr(self._v),
                          bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins, *self.stream_config(), exc.stream)
        else:
            _lib.call("csr_spmv_classical_" + suf, n, ptr(self._rp), ptr(self._ci), ptr(self._v),
                      bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins, self._subwarp_arg(), exc.stream)

    def _subwarp_arg(self):
        """The classical kernel's sub-warp width, flagged B200SP_SUBWARP_EVEN_NNZ
        when the entry count is even (aligned pair loads stay inside the arrays)."""
        return self.subwarp() | (self.SUBWARP_EVEN_NNZ if self.nnz % 2 == 0 else 0)

    SUBWARP_EVEN_NNZ = 0x100  # include/b200sp.h

    # -- conversions -------------------------------------------------------------------
    def _to_csr(self, **kw):
        return self

    @classmethod
    def _from_csr(cls, csr, strategy=None, exec=None, **_):
        target = exec or csr.exec
        return cls._from_device(target, csr.size, csr._rp.clone().to(target.device),
                                csr._ci.clone().to(target.device), csr._v.clone().to(target.device),
                                strategy=strategy or csr._requested)

    def to_data(self):
        rp = self._rp.cpu().numpy().astype(np.int64)
        rows = np.repeat(np.arange(self.size.rows, dtype=np.int64), np.diff(rp))
        return MatrixData(self.size, rows, self._ci.cpu().numpy().astype(np.int64),
                          self._v.cpu().numpy().astype(np.float64))


# ---------------------------------------------------------------------------
# Coo (src/formats.py:224-265)
# ---------------------------------------------------------------------------
COO_CHUNK = 256


class Coo(_Sparse):
    """Coordinate format, entries sorted by (row, col)."""

    #: entries per warp chunk of the SpMV kernel (128 or 256)
    chunk = COO_CHUNK

    def __init__(self, exc, size, row_idxs, col_idxs, vals, index_dtype=None, value_dtype=None):
        super().__init__(exc, size)
        _check_index_dtype(index_dtype)
        vt = _np_vt(value_dtype or (getattr(vals, "dtype", None) if not isinstance(vals, (list, tuple))
                                    else None) or config.DEFAULT_VALUE_DTYPE)
        if not (torch is not None and isinstance(row_idxs, torch.Tensor)):
            r = np.asarray(row_idxs, dtype=np.int64).reshape(-1)
            if r.size > 1 and np.any(np.diff(r) < 0):
                raise Unsupported("Coo entries must be sorted by row (use from_data)")
        self._ri = _to_device(exc, row_idxs, torch.int32)
        self._ci = _to_device(exc, col_idxs, torch.int32)
        self._v = _to_device(exc, vals, _torch_vt(vt))
        self._ws = None

    @classmethod
    def _from_device(cls, exc, size, ri, ci, v):
        obj = cls.__new__(cls)
        _Sparse.__init__(obj, exc, size)
        obj._ri, obj._ci, obj._v = ri, ci, v
        obj._ws = None
        return obj

    @property
    def nnz(self):
        return int(self._v.numel())

    @property
    def row_idxs(self):
        return DeviceView(self._ri)

    @property
    def col_idxs(self):
        return DeviceView(self._ci)

    @property
    def vals(self):
        return DeviceView(self._v)

    def _workspace(self):
        """carry buffers + the list of rows that hold no entry (prefilled)."""
        if self._ws is None:
            exc = self.exec
            nch = max(1, math.ceil(self.nnz / 128))  # covers both chunk sizes
            head = torch.empty(nch, dtype=self._v.dtype, device=exc.device)
            tail = torch.empty(nch, dtype=self._v.dtype, device=exc.device)
            crows = torch.empty(2 * nch, dtype=torch.int32, device=exc.device)  # per chunk (head, tail) rows
            n = self.size.rows
            rp = torch.empty(n + 1, dtype=torch.int32, device=exc.device)
            _lib.call("coo_to_csr_ptrs", self.nnz, n, ptr(self._ri), ptr(rp), exc.stream)
            flags = torch.empty(max(n, 1), dtype=torch.int32, device=exc.device)
            _lib.call("empty_row_flags", n, ptr(rp), ptr(flags), exc.stream)
            pos = _scan(exc, flags[:n])
            ne = int(pos[-1].item())
            empty = torch.empty(max(ne, 1), dtype=torch.int32, device=exc.device)
            _lib.call("compact_flags", n, ptr(flags), ptr(pos), ptr(empty), exc.stream)
            self._ws = (head, tail, empty, ne, crows)
        return self._ws

    def _launch_column(self, exc, suf, bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins,
                       prefill=True):
        head, tail, empty, ne, crows = self._workspace()
        if prefill and ne:
            _lib.call("rows_scale_" + suf, ne, ptr(empty), xp, xs, b_h, b_p, xin, xins, exc.stream)
        _lib.call("coo_spmv_" + suf, self.nnz, self.chunk, ptr(self._ri), ptr(self._ci), ptr(self._v),
                  bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins, ptr(head), ptr(tail), ptr(crows), exc.stream)

    def _to_csr(self, **kw):
        exc = self.exec
        n = self.size.rows
        rp = torch.empty(n + 1, dtype=torch.int32, device=exc.device)
        _lib.call("coo_to_csr_ptrs", self.nnz, n, ptr(self._ri), ptr(rp), exc.stream)
        return Csr._from_device(exc, self.size, rp, self._ci.clone(), self._v.clone(), **kw)

    @classmethod
    def _from_csr(cls, csr, exec=None, **_):
        exc = csr.exec
        ri = torch.empty(csr.nnz, dtype=torch.int32, device=exc.device)
        _lib.call("csr_to_coo_rows", csr.size.rows, ptr(csr._rp), ptr(ri), exc.stream)
        target = exec or exc
        return cls._from_device(target, csr.size, ri.to(target.device), csr._ci.clone().to(target.device),
                                csr._v.clone().to(target.device))


# ---------------------------------------------------------------------------
# Ell (no reference implementation)
# ---------------------------------------------------------------------------
def _ell_stride(n):
    return max(1, (n + 31) // 32 * 32)


class Ell(_Sparse):
    """ELLPACK: ``num_stored_elements_per_row`` slots per row, column-major
    with ``stride`` >= rows (rounded to 32 for aligned, coalesced columns);
    padding slots hold column -1 and value 0."""

    def __init__(self, exc, size, col_idxs, vals, num_stored_elements_per_row, stride=None,
                 value_dtype=None):
        super().__init__(exc, size)
        n = self.size.rows
        self.width = int(num_stored_elements_per_row)
        self.stride = int(stride if stride is not None else _ell_stride(n))
        if self.stride < n:
            raise DimensionMismatch("ell stride must be >= number of rows")
        vt = _np_vt(value_dtype or getattr(vals, "dtype", None) or config.DEFAULT_VALUE_DTYPE)
        self._ci = _to_device(exc, col_idxs, torch.int32).reshape(-1)
        self._v = _to_device(exc, vals, _torch_vt(vt)).reshape(-1)
        if self._ci.numel() != self.width * self.stride or self._v.numel() != self.width * self.stride:
            raise DimensionMismatch("ell arrays must hold width * stride entries")

    @classmethod
    def _from_device(cls, exc, size, ci, v, width, stride):
        obj = cls.__new__(cls)
        _Sparse.__init__(obj, exc, size)
        obj._ci, obj._v, obj.width, obj.stride = ci, v, int(width), int(stride)
        return obj

    @property
    def num_stored_elements_per_row(self):
        return self.width

    @property
    def col_idxs(self):
        return DeviceView(self._ci)

    @property
    def vals(self):
        return DeviceView(self._v)

    @property
    def num_stored_elements(self):
        return self.width * self.stride

    def _launch_column(self, exc, suf, bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins):
        _lib.call("ell_spmv_" + suf, self.size.rows, self.width, self.stride, ptr(self._ci), ptr(self._v),
                  bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins, exc.stream)

    def _row_lengths(self):
        n = self.size.rows
        lens = torch.empty(max(n, 1), dtype=torch.int32, device=self.exec.device)
        _lib.call("ell_row_lengths", n, self.width, self.stride, ptr(self._ci), ptr(lens), self.exec.stream)
        return lens[:n]

    def _to_csr(self, **kw):
        exc = self.exec
        n = self.size.rows
        rp = _scan(exc, self._row_lengths())
        nnz = int(rp[-1].item())
        ci = torch.empty(nnz, dtype=torch.int32, device=exc.device)
        v = torch.empty(nnz, dtype=self._v.dtype, device=exc.device)
        _lib.call("ell_to_csr_fill_" + _lib.suffix(self._v.dtype), n, self.width, self.stride,
                  ptr(self._ci), ptr(self._v), ptr(rp), ptr(ci), ptr(v), exc.stream)
        return Csr._from_device(exc, self.size, rp, ci, v, **kw)

    @classmethod
    def _from_csr(cls, csr, width=None, stride=None, exec=None, **_):
        exc = csr.exec
        n = csr.size.rows
        w = csr._row_stats() if width is None else int(width)
        st = _ell_stride(n) if stride is None else int(stride)
        ci = torch.empty(w * st, dtype=torch.int32, device=exc.device)
        v = torch.empty(w * st, dtype=csr._v.dtype, device=exc.device)
        _lib.call("csr_to_ell_" + _lib.suffix(csr._v.dtype), n, ptr(csr._rp), ptr(csr._ci), ptr(csr._v),
                  w, st, ptr(ci), ptr(v), exc.stream)
        target = exec or exc
        return cls._from_device(target, csr.size, ci.to(target.device), v.to(target.device), w, st)


# ---------------------------------------------------------------------------
# Sellp (no reference implementation)
# ---------------------------------------------------------------------------
SELLP_SLICE = 64


class Sellp(_Sparse):
    """Sliced ELLPACK: slices of ``slice_size`` rows, each column-major with
    its own length (max row length in the slice rounded up to
    ``stride_factor``); ``slice_sets`` is the exclusive prefix of lengths."""

    def __init__(self, exc, size, slice_lengths, slice_sets, col_idxs, vals, slice_size=SELLP_SLICE,
                 stride_factor=1, value_dtype=None):
        super().__init__(exc, size)
        self.slice_size = int(slice_size)
        self.stride_factor = int(stride_factor)
        vt = _np_vt(value_dtype or getattr(vals, "dtype", None) or config.DEFAULT_VALUE_DTYPE)
        self._sl = _to_device(exc, slice_lengths, torch.int32)
        self._ss = _to_device(exc, slice_sets, torch.int32)
        self._ci = _to_device(exc, col_idxs, torch.int32)
        self._v = _to_device(exc, vals, _torch_vt(vt))
        ns = math.ceil(self.size.rows / self.slice_size)
        if self._sl.numel() != ns or self._ss.numel() != ns + 1:
            raise DimensionMismatch("sellp: slice_lengths needs one entry per slice and "
                                    "slice_sets one more")

    @classmethod
    def _from_device(cls, exc, size, sl, ss, ci, v, slice_size, stride_factor):
        obj = cls.__new__(cls)
        _Sparse.__init__(obj, exc, size)
        obj._sl, obj._ss, obj._ci, obj._v = sl, ss, ci, v
        obj.slice_size, obj.stride_factor = int(slice_size), int(stride_factor)
        return obj

    @property
    def slice_lengths(self):
        return DeviceView(self._sl)

    @property
    def slice_sets(self):
        return DeviceView(self._ss)

    @property
    def col_idxs(self):
        return DeviceView(self._ci)

    @property
    def vals(self):
        return DeviceView(self._v)

    @property
    def num_stored_elements(self):
        return int(self._v.numel())

    def _launch_column(self, exc, suf, bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins):
        _lib.call("sellp_spmv_" + suf, self.size.rows, self.slice_size, ptr(self._sl), ptr(self._ss),
                  ptr(self._ci), ptr(self._v), bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins, exc.stream)

    def _to_csr(self, **kw):
        exc = self.exec
        n = self.size.rows
        lens = torch.empty(max(n, 1), dtype=torch.int32, device=exc.device)
        _lib.call("sellp_row_lengths", n, self.slice_size, ptr(self._sl), ptr(self._ss), ptr(self._ci),
                  ptr(lens), exc.stream)
        rp = _scan(exc, lens[:n])
        nnz = int(rp[-1].item())
        ci = torch.empty(nnz, dtype=torch.int32, device=exc.device)
        v = torch.empty(nnz, dtype=self._v.dtype, device=exc.device)
        _lib.call("sellp_to_csr_fill_" + _lib.suffix(self._v.dtype), n, self.slice_size, ptr(self._sl),
                  ptr(self._ss), ptr(self._ci), ptr(self._v), ptr(rp), ptr(ci), ptr(v), exc.stream)
        return Csr._from_device(exc, self.size, rp, ci, v, **kw)

    @classmethod
    def _from_csr(cls, csr, slice_size=SELLP_SLICE, stride_factor=1, exec=None, **_):
        exc = csr.exec
        n = csr.size.rows
        ns = math.ceil(n / slice_size)
        sl = torch.empty(max(ns, 1), dtype=torch.int32, device=exc.device)
        _lib.call("sellp_slice_lengths", n, ptr(csr._rp), slice_size, stride_factor, ptr(sl), exc.stream)
        sl = sl[:ns]
        ss = _scan(exc, sl)
        total = int(ss[-1].item())
        ci = torch.empty(total * slice_size, dtype=torch.int32, device=exc.device)
        v = torch.empty(total * slice_size, dtype=csr._v.dtype, device=exc.device)
        _lib.call("csr_to_sellp_" + _lib.suffix(csr._v.dtype), n, ptr(csr._rp), ptr(csr._ci), ptr(csr._v),
                  slice_size, ptr(sl), ptr(ss), ptr(ci), ptr(v), exc.stream)
        target = exec or exc
        return cls._from_device(target, csr.size, sl.to(target.device), ss.to(target.device),
                                ci.to(target.device), v.to(target.device), slice_size, stride_factor)


# ---------------------------------------------------------------------------
# Hybrid = Ell + Coo (no reference implementation)
# ---------------------------------------------------------------------------
class HybridStrategy:
    """Chooses the Ell width from the row-length histogram (host decision on
    a device-computed histogram)."""

    def width(self, hist, n, vt_bytes):
        raise NotImplementedError


class column_limit(HybridStrategy):
    def __init__(self, num_columns=0):
        self.num_columns = int(num_columns)

    def width(self, hist, n, vt_bytes):
        return self.num_columns


class imbalance_limit(HybridStrategy):
    """Width = row length at quantile ``percent`` of the sorted row lengths."""

    def __init__(self, percent=0.8):
        if not 0.0 <= percent <= 1.0:
            raise ValueError("percent must lie in [0, 1]")
        self.percent = float(percent)

    def width(self, hist, n, vt_bytes):
        if n == 0:
            return 0
        rank = min(n - 1, int(math.floor(self.percent * n)))
        cum = np.cumsum(hist)
        return int(np.searchsorted(cum, rank + 1))


class minimal_storage_limit(HybridStrategy):
    """Width minimising Ell bytes n*w*(VT+4) + Coo bytes overflow(w)*(VT+8)."""

    def width(self, hist, n, vt_bytes):
        if n == 0:
            return 0
        hist = np.asarray(hist, dtype=np.float64)
        lens = np.arange(hist.size, dtype=np.float64)
        cum = np.cumsum(hist)
        total = float((hist * lens).sum())
        # entries beyond width w: over[w+1] = over[w] - #(rows longer than w)
        over = np.empty(hist.size)
        over[0] = total
        over[1:] = total - np.cumsum(n - cum[:-1])
        cost = n * lens * (vt_bytes + 4) + over * (vt_bytes + 8)
        return int(np.argmin(cost))


class automatic(imbalance_limit):
    """Default split: the row length at the 80th percentile (Ginkgo's
    imbalance-limit rule). On the C3 power law this is width 16 -- 371.9 us
    -- where the storage-minimising width 6 takes 421.2 us (the Ell pass is
    the cheaper one per entry even with its padding; widths 0-24 in
    profiles/r03_hybrid_width.txt); on the stencils every row fits (all Ell)."""

    def __init__(self):
        super().__init__(0.8)


class Hybrid(_Sparse):
    """Ell part (first ``width`` entries of each row) + Coo part (the rest)."""

    def __init__(self, exc, size, ell, coo, strategy=None):
        super().__init__(exc, size)
        self.ell, self.coo = ell, coo
        self.hybrid_strategy = strategy or automatic()

    @property
    def _v(self):
        return self.ell._v

    @property
    def nnz(self):
        return self.coo.nnz + int((self.ell._ci >= 0).sum().item())

    def _launch_column(self, exc, suf, bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins):
        self.ell._launch_column(exc, suf, bp, bs, xp, xs, a_h, a_p, b_h, b_p, xin, xins)
        if self.coo.nnz:
            # accumulate: x += alpha * A_coo b (rows absent from the Coo part untouched)
            self.coo._launch_column(exc, suf, bp, bs, xp, xs, a_h, a_p, 1.0, 0, xp, xs, prefill=False)

    def _to_csr(self, **kw):
        exc = self.exec
        n = self.size.rows
        ell_len = self.ell._row_lengths()
        crp = torch.empty(n + 1, dtype=torch.int32, device=exc.device)
        _lib.call("coo_to_csr_ptrs", self.coo.nnz, n, ptr(self.coo._ri), ptr(crp), exc.stream)
        lens = ell_len.clone()
        _lib.call("add_csr_lengths", n, ptr(crp), ptr(lens), exc.stream)
        rp = _scan(exc, lens)
        nnz = int(rp[-1].item())
        ci = torch.empty(nnz, dtype=torch.int32, device=exc.device)
        v = torch.empty(nnz, dtype=self._v.dtype, device=exc.device)
        suf = _lib.suffix(self._v.dtype)
        _lib.call("ell_to_csr_fill_" + suf, n, self.ell.width, self.ell.stride, ptr(self.ell._ci),
                  ptr(self.ell._v), ptr(rp), ptr(ci), ptr(v), exc.stream)
        _lib.call("hybrid_coo_append_" + suf, n, ptr(rp), ptr(ell_len), ptr(crp), ptr(self.coo._ci),
                  ptr(self.coo._v), ptr(ci), ptr(v), exc.stream)
        return Csr._from_device(exc, self.size, rp, ci, v, **kw)

    @classmethod
    def _from_csr(cls, csr, strategy=None, exec=None, **_):
        exc = csr.exec
        strategy = strategy or automatic()
        n = csr.size.rows
        if isinstance(strategy, column_limit):
            w = strategy.num_columns
        else:
            nbins = max(2, min(csr._row_stats() + 1, 1 << 16))
            hist = torch.empty(nbins, dtype=torch.int64, device=exc.device)
            _lib.call("length_histogram", n, ptr(csr._rp), nbins, ptr(hist), exc.stream)
            w = strategy.width(hist.cpu().numpy().astype(np.float64), n, csr._v.element_size())
        ell = Ell._from_csr(csr, width=w)
        cnt = torch.empty(max(n, 1), dtype=torch.int32, device=exc.device)
        _lib.call("hybrid_overflow_counts", n, ptr(csr._rp), w, ptr(cnt), exc.stream)
        offs = _scan(exc, cnt[:n])
        nc = int(offs[-1].item())
        crow = torch.empty(nc, dtype=torch.int32, device=exc.device)
        cci = torch.empty(nc, dtype=torch.int32, device=exc.device)
        cv = torch.empty(nc, dtype=csr._v.dtype, device=exc.device)
        _lib.call("csr_to_hybrid_coo_" + _lib.suffix(csr._v.dtype), n, ptr(csr._rp), ptr(csr._ci),
                  ptr(csr._v), w, ptr(offs), ptr(crow), ptr(cci), ptr(cv), exc.stream)
        coo = Coo._from_device(exc, csr.size, crow, cci, cv)
        out = cls(exc, csr.size, ell, coo, strategy)
        if exec is not None and exec is not exc:
            return convert(out, Hybrid, exec=exec)
        return out


# ---------------------------------------------------------------------------
# StencilMatrix (src/formats.py:268-298): matrix-free tridiagonal operator
# ---------------------------------------------------------------------------
class StencilMatrix(LinOp):
    """Matrix-free 3-point stencil operator (tridiagonal action) on the
    device; converts to Csr only, like the reference."""

    def __init__(self, exc, n, left, center, right, value_dtype=None):
        _require_cuda(exc)
        super().__init__(exc, Dim2(n, n))
        vt = _np_vt(value_dtype or config.DEFAULT_VALUE_DTYPE)
        self.coefficients = np.asarray([left, center, right], dtype=vt)

    def _apply_impl(self, b, x):
        bt, xt = b.values, x.values
        l, c, r = (float(v) for v in self.coefficients)
        _lib.call("stencil3_apply_" + _lib.suffix(xt.dtype), xt.shape[0], xt.shape[1], l, c, r, ptr(bt),
                  bt.stride(0), ptr(xt), xt.stride(0), self.exec.stream)

    def to_data(self):
        from .problems import tridiagonal

        left, center, right = (float(v) for v in self.coefficients)
        n = self.size.rows
        i = np.arange(n, dtype=np.int64)
        cols = np.stack([i - 1, i, i + 1], axis=1)
        vals = np.broadcast_to(np.array([left, center, right]), (n, 3))
        keep = np.stack([i > 0, np.ones(n, bool), i < n - 1], axis=1)
        return MatrixData(self.size, np.repeat(i, 3).reshape(n, 3)[keep], cols[keep], vals[keep])

    def convert_to(self, kind, **kw):
        if kind is Csr or (isinstance(kind, str) and kind.lower() == "csr"):
            return Csr.from_data(self.exec, self.to_data(), value_dtype=self.coefficients.dtype)
        raise Unsupported("stencil matrices only convert to CSR")

    def clone_to(self, target):
        return StencilMatrix(target, self.size.rows, *map(float, self.coefficients),
                             value_dtype=self.coefficients.dtype)


# ---------------------------------------------------------------------------
# conversions (src/formats.py:301-329)
# ---------------------------------------------------------------------------
_FORMAT_NAMES = {"dense": Dense, "csr": Csr, "coo": Coo, "ell": Ell, "sellp": Sellp, "hybrid": Hybrid}


def _resolve(target):
    if isinstance(target, str):
        key = target.lower()
        named = {"csr_classical": "classical", "csr_lb": "load_balance",
                 "csr_load_balance": "load_balance", "csr_stream": "stream"}
        if key in named:
            return Csr, {"strategy": named[key]}
        if key == "csr_pipe":
            return Csr, {"strategy": "stream", "stream_impl": "tma"}
        try:
            return _FORMAT_NAMES[key], {}
        except KeyError:
            raise Unsupported(f"unknown format {target!r}") from None
    if target in _FORMAT_NAMES.values():
        return target, {}
    raise Unsupported(f"no conversion to {target}")


def convert(a, target, **params):
    """Value-equivalent copy of ``a`` in another format (device-side, Csr hub).

    Dense -> sparse drops explicit zeros (as in the reference). Extra keyword
    parameters reach the target constructor (``strategy``, ``width``,
    ``slice_size``, ``stride_factor``)."""
    if isinstance(a, StencilMatrix):  # assembles to Csr only (src/formats.py:283-298)
        return a.convert_to(target, **params)
    cls, extra = _resolve(target)
    params = {**extra, **params}
    impl = params.pop("stream_impl", None)
    csr_kw = {"strategy": params.pop("strategy")} if cls is Csr and "strategy" in params else {}
    if isinstance(a, Csr) and cls is Csr:
        out = Csr._from_csr(a, **csr_kw, **params)
    else:
        csr = a._to_csr(**csr_kw)
        if cls is Csr:
            out = csr if "exec" not in params else Csr._from_csr(csr, **params)
        else:
            return cls._from_csr(csr, **params)
    if impl is not None:
        out._stream_impl = impl
    return out


def matrix_from_data(exc, data, fmt="csr", **params):
    cls, extra = _resolve(fmt)
    if cls is Dense:
        return Dense(exc, data.to_dense_array(), value_dtype=params.get("value_dtype"))
    csr = Csr._from_host_data(exc, data, params.pop("value_dtype", None))
    if cls is Csr:
        if extra or params:
            csr.set_strategy((extra or params).get("strategy", "automatic"))
        return csr
    return cls._from_csr(csr, **params)
