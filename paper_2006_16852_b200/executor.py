"""Executors: memory arenas plus kernel dispatch (the plugin point).

The reference routes every kernel through ``Executor.run(op)`` ->
``_dispatch`` -> ``op.<kind>(exc)`` (src/executor.py:95-154) and adds a
backend as "a new Executor subclass plus a per-kernel Operation variant"
(PAPER.md:1537-1555). This module is that backend:

* ``CudaExecutor`` -- one B200; ``_dispatch`` calls ``op.cuda(self)``, which
  launches a hand-written sm_100a kernel through the C ABI (``_lib``) on the
  executor's current CUDA stream. A missing variant raises
  KernelNotImplemented exactly like the reference (src/executor.py:85-89).
* ``HostExecutor`` -- the ``master`` arena: host memory only (pinned when a
  GPU is present) used for interchange and host<->device migration. It runs
  no numeric kernels: there is no CPU fallback on this path.

Device buffers are torch tensors (plumbing only: allocation, streams, copies).
"""

from __future__ import annotations

from enum import Enum

import numpy as np

from . import config
from .errors import KernelNotImplemented, OpalgError
from .loggers import EventKind, Loggable

try:  # torch is the device-memory / stream plumbing
    import torch
except Exception:  # pragma: no cover - torch is part of the image
    torch = None


class ExecutorKind(Enum):
    CUDA = "cuda"
    HOST = "host"


class Operation:
    """A kernel with one variant per executor kind (src/executor.py:74-92).

    ``cuda(exc)`` launches the sm_100a kernel; ``host(exc)`` exists only for
    pure memory operations (copy/fill on host arenas).
    """

    name = "operation"

    def cuda(self, exc):
        raise KernelNotImplemented(f"{self.name}: no cuda kernel")

    def host(self, exc):
        raise KernelNotImplemented(
            f"{self.name}: host executors run no numeric kernels (no CPU fallback)")


class Executor(Loggable):
    kind: ExecutorKind

    @property
    def master(self):
        return self

    def run(self, op):
        """Execute ``op`` (stream-ordered; observably synchronous: every host
        read synchronises)."""
        self._log(EventKind.OPERATION_LAUNCHED, {"op": op.name})
        self._dispatch(op)
        self._log(EventKind.OPERATION_COMPLETED, {"op": op.name})

    def _dispatch(self, op):
        raise NotImplementedError

    # -- allocation ----------------------------------------------------
    def alloc(self, shape, dtype):
        raise NotImplementedError

    def zeros(self, shape, dtype):
        raise NotImplementedError


def _np_dtype(dtype):
    if torch is not None and isinstance(dtype, torch.dtype):
        return {torch.float64: np.dtype("float64"), torch.float32: np.dtype("float32"),
                torch.int32: np.dtype("int32"), torch.int64: np.dtype("int64"),
                torch.uint8: np.dtype("uint8")}[dtype]
    return np.dtype(dtype)


def _torch_dtype(dtype):
    if torch is not None and isinstance(dtype, torch.dtype):
        return dtype
    return {"float64": torch.float64, "float32": torch.float32, "int32": torch.int32,
            "int64": torch.int64, "uint8": torch.uint8, "uint32": torch.int32,
            "bool": torch.bool}[np.dtype(dtype).name]


class HostExecutor(Executor):
    """Host memory arena (the CUDA executor's ``master``). Allocations are
    numpy arrays backed by pinned memory when a GPU is visible, so
    host<->device migrations run at full PCIe/NVLink-C2C speed."""

    kind = ExecutorKind.HOST

    def __init__(self, pinned=None):
        super().__init__()
        if pinned is None:
            pinned = torch is not None and torch.cuda.is_available()
        self.pinned = bool(pinned)

    def _dispatch(self, op):
        op.host(self)

    def alloc(self, shape, dtype):
        shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        if self.pinned:
            t = torch.empty(shape, dtype=_torch_dtype(dtype), pin_memory=True)
            arr = t.numpy()
        else:
            arr = np.empty(shape, dtype=_np_dtype(dtype))
        self._log(EventKind.ALLOCATION_COMPLETED, {"executor": self.uid, "bytes": arr.nbytes})
        return arr

    def zeros(self, shape, dtype):
        a = self.alloc(shape, dtype)
        a[...] = 0
        return a

    def __repr__(self):
        return f"HostExecutor(pinned={self.pinned})"


class CudaExecutor(Executor):
    """One CUDA device. Immutable and shareable; launches go to the device's
    *current* torch stream, so the executor composes with
    ``torch.cuda.stream(...)`` and CUDA-graph capture."""

    kind = ExecutorKind.CUDA

    def __init__(self, device_id=None, master=None):
        super().__init__()
        if torch is None or not torch.cuda.is_available():
            raise OpalgError("CudaExecutor needs a CUDA device (none visible)")
        from . import _lib

        _lib._load()  # fail loudly now if the extension is missing
        self.device_id = config.DEFAULT_DEVICE if device_id is None else int(device_id)
        self.device = torch.device("cuda", self.device_id)
        self._master = master if master is not None else HostExecutor()
        self._ws = {}

    @property
    def master(self):
        return self._master

    def _dispatch(self, op):
        with torch.cuda.device(self.device):
            op.cuda(self)

    @property
    def stream(self):
        """Raw cudaStream_t of the current stream (passed to the C ABI)."""
        return torch.cuda.current_stream(self.device).cuda_stream

    def alloc(self, shape, dtype):
        t = torch.empty(shape, dtype=_torch_dtype(dtype), device=self.device)
        self._log(EventKind.ALLOCATION_COMPLETED,
                  {"executor": self.uid, "bytes": t.numel() * t.element_size()})
        return t

    def zeros(self, shape, dtype):
        return torch.zeros(shape, dtype=_torch_dtype(dtype), device=self.device)

    def synchronize(self):
        torch.cuda.synchronize(self.device)

    def reduce_workspace(self, dtype):
        """(partials, counter) scratch for the deterministic dot/norm kernels.
        The counter self-resets, so one workspace per dtype serves every call
        on this executor's stream order."""
        from . import _lib

        key = ("red", str(dtype))
        ws = self._ws.get(key)
        if ws is None:
            n = int(_lib.query("reduce_workspace_elems"))
            ws = (torch.empty(n, dtype=_torch_dtype(dtype), device=self.device),
                  torch.zeros(1, dtype=torch.int32, device=self.device))
            self._ws[key] = ws
        return ws

    def __repr__(self):
        return f"CudaExecutor(device={self.device_id})"


def create_executor(kind="cuda", device_id=None, **_):
    """Build an executor from an ExecutorKind or its name (src/executor.py:253-267)."""
    if isinstance(kind, str):
        try:
            kind = ExecutorKind(kind)
        except ValueError:
            raise OpalgError(f"unknown executor kind: {kind!r} (this backend provides "
                             "'cuda' and the host arena 'host')") from None
    if kind is ExecutorKind.CUDA:
        return CudaExecutor(device_id)
    if kind is ExecutorKind.HOST:
        return HostExecutor()
    raise OpalgError(f"unknown executor kind: {kind}")


def ptr(t):
    """Raw device pointer of a tensor (0 for None)."""
    return 0 if t is None else t.data_ptr()


class DeviceView:
    """Host-side, numpy-compatible view of a device tensor.

    Reading (``np.asarray(view)``, indexing, arithmetic) synchronises and
    copies to the host; item assignment writes through to the device. This
    keeps reference-style code that touches ``.data`` working unchanged; the
    hot path never goes through it.
    """

    __slots__ = ("_t",)
    __array_priority__ = 100

    def __init__(self, tensor):
        self._t = tensor

    @property
    def tensor(self):
        return self._t

    def numpy(self):
        return self._t.detach().cpu().numpy()

    def __array__(self, dtype=None, copy=None):
        a = self.numpy()
        return a if dtype is None else a.astype(dtype)

    @property
    def shape(self):
        return tuple(self._t.shape)

    @property
    def dtype(self):
        return _np_dtype(self._t.dtype)

    @property
    def size(self):
        return int(self._t.numel())

    @property
    def ndim(self):
        return self._t.dim()

    @property
    def itemsize(self):
        return self._t.element_size()

    @property
    def nbytes(self):
        return self.size * self.itemsize

    @property
    def strides(self):
        return tuple(s * self.itemsize for s in self._t.stride())

    def __len__(self):
        return int(self._t.shape[0])

    def __getitem__(self, idx):
        return self.numpy()[idx]

    def __setitem__(self, idx, value):
        host = self.numpy()
        host[idx] = value
        self._t.copy_(torch.from_numpy(np.ascontiguousarray(host)).to(self._t.device))

    def copy(self):
        return self.numpy().copy()

    def astype(self, dtype, copy=True):
        return self.numpy().astype(dtype)

    def __getattr__(self, name):
        return getattr(self.numpy(), name)

    def __repr__(self):
        return f"DeviceView({self.numpy()!r})"

    def __iter__(self):
        return iter(self.numpy())

    def __eq__(self, other):
        return self.numpy() == np.asarray(other)

    def __ne__(self, other):
        return self.numpy() != np.asarray(other)

    def __bool__(self):
        return bool(self.numpy())

    def _binop(name):
        def f(self, other):
            return getattr(self.numpy(), name)(np.asarray(other))
        return f

    for _n in ("__add__", "__radd__", "__sub__", "__rsub__", "__mul__", "__rmul__",
               "__truediv__", "__rtruediv__", "__matmul__", "__rmatmul__", "__lt__",
               "__le__", "__gt__", "__ge__", "__pow__", "__and__", "__or__"):
        locals()[_n] = _binop(_n)
    del _n, _binop

    def __neg__(self):
        return -self.numpy()

    def __abs__(self):
        return abs(self.numpy())


class StorageMode(Enum):
    OWNING = "owning"
    VIEW = "view"


class Array:
    """Fixed-size buffer resident on one executor (src/executor.py:270-334):
    a torch tensor on a CudaExecutor, a (pinned) ndarray on the host arena.
    Owning arrays hold their own storage; views alias caller memory and never
    release it; ``copy_to`` is always a deep, owning copy."""

    def __init__(self, exc, size=None, data=None, mode=StorageMode.OWNING, dtype=None):
        self.exec = exc
        self.mode = mode
        dt = np.dtype(dtype or (getattr(data, "dtype", None) if data is not None else None)
                      or config.DEFAULT_VALUE_DTYPE)
        if data is not None:
            if isinstance(exc, CudaExecutor):
                src = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.asarray(data, dtype=dt))
                t = src.to(exc.device)
                # owning: never alias the caller's buffer
                self.data = t.clone() if mode is StorageMode.OWNING and t.data_ptr() == src.data_ptr() else t
            else:
                arr = np.asarray(data, dtype=dt)
                self.data = arr.copy() if mode is StorageMode.OWNING else arr
        else:
            self.data = (torch.empty(int(size), dtype=_torch_dtype(dt), device=exc.device)
                         if isinstance(exc, CudaExecutor) else exc.alloc(int(size), dt))

    @classmethod
    def view(cls, exc, size, buffer):
        """Non-owning view over the first ``size`` elements of ``buffer``."""
        buf = buffer.reshape(-1) if hasattr(buffer, "reshape") else np.asarray(buffer).reshape(-1)
        n = buf.numel() if isinstance(buf, torch.Tensor) else buf.size
        if size > n:
            raise OpalgError("view exceeds the underlying buffer")
        obj = cls.__new__(cls)
        obj.exec, obj.mode, obj.data = exc, StorageMode.VIEW, buf[:size]
        return obj

    def __len__(self):
        return int(self.data.numel() if isinstance(self.data, torch.Tensor) else self.data.size)

    def copy_to(self, target):
        """Deep copy onto ``target`` (always owning; the source is unchanged)."""
        out = Array(target, size=len(self), dtype=str(self.data.dtype).replace("torch.", ""))
        if isinstance(out.data, torch.Tensor):
            out.data.copy_(torch.as_tensor(self.data).to(out.data.device))
        else:
            out.data[...] = self.data.cpu().numpy() if isinstance(self.data, torch.Tensor) else self.data
        return out
