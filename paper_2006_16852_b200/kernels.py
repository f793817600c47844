"""Operations (one ``cuda`` variant each) behind the formats and Dense.

Each class mirrors one reference kernel (src/kernels.py) and launches the
corresponding sm_100a kernel of libb200sp through ``_lib.call``. Vectors are
Dense (n, m) blocks; SpMV launches once per right-hand-side column (m = 1 on
every benchmarked configuration).
"""

from __future__ import annotations

from . import _lib
from .executor import Operation, ptr


def _isz(t):
    return t.element_size()


def coef_column(alpha, j, dtype_suffix):
    """(host value, device pointer) of a scalar coefficient for column j.

    Numbers stay on the host; a 1x1 / 1xm Dense on the device is read by the
    kernel through its pointer (no host sync); a host Dense is read directly.
    """
    if alpha is None:
        return 0.0, 0
    if isinstance(alpha, (int, float)):
        return float(alpha), 0
    from .formats import Dense

    if isinstance(alpha, Dense):
        col = j if alpha.size.cols > 1 else 0
        if alpha.on_device:
            t = alpha.values
            return 0.0, t.data_ptr() + col * t.stride(1) * _isz(t)
        return float(alpha.values[0, col]), 0
    return float(alpha), 0


class FillOp(Operation):
    name = "fill"

    def __init__(self, x, value):
        self.x, self.value = x, value

    def cuda(self, exc):
        t = self.x.values
        _lib.call("fill_" + _lib.suffix(t.dtype), t.shape[0], t.shape[1], ptr(t), t.stride(0),
                  float(self.value), exc.stream)

    def host(self, exc):
        self.x.values[...] = self.value


class CopyOp(Operation):
    """dst <- src (same shape); cross-executor copies are migrations."""

    name = "copy"

    def __init__(self, src, dst):
        self.src, self.dst = src, dst

    def cuda(self, exc):
        s, d = self.src.values, self.dst.values
        _lib.call("copy_" + _lib.suffix(d.dtype), d.shape[0], d.shape[1], ptr(s), s.stride(0),
                  ptr(d), d.stride(0), exc.stream)

    def host(self, exc):
        self.dst.values[...] = self.src.values


class ScaleOp(Operation):
    name = "scale"

    def __init__(self, alpha, x):
        self.alpha, self.x = alpha, x

    def cuda(self, exc):
        t = self.x.values
        suf = _lib.suffix(t.dtype)
        a, ap = _vector_coef(self.alpha, t)
        _lib.call("scale_" + suf, t.shape[0], t.shape[1], a, ap, ptr(t), t.stride(0), exc.stream)


class AddScaledOp(Operation):
    """y <- y + alpha * x."""

    name = "add_scaled"

    def __init__(self, alpha, x, y):
        self.alpha, self.x, self.y = alpha, x, y

    def cuda(self, exc):
        x, y = self.x.values, self.y.values
        suf = _lib.suffix(y.dtype)
        a, ap = _vector_coef(self.alpha, y)
        _lib.call("add_scaled_" + suf, y.shape[0], y.shape[1], a, ap, ptr(x), x.stride(0), ptr(y),
                  y.stride(0), exc.stream)


def _vector_coef(alpha, t):
    """Per-column coefficient for the BLAS-1 kernels: (host, dev ptr to m contiguous)."""
    from .formats import Dense

    if isinstance(alpha, Dense):
        if alpha.on_device:
            a = alpha.values
            if a.shape[1] == t.shape[1] and a.stride(1) == 1:
                return 0.0, a.data_ptr()
            if a.shape[1] == 1 and t.shape[1] == 1:
                return 0.0, a.data_ptr()
            # broadcast a 1x1 coefficient over m columns
            return 0.0, a.expand(1, t.shape[1]).contiguous().data_ptr()
        vals = alpha.values
        if vals.shape[1] == 1:
            return float(vals[0, 0]), 0
        alpha = vals
    if hasattr(alpha, "shape"):  # host (1, m) array
        import torch

        dev = torch.as_tensor(alpha, dtype=t.dtype).reshape(1, -1).to(t.device)
        if dev.shape[1] == 1:
            return float(dev[0, 0]), 0
        return 0.0, dev.contiguous().data_ptr()
    return float(alpha), 0


class DotOp(Operation):
    """out[0, j] <- sum_i x[i, j] y[i, j] (deterministic two-level reduction)."""

    name = "dot"

    def __init__(self, x, y, out, norm=False):
        self.x, self.y, self.out, self.norm = x, y, out, norm

    def cuda(self, exc):
        x, y, o = self.x.values, self.y.values, self.out.values
        suf = _lib.suffix(x.dtype)
        part, counter = exc.reduce_workspace(x.dtype)
        if o.stride(1) != 1:
            raise ValueError("dot output must be contiguous")
        if self.norm:
            _lib.call("norm2_" + suf, x.shape[0], x.shape[1], ptr(x), x.stride(0), ptr(o),
                      ptr(part), ptr(counter), exc.stream)
        else:
            _lib.call("dot_" + suf, x.shape[0], x.shape[1], ptr(x), x.stride(0), ptr(y),
                      y.stride(0), ptr(o), ptr(part), ptr(counter), exc.stream)


class SpmvOp(Operation):
    """x = alpha * A b + beta * x_in for any device format (one launch per
    column; the format object supplies ``_launch_column``)."""

    def __init__(self, mat, b, x, alpha=1.0, beta=None, x_in=None):
        self.mat, self.b, self.x = mat, b, x
        self.alpha, self.beta, self.x_in = alpha, beta, x_in
        self.name = type(mat).__name__.lower() + "_spmv"

    def cuda(self, exc):
        b, x = self.b.values, self.x.values
        xin = self.x_in.values if self.x_in is not None else None
        suf = _lib.suffix(x.dtype)
        isz = _isz(x)
        for j in range(x.shape[1]):
            a_h, a_p = coef_column(self.alpha, j, suf)
            b_h, b_p = coef_column(self.beta, j, suf) if xin is not None else (0.0, 0)
            self.mat._launch_column(
                exc, suf,
                b.data_ptr() + j * b.stride(1) * isz, b.stride(0),
                x.data_ptr() + j * x.stride(1) * isz, x.stride(0),
                a_h, a_p, b_h, b_p,
                0 if xin is None else xin.data_ptr() + j * xin.stride(1) * isz,
                0 if xin is None else xin.stride(0))
