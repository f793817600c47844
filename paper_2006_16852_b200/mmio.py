"""Matrix Market exchange format (reference src/mmio.py:1-150).

Reading runs the native parser of libb200sp (csrc/mmio.cu: a two-pass,
multi-threaded parse of the file image with the reference's accepted subset,
messages and 1-based error line numbers); the triples then feed the device
assembly (``matrix_from_data`` canonicalises on the GPU). Writing produces the
reference's canonical text byte for byte (coordinate / real / general,
1-based, sorted, ``repr`` of every value), so ``write(read(f))`` is
byte-identical on canonical files.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .base import Dim2
from .errors import ParseError, Unsupported
from .formats import MatrixData

_WRITE_HEADER = "%%MatrixMarket matrix coordinate real general"


def _call(name, *args, err_line=None):
    _lib._load()
    rc = _lib._funcs[name](*args)
    if rc != 0:
        msg = _lib._funcs["last_error"]().decode(errors="replace")
        if rc == 4:
            raise Unsupported(msg)
        line = int(err_line.value) if err_line is not None and err_line.value else None
        raise ParseError(msg, line=line)


def read_matrix_market_bytes(buf, threads=0) -> MatrixData:
    """Parse a Matrix Market file image (bytes) into coordinate data."""
    if isinstance(buf, str):
        buf = buf.encode("ascii")
    buf = bytes(buf)
    n = len(buf)
    cbuf = ctypes.c_char_p(buf)
    info = (ctypes.c_int64 * 7)()
    err = ctypes.c_int64(0)
    _call("mm_header", cbuf, n, info, ctypes.byref(err), err_line=err)
    count = ctypes.c_int64(0)
    _call("mm_count", cbuf, n, info, int(threads), ctypes.byref(count))
    cap = max(int(count.value), 0)
    rows = np.empty(cap, dtype=np.int64)
    cols = np.empty(cap, dtype=np.int64)
    vals = np.empty(cap, dtype=np.float64)
    got = ctypes.c_int64(0)
    _call("mm_parse", cbuf, n, info, int(threads), rows.ctypes.data, cols.ctypes.data, vals.ctypes.data, cap,
          ctypes.byref(got), ctypes.byref(err), err_line=err)
    nr, nc = int(info[2]), int(info[3])
    if info[0]:  # array: column-major values -> dense triples (src/mmio.py:114-126)
        dense = vals[:nr * nc].reshape((nc, nr)).T
        return MatrixData.from_dense_array(dense, drop_zeros=False)
    k = int(got.value)
    return MatrixData(Dim2(nr, nc), rows[:k], cols[:k], vals[:k])


def read_matrix_market(stream) -> MatrixData:
    """Parse a Matrix Market text stream (src/mmio.py:38-78)."""
    return read_matrix_market_bytes(stream.read())


def read_matrix_market_file(path, threads=0) -> MatrixData:
    with open(path, "rb") as fh:
        return read_matrix_market_bytes(fh.read(), threads)


def write_matrix_market(stream, data: MatrixData):
    """Coordinate / real / general with 1-based sorted entries (src/mmio.py:129-135)."""
    data = data.canonicalize()
    stream.write(_WRITE_HEADER + "\n")
    stream.write(f"{data.size.rows} {data.size.cols} {data.nnz}\n")
    stream.write("".join(f"{r} {c} {v!r}\n" for r, c, v in
                         zip((data.rows + 1).tolist(), (data.cols + 1).tolist(), data.vals.tolist())))


def write_matrix_market_array(stream, dense_array):
    """Dense matrix in array / real / general form, column-major (src/mmio.py:138-144)."""
    arr = np.asarray(dense_array, dtype=np.float64)
    stream.write("%%MatrixMarket matrix array real general\n")
    stream.write(f"{arr.shape[0]} {arr.shape[1]}\n")
    stream.write("".join(f"{v!r}\n" for v in arr.T.reshape(-1).tolist()))
