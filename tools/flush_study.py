"""How the L2 flush between timed steps changes C2 SpMV times.

A write-only flush (fill of a 256 MiB buffer) leaves ~L2-size dirty lines
that are written back to HBM *inside* the next timed kernel; a write + read
flush leaves L2 clean and equally cold for the matrix. Also times a pure
read stream of the same byte count (dot of two 44.4M-element vectors) as
the read roofline the SpMV kernels can reach.

    python tools/flush_study.py [--reps 20]
"""
import argparse
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2006_16852_b200 as b2  # noqa: E402
from bench import bytes_format, peaks  # noqa: E402
from paper_2006_16852_b200 import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--dtype", default="float64")
args = ap.parse_args()

exc = b2.CudaExecutor(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
peak, _ = peaks()


def do_flush(mode):
    if mode in ("write", "write+read"):
        flush.fill_(1)
    if mode == "write+read":
        flush.view(torch.int64).sum()  # evicts the dirty lines outside the timed region


def timeit(fn, mode):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
    for s, e in ev:
        do_flush(mode)
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in ev) * 1e-3


vt = 8 if args.dtype == "float64" else 4
a = problems.stencil(exc, "27pt", 128, value_dtype=args.dtype)
n = a.size.rows
b = b2.Dense(exc, np.random.default_rng(0).standard_normal((n, 1)), value_dtype=args.dtype)
x = b2.Dense.zeros(exc, n, 1, value_dtype=args.dtype)
modes = ("write", "write+read", "none")
print(f"C2 27-pt 128^3 {args.dtype}; frac vs {peak} GB/s")
for fmt in ("csr", "csr_lb", "coo", "ell", "sellp", "hybrid"):
    m = b2.convert(a, fmt)
    by = bytes_format(m, vt)
    row = []
    for mode in modes:
        t = timeit(lambda: m.apply(b, x), mode)
        row.append(f"{mode}: {t * 1e6:7.1f} us {by / t / 1e9 / peak:.3f}")
    print(f"{fmt:8s} " + " | ".join(row))
    del m
    torch.cuda.empty_cache()

# pure read stream of the Csr byte count
by = bytes_format(b2.convert(a, "csr"), vt)
k = by // 16
u = b2.Dense.zeros(exc, k, 1)
w = b2.Dense.zeros(exc, k, 1)
out = b2.Dense.zeros(exc, 1, 1)
for mode in modes:
    t = timeit(lambda: u.compute_dot(w, out), mode)
    print(f"dot read stream {by / 1e6:.0f} MB {mode}: {t * 1e6:7.1f} us {by / t / 1e9:7.1f} GB/s "
          f"{by / t / 1e9 / peak:.3f}")
cp_src = torch.empty(by // 2, dtype=torch.uint8, device="cuda")
cp_dst = torch.empty_like(cp_src)
for mode in modes:
    t = timeit(lambda: cp_dst.copy_(cp_src), mode)
    print(f"torch copy {by / 2e6:.0f}+{by / 2e6:.0f} MB {mode}: {t * 1e6:7.1f} us {by / t / 1e9:7.1f} GB/s")
