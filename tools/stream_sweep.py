"""Sweep CSR-stream (shape, chunk) variants on a stencil (CUDA events, L2 flushed).

    python tools/stream_sweep.py [--matrix 27pt] [--grid 128] [--dtype float64]
"""
import argparse
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2006_16852_b200 as b2  # noqa: E402
from bench import bytes_csr, peaks  # noqa: E402
from paper_2006_16852_b200 import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--matrix", default="27pt")
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--dtype", default="float64")
ap.add_argument("--reps", type=int, default=20)
args, _ = ap.parse_known_args()
exc = b2.CudaExecutor(0)
a = problems.stencil(exc, args.matrix, args.grid, value_dtype=args.dtype)
n, nnz = a.size.rows, a.nnz
vt = 8 if args.dtype == "float64" else 4
b = b2.Dense(exc, np.random.default_rng(0).standard_normal((n, 1)), value_dtype=args.dtype)
x = b2.Dense.zeros(exc, n, 1, value_dtype=args.dtype)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
peak, _ = peaks()
by = bytes_csr(n, nnz, vt)
print(f"matrix={args.matrix} g={args.grid} n={n} nnz={nnz} dtype={args.dtype}")
cases = [("ld", s, c, 0) for s in ((1, 1), (1, 2), (1, 4)) for c in (4096,)]
cases += [("ld", s, c, 1) for s in ((1, 1), (2, 1), (1, 2), (1, 4)) for c in (1024, 2048, 2728, 4096)]
if "--tma" in sys.argv:
    cases += [("tma", (1, r), c, 0) for r in (1, 2, 4) for c in (1024, 2048, 4096)]
for impl, shape, cap, gr in cases:
    if True:
        m = b2.convert(a, "csr")
        m.set_strategy("stream", stream_shape=shape, stream_cap=cap, stream_impl=impl, gather_in_reduce=gr)
        impl = impl + ("+gr" if gr else "")
        for _ in range(3):
            m.apply(b, x)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
        for s, e in ev:
            flush.fill_(1)
            s.record()
            m.apply(b, x)
            e.record()
        torch.cuda.synchronize()
        t = statistics.median(s.elapsed_time(e) for s, e in ev) * 1e-3
        print(f"{impl:3s} shape {shape[0]}x{shape[1]} cap {cap:5d}: {t * 1e6:8.1f} us {by / t / 1e9:7.1f} GB/s "
              f"frac {by / t / 1e9 / peak:.3f}")
