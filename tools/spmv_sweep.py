"""Time SpMV variants on C2 (CUDA events, L2 flushed between reps).

    python tools/spmv_sweep.py [--grid 128] [--dtype float64] [--matrix 27pt|powerlaw]
"""
import argparse
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import problems  # noqa: E402
from bench import bytes_csr, bytes_format, peaks  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--dtype", default="float64")
ap.add_argument("--matrix", default="27pt")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()

exc = b2.CudaExecutor(0)
if args.matrix == "powerlaw":
    a = problems.power_law(exc, 4194304, seed=0, value_dtype=args.dtype)
else:
    a = problems.stencil(exc, args.matrix, args.grid, value_dtype=args.dtype)
n, nnz = a.size.rows, a.nnz
vt = 8 if args.dtype == "float64" else 4
b = b2.Dense(exc, np.random.default_rng(0).standard_normal((n, 1)), value_dtype=args.dtype)
x = b2.Dense.zeros(exc, n, 1, value_dtype=args.dtype)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
peak, _ = peaks()


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
    for s, e in ev:
        flush.fill_(1)
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in ev) * 1e-3


variants = []
for sw in (4, 8, 16, 32):
    m = b2.convert(a, "csr")
    m.set_strategy("classical", subwarp=sw)
    variants.append((f"csr_classical_sw{sw}", m))
variants.append(("csr_lb", b2.convert(a, "csr_lb")))
variants.append(("csr_stream", b2.convert(a, "csr_stream")))
for shape in ((1, 1), (2, 1), (4, 1), (1, 2), (1, 4), (1, 8)):
    m = b2.convert(a, "csr")
    m.set_strategy("stream", stream_shape=shape)
    variants.append((f"csr_stream_{shape[0]}x{shape[1]}", m))
if args.matrix == "powerlaw":
    variants = [v for v in variants if v[0] in ("csr_lb", "csr_stream", "csr_classical_sw32")]
for ch in (128, 256):
    m = b2.convert(a, "coo")
    m.chunk = ch
    variants.append((f"coo_chunk{ch}", m))
if args.matrix != "powerlaw":
    variants += [("ell", b2.convert(a, "ell")), ("sellp", b2.convert(a, "sellp"))]
variants += [("hybrid", b2.convert(a, "hybrid"))]
print(f"matrix={args.matrix} n={n} nnz={nnz} dtype={args.dtype}")
for name, m in variants:
    t = timeit(lambda: m.apply(b, x))
    by = bytes_format(m, vt)
    print(f"{name:22s} {t * 1e6:8.1f} us  {by / t / 1e9:7.1f} GB/s  frac {by / t / 1e9 / peak:.3f}  "
          f"useful {bytes_csr(n, nnz, vt) / t / 1e9:7.1f} GB/s")
