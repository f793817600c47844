"""Csr stream variants on stencils: register-staged ("ld") vs the persistent
TMA pipeline ("tma"), over rows-per-thread / stages (CUDA events; L2 flushed
by a 256 MiB write then a 256 MiB read between reps).

    python tools/pipe_sweep.py [--matrix 27pt] [--grid 128] [--dtype float64]
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
from oracle import spmv as OS  # noqa: E402
from paper_2006_16852_b200 import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--matrix", default="27pt")
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--dtype", default="float64")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
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
ref = None
cases = [("ld", None)]
for shape, nt in (((2, 1), 256), ((2, 2), 256), ((1, 1), 256), ((2, 1), 512), ((2, 2), 512), ((4, 1), 512),
                  ((4, 2), 512)):
    for stages in (2, 3):
        cases.append(("tma", (shape, nt, stages)))
cases.append(("tma-default", None))
for impl, cfg in cases:
    m = b2.convert(a, "csr")
    if impl == "ld":
        m.set_strategy("stream", stream_impl="ld")
    elif impl == "tma-default":
        m.set_strategy("stream", stream_impl="tma")
    else:
        shape, nt, stages = cfg
        m.set_strategy("stream", stream_impl="tma", stream_shape=shape, stream_stages=stages, stream_consumers=nt)
        rows = nt // shape[0] * shape[1]
        # stage = the whole tile (rows x max row length)
        cap = (rows * 27 + 8) // 4 * 4 if args.matrix == "27pt" else (rows * 7 + 8) // 4 * 4
        m._stream_cap = cap
        per_cta = 256 + stages * (((rows + 4) // 4 * 4) * 4 + cap * (4 + vt))
        if per_cta > 226 * 1024:
            continue
    x.fill(float("nan"))
    m.apply(b, x)
    out = np.asarray(x.data)
    if ref is None:
        ref = out.copy()
    err = OS.rel_error_inf(out, ref)
    for _ in range(3):
        m.apply(b, x)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
    for s, e in ev:
        flush.fill_(1)
        flush.view(torch.int64).sum()
        s.record()
        m.apply(b, x)
        e.record()
    torch.cuda.synchronize()
    t = statistics.median(s.elapsed_time(e) for s, e in ev) * 1e-3
    cfg = m.tma_config() if impl.startswith("tma") else m.stream_config()
    print(f"{impl:3s} cfg {str(cfg):24s}: {t * 1e6:8.1f} us {by / t / 1e9:7.1f} GB/s frac {by / t / 1e9 / peak:.3f}"
          f"  err-vs-ld {err:.1e}")
