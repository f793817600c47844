"""Launch every C2 SpMV variant a few times (target for ncu captures).

    python tools/spmv_probe.py [--grid 128] [--reps 3] [--dtype float64]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--dtype", default="float64")
ap.add_argument("--formats", default="csr_classical,csr_lb,coo,ell,sellp,hybrid")
ap.add_argument("--matrix", default="27pt")
ap.add_argument("--pipe", default="", help="rpt,stages,consumers for csr_pipe")
args = ap.parse_args()

exc = b2.CudaExecutor(0)
a = problems.stencil(exc, args.matrix, args.grid, value_dtype=args.dtype)
n = a.size.rows
b = b2.Dense(exc, np.random.default_rng(0).standard_normal((n, 1)), value_dtype=args.dtype)
x = b2.Dense.zeros(exc, n, 1, value_dtype=args.dtype)
for fmt in args.formats.split(","):
    m = b2.convert(a, fmt)
    if fmt == "csr_pipe" and args.pipe:
        rpt, stages, nt = (int(v) for v in args.pipe.split(","))
        m.set_strategy("stream", stream_impl="tma", stream_shape=(1, rpt), stream_stages=stages,
                       stream_consumers=nt)
    for _ in range(args.reps):
        m.apply(b, x)
    exc.synchronize()
    del m
print("probe done")
