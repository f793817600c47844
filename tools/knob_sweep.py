"""Time one C2 format under different b200sp_set_tuning knob settings
(CUDA events; L2 flushed by a 256 MiB write then read between reps).

    python tools/knob_sweep.py --format sellp --knobs "sellp_per_sm=16,0 sellp_unroll=4,8" [--dtype float32]
"""
import argparse
import itertools
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2006_16852_b200 as b2  # noqa: E402
from bench import bytes_format, peaks  # noqa: E402
from oracle import spmv as OS  # noqa: E402
from paper_2006_16852_b200 import _lib, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--format", default="csr_classical")
ap.add_argument("--knobs", default="")
ap.add_argument("--matrix", default="27pt")
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--dtype", default="float64")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--subwarp", default="", help="comma list of classical sub-warp sizes to sweep")
args = ap.parse_args()
exc = b2.CudaExecutor(0)
if args.matrix == "powerlaw":
    a = problems.power_law(exc, 4194304, seed=0, value_dtype=args.dtype)
else:
    a = problems.stencil(exc, args.matrix, args.grid, value_dtype=args.dtype)
n = a.size.rows
vt = 8 if args.dtype == "float64" else 4
b = b2.Dense(exc, np.random.default_rng(0).standard_normal((n, 1)), value_dtype=args.dtype)
x = b2.Dense.zeros(exc, n, 1, value_dtype=args.dtype)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
peak, _ = peaks()
ref = None
knobs = [(k.split("=")[0], [int(v) for v in k.split("=")[1].split(",")]) for k in args.knobs.split()]
fmts = args.format.split(",")
if args.subwarp:
    fmts = [f"csr_classical/{sw}" for sw in args.subwarp.split(",")]
for fmt in fmts:
    attrs = {}
    if ":" in fmt:  # e.g. coo:chunk=128
        fmt, kv = fmt.split(":")
        attrs = {k: (int(v) if v.lstrip("-").isdigit() else v) for k, v in (p.split("=") for p in kv.split(";"))}
    m = b2.convert(a, fmt.split("/")[0])
    for k, v in attrs.items():
        setattr(m, k, v)
    if "/" in fmt:
        m.set_strategy("classical", subwarp=int(fmt.split("/")[1]))
    by = bytes_format(m, vt)
    print(f"{fmt} {args.matrix} g={args.grid} {args.dtype}: {by / 1e6:.1f} MB/SpMV")
    for combo in itertools.product(*[vals for _, vals in knobs]) if knobs else [()]:
        for (k, _), val in zip(knobs, combo):
            _lib.set_tuning(k, val)
        if hasattr(m, "_plan"):
            m._plan = None  # plans depend on knobs (lb_tile)
        x.fill(float("nan"))  # a variant that skips rows must not inherit the previous output
        m.apply(b, x)
        out = np.asarray(x.data).copy()
        if ref is None:
            ref = out
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
        desc = " ".join(f"{k}={v}" for (k, _), v in zip(knobs, combo))
        print(f"  {desc:40s}: {t * 1e6:8.1f} us {by / t / 1e9:7.1f} GB/s frac {by / t / 1e9 / peak:.3f} err {err:.1e}")
    del m
    torch.cuda.empty_cache()
