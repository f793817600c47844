"""Hybrid Ell width on C3 (4,194,304-row power law, SURVEY row lengths, fp64):
CUDA events, L2 flushed between reps, mean of 10.

    python tools/hybrid_width_sweep.py [--widths 8,12,16,20,24,32]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import formats, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--widths", default="8,12,16,20,24,32")
args = ap.parse_args()
exc = b2.CudaExecutor(0)
a = problems.power_law(exc, 4194304, seed=0, lengths="rng")
n = a.size.rows
b = b2.Dense(exc, np.random.default_rng(0).standard_normal((n, 1)))
x = b2.Dense.zeros(exc, n, 1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(m, reps=10):
    m.apply(b, x)
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        flush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        m.apply(b, x)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return float(np.mean(ts))


cases = [("auto", formats.automatic())] + [(f"w{w}", formats.column_limit(int(w))) for w in args.widths.split(",")]
for label, strat in cases:
    h = b2.convert(a, "hybrid", strategy=strat)
    print(f"{label:6s} width {h.ell.width} coo nnz {h.coo.nnz}"
          f" {timed(h):7.1f} us", flush=True)
print(f"coo    {timed(b2.convert(a, 'coo')):7.1f} us")
