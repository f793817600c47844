"""Does copy-engine traffic slow the SpMV? One C2 row chunk (1/8 of the rows;
also a 1-row launch, i.e. an almost empty kernel, and the full matrix) timed alone, during a 16.8 MB pinned H2D copy, during a D2H copy, and during
both (CUDA events on the kernel's stream, median of 20).

  python tools/e2e_interference_probe.py
"""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import _lib, problems  # noqa: E402

exc = b2.CudaExecutor(0)
m = problems.stencil(exc, "27pt", 128)
n = m.size.rows
bd = torch.randn(n, dtype=torch.float64, device="cuda")
xd = torch.zeros(n, dtype=torch.float64, device="cuda")
hb = torch.empty(4 * n, dtype=torch.float64).pin_memory()
hx = torch.empty(4 * n, dtype=torch.float64).pin_memory()
db = torch.empty(4 * n, dtype=torch.float64, device="cuda")
s_k, s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
sw = m._subwarp_arg()


def chunk(rows):
    r0, r1 = 0, rows
    _lib.call("csr_spmv_classical_f64", r1 - r0, m._rp.data_ptr(), m._ci.data_ptr(), m._v.data_ptr(), bd.data_ptr(), 1,
              xd.data_ptr(), 1, 1.0, 0, 0.0, 0, 0, 0, sw, s_k.cuda_stream)


def timed(rows, h2d, d2h, reps=20):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        if h2d:
            with torch.cuda.stream(s_in):
                db.copy_(hb, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s_out):
                hx.copy_(db, non_blocking=True)
        torch.cuda._sleep(20000)  # let the copies start
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s_k):
            torch.cuda._sleep(20000)
            a.record(s_k)
            chunk(rows)
            b.record(s_k)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


for rows in (1, n // 8, n):
    print(f"rows {rows:8d}: alone {timed(rows, 0, 0):7.1f} us | during H2D {timed(rows, 1, 0):7.1f} us | "
          f"during D2H {timed(rows, 0, 1):7.1f} us | during both {timed(rows, 1, 1):7.1f} us", flush=True)
