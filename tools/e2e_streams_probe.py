"""C2 e2e (Csr.apply, pinned host b and x) vs the host pipeline's chunk count
and stream counts (H2D, SpMV, D2H); every result checked bit for bit against
the device SpMV.

  python tools/e2e_streams_probe.py
"""
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import problems  # noqa: E402
from paper_2006_16852_b200.formats import Csr  # noqa: E402

exc = b2.CudaExecutor(0)
a = problems.stencil(exc, "27pt", 128)
n = a.size.rows
bv = np.random.default_rng(0).standard_normal((n, 1))
b = b2.Dense(exc.master, bv)
x = b2.Dense.zeros(exc.master, n, 1)
ref = b2.Dense.zeros(exc, n, 1)
a.apply(b2.Dense(exc, bv), ref)
ref = ref.values.cpu().numpy()


def run(k, streams, reps=30):  # needs Csr.HOST_PIPELINE_STREAMS (removed after the sweep; see profiles/r03_e2e_streams.txt)
    Csr.HOST_PIPELINE_CHUNKS = k
    Csr.HOST_PIPELINE_STREAMS = streams
    a._pplan = None
    np.asarray(x.values)[:] = 0
    for _ in range(3):
        a.apply(b, x)
    ok = np.array_equal(np.asarray(x.values), ref)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.apply(b, x)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3, min(ts) * 1e3, ok


for rnd in range(2):
    for k in (6, 8, 12):
        for streams in ((1, 1, 1), (2, 1, 2), (1, 2, 1), (2, 2, 2), (3, 2, 3)):
            med, mn, ok = run(k, streams)
            print(f"round {rnd} chunks {k:2d} streams {streams}: median {med:.3f} ms  min {mn:.3f} ms  bitwise {ok}",
                  flush=True)
