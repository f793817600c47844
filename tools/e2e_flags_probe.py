"""C2 e2e (Csr.apply with pinned host b and x): the flag-driven persistent
pipeline (HOST_PIPELINE_MODE "flags", b200sp_csr_spmv_pipe) against the
event-driven one ("events"), per chunk count; each result is checked against
the device SpMV bit for bit.

  python tools/e2e_flags_probe.py
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
host = exc.master
a = problems.stencil(exc, "27pt", 128)
n = a.size.rows
rng = np.random.default_rng(0)
bv = rng.standard_normal((n, 1))
b = b2.Dense(host, bv)
x = b2.Dense.zeros(host, n, 1)
ref = b2.Dense.zeros(exc, n, 1)
a.apply(b2.Dense(exc, bv), ref)
ref = ref.values.cpu().numpy()


def run(mode, k, reps=30):
    Csr.HOST_PIPELINE_MODE = mode
    Csr.HOST_PIPELINE_CHUNKS = k
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


from paper_2006_16852_b200 import _lib  # noqa: E402

for rnd in range(2):
    med, mn, ok = run("events", 8)
    print(f"round {rnd} events chunks  8: median {med:.3f} ms  min {mn:.3f} ms  bitwise {ok}", flush=True)
    for backoff in (0, 64, 500):
        for per_sm in (0, 1):
            _lib.set_tuning("pipe_backoff", backoff)
            _lib.set_tuning("pipe_per_sm", per_sm)
            for k in (2, 4, 8):
                med, mn, ok = run("flags", k)
                print(f"round {rnd} flags backoff {backoff:3d} per_sm {per_sm} chunks {k:2d}: median {med:.3f} ms  "
                      f"min {mn:.3f} ms  bitwise {ok}", flush=True)
