"""ILU apply time vs the triangular-solve claim granularity (knobs)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import _lib, problems  # noqa: E402

exc = b2.CudaExecutor(0)
a = problems.stencil(exc, "7pt", 128)
n = a.size.rows
pre = b2.Ilu(exc, sweeps=5).generate(a)
b = b2.Dense(exc, np.random.default_rng(0).standard_normal((n, 1)))
ref = None
from paper_2006_16852_b200.solvers.triangular import TriangularSolver  # noqa: E402

for mode, per_sm in (("syncfree", 0), ("coop", 1), ("coop", 2), ("coop", 4)):
    TriangularSolver.LEVEL_SYNC = mode == "coop"
    _lib.set_tuning("trs_coop_per_sm", per_sm)
    thread_rows, per_claim = mode, per_sm
    z = b2.Dense.zeros(exc, n, 1)
    pre.apply(b, z)
    out = np.asarray(z.data).copy()
    if ref is None:
        ref = out
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        pre.apply(b, z)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / 5
    print(f"{thread_rows} per_sm {per_claim}: ILU apply {t * 1e3:7.3f} ms "
          f"(max diff vs first {np.abs(out - ref).max():.1e})")
