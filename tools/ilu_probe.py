"""ILU(0)-preconditioned CG on a 7-point Poisson problem: ParILU generation
time, triangular-solve time per apply, iterations, ms per iteration."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import problems  # noqa: E402

exc = b2.CudaExecutor(0)
for g in (64, 128):
    a = problems.stencil(exc, "7pt", g)
    n = a.size.rows
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pre = b2.Ilu(exc, sweeps=5).generate(a)
    torch.cuda.synchronize()
    gen = time.perf_counter() - t0
    b = b2.Dense(exc, np.ones((n, 1)))
    z = b2.Dense.zeros(exc, n, 1)
    pre.apply(b, z)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        pre.apply(b, z)
    torch.cuda.synchronize()
    app = (time.perf_counter() - t0) / 10
    for name, p in (("none", None), ("ilu", b2.Ilu(exc, sweeps=5)), ("bj32", b2.Jacobi(exc, block_size=32))):
        s = b2.Cg(exc, criteria=[b2.Iteration(5000), b2.ResidualNormReduction(1e-8)], preconditioner=p).generate(a)
        x = b2.Dense.zeros(exc, n, 1)
        s.apply(b, x)
        x = b2.Dense.zeros(exc, n, 1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.apply(b, x)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        it = s.last_status.iterations
        print(f"7pt {g}^3 CG+{name}: {it} iterations, {t * 1e3:.1f} ms, {t / it * 1e3:.3f} ms/iter")
    print(f"7pt {g}^3: ParILU(5 sweeps)+trs setup {gen * 1e3:.1f} ms; ILU apply (L then U solve) {app * 1e3:.3f} ms")
