"""C1 CG (5-point 256^2) us per iteration vs the cooperative kernel's block
count, for the global-memory kernel (coop_resident 0) and the
register-resident one (coop_resident 1); the two must give bitwise the same x
at the same block count."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import _lib, problems  # noqa: E402

exc = b2.CudaExecutor(0)
a = problems.stencil(exc, "5pt", 256)
n = a.size.rows
s = b2.Cg(exc, criteria=[b2.Iteration(10000), b2.ResidualNormReduction(1e-8)]).generate(a)
b = b2.Dense(exc, np.ones((n, 1)))
xs = {}
for res in (0, 1):
    _lib.set_tuning("coop_resident", res)
    for blocks in (0, 128, 148, 256):
        _lib.set_tuning("coop_blocks", blocks)
        ts = []
        for r in range(4):
            x = b2.Dense.zeros(exc, n, 1)
            exc.synchronize()
            t0 = time.perf_counter()
            s.apply(b, x)
            ts.append(time.perf_counter() - t0)
        it = s.last_status.iterations
        xs[res, blocks] = np.asarray(x.data).copy()
        same = "" if res == 0 else f"  bitwise = res0: {np.array_equal(xs[0, blocks], xs[1, blocks])}"
        print(f"coop_resident {res} coop_blocks {blocks:4d}: {np.median(ts[1:]) / it * 1e6:7.2f} us/iter "
              f"({it} iterations){same}", flush=True)
_lib.set_tuning("coop_resident", 1)
_lib.set_tuning("coop_blocks", 0)
