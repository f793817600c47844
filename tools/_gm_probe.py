import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2006_16852_b200 as b2
exc = b2.CudaExecutor(0)
a = b2.Coo(exc, (1, 1), [0], [0], [1.0])
for k in (100, 30):
    s = b2.Gmres(exc, criteria=[b2.Iteration(1000)], krylov_dim=k).generate(a)
    for r in range(3):
        x = b2.Dense.zeros(exc, 1, 1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.apply(b2.Dense(exc, [[float("nan")]]), x)
        t1 = time.perf_counter()
        print(k, r, s.last_status.iterations, f"{(t1 - t0) * 1e3:.2f} ms")
