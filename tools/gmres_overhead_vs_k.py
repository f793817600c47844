"""GMRES(k) on the paper's 1x1 overhead system (b = NaN, 1000 iterations): us per
iteration vs the Krylov dimension k (profiles/r03_overhead_tiny.txt)."""
import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2006_16852_b200 as b2
exc = b2.create_executor("cuda")
a = b2.matrix_from_data(exc, b2.MatrixData((1, 1), np.array([0]), np.array([0]), np.array([1.0])), "coo")
for k in (2, 5, 10, 30, 100):
    s = b2.Gmres(exc, criteria=[b2.Iteration(1000)], krylov_dim=k).generate(a)
    ts = []
    for r in range(5):
        x = b2.Dense.zeros(exc, 1, 1)
        exc.synchronize(); t0 = time.perf_counter()
        s.apply(b2.Dense(exc, np.full((1, 1), np.nan)), x)
        ts.append(time.perf_counter() - t0)
    print(k, f"{min(ts[1:]) / 1000 * 1e6:.3f} us/iter", s.last_status.iterations)
