"""Reference arm check (build container only: imports /root/reference): the
stock reference ParallelExecutor Csr.apply vs the oracle port bench.py times
(oracle/cpu_baseline.py) on the full C2 matrix -- time and bitwise result.

    python tools/ref_arm_gap.py
"""
import os, sys, time, statistics
import numpy as np
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/repo")
import opalg
from opalg import Csr, Dense, Dim2
from oracle import problems as P
from oracle import cpu_baseline as CB
g = 128
n, r, c, v = P.stencil3d(g, "27pt")
rp, ci, vals = P.to_csr(n, r, c, v)
del r, c, v
rng = np.random.default_rng(0)
b = rng.standard_normal((n, 1))
workers = os.cpu_count()
exc = opalg.ParallelExecutor(workers)
A = Csr(exc, Dim2(n, n), rp.astype(np.int32), ci.astype(np.int32), vals)
B = Dense(exc, b); X = Dense.zeros(exc, n, 1)
A.apply(B, X)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); A.apply(B, X); ts.append(time.perf_counter() - t0)
t_ref = statistics.median(ts)
port = CB.ParallelCsr(rp.astype(np.int32), ci.astype(np.int32), vals, workers)
out = np.zeros((n, 1)); port.apply(b, out)
ts2 = []
for _ in range(5):
    t0 = time.perf_counter(); port.apply(b, out); ts2.append(time.perf_counter() - t0)
t_port = statistics.median(ts2)
same = np.array_equal(np.asarray(out).reshape(-1), X.data.reshape(-1))
byts = vals.size * 12 + (n + 1) * 4 + 2 * n * 8
print(f"workers {workers}: stock opalg ParallelExecutor {t_ref*1e3:.1f} ms ({byts/t_ref/1e9:.2f} GB/s), port {t_port*1e3:.1f} ms ({byts/t_port/1e9:.2f} GB/s), port/stock time {t_port/t_ref:.3f}, bitwise {same}")
