"""The paper's overhead benchmark with the tiny single-thread solvers off / on
(b200sp_set_tuning("coop_tiny", 0/1)): python tools/overhead_probe.py"""
import sys, json
sys.path.insert(0, "/root/repo")
from paper_2006_16852_b200 import _lib, CudaExecutor
from paper_2006_16852_b200.profile import run_overhead
exc = CudaExecutor(0)
for v in (0, 1, 0, 1):  # coop_tiny
    _lib.set_tuning("coop_tiny", v)
    r = run_overhead(iters=1000, runs=10, executor=exc)
    print(v, {k: round(x["time_per_iteration_us"], 3) for k, x in r["solvers"].items()}, flush=True)
