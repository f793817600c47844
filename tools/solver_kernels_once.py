"""A few iterations of C4 BiCGSTAB / GMRES(30) + block-Jacobi(32) and C5-shaped CG
(7-point 256^3): the launch target for the solver-kernel ncu capture in
profiles/r03b_ncu_solvers.txt:

    ncu --set full --clock-control none -k regex:"bicg_step|csr_spmv_dot|jacobi_apply|cg_step|gmres_mgs" \
        -c 12 -o gpurun_out/solvers python tools/solver_kernels_once.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import problems  # noqa: E402

exc = b2.CudaExecutor(0)
for kind, solver, kw in (("convdiff", "bicgstab", {}), ("convdiff", "gmres", {"krylov_dim": 30}), ("7pt", "cg", {})):
    a = problems.stencil(exc, kind, 256)
    n = a.size.rows
    pre = b2.Jacobi(exc, block_size=32) if kind == "convdiff" else None
    s = b2.SOLVER_FACTORIES[solver](exc, criteria=[b2.Iteration(4)], preconditioner=pre, **kw).generate(a)
    b = b2.Dense.wrap(exc, torch.ones((n, 1), dtype=torch.float64, device=exc.device))
    x = b2.Dense.wrap(exc, torch.zeros((n, 1), dtype=torch.float64, device=exc.device))
    s.apply(b, x)
    exc.synchronize()
