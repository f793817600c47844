"""How much do the C4 / C5 iteration counts move under an equally valid change
of the reductions' summation partition (knob kry_grid_div: the grid-stride
dot products and their block order)? The reference's own two CPU executors
also sum differently (ReferenceExecutor: one NumPy pairwise sum;
ParallelExecutor: 8 blocks). Prints one JSON line per (case, partition).

    python tools/rounding_sensitivity.py [--grid 256]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import _lib, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--divs", default="1,2,3,4,5,8")
args = ap.parse_args()
exc = b2.CudaExecutor(0)
cases = [("c4_bicgstab_bj32", "convdiff", "bicgstab", 32, {}), ("c4_gmres30_bj32", "convdiff", "gmres", 32, {"krylov_dim": 30}),
         ("c5_cg", "7pt", "cg", 0, {})]
mats = {}
for name, kind, solver, bs, kw in cases:
    a = mats.get(kind) or mats.setdefault(kind, problems.stencil(exc, kind, args.grid))
    n = a.size.rows
    for div in [int(d) for d in args.divs.split(",")]:
        _lib.set_tuning("kry_grid_div", div)
        pre = b2.Jacobi(exc, block_size=bs) if bs else None
        s = b2.SOLVER_FACTORIES[solver](exc, criteria=[b2.Iteration(20000), b2.ResidualNormReduction(1e-8)],
                                        preconditioner=pre, **kw).generate(a)
        b = b2.Dense.wrap(exc, torch.ones((n, 1), dtype=torch.float64, device=exc.device))
        x = b2.Dense.wrap(exc, torch.zeros((n, 1), dtype=torch.float64, device=exc.device))
        s.apply(b, x)
        st = s.last_status
        bd = None if st.breakdown is None else f"{st.breakdown.reason} @ {st.breakdown.iteration}"
        res = None
        if kind == "convdiff" or True:
            ax = b2.Dense.wrap(exc, torch.empty((n, 1), dtype=torch.float64, device=exc.device))
            a.apply(x, ax)
            res = float(torch.linalg.vector_norm(b.values - ax.values) / np.sqrt(n))
        print(json.dumps({"case": name, "grid": args.grid, "kry_grid_div": div, "iterations": st.iterations,
                          "converged": st.converged, "breakdown": bd, "true_rel_residual": res}), flush=True)
_lib.set_tuning("kry_grid_div", 1)
