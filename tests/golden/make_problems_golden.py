"""SHA-256 of the reference's host generators' raw triples (src/problems.py),
produced by running the reference in the build container:
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_problems_golden.py"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from opalg import problems  # noqa: E402


def digest(d):
    h = hashlib.sha256()
    for a in (np.asarray(d.rows, np.int64), np.asarray(d.cols, np.int64), np.asarray(d.vals, np.float64)):
        h.update(a.tobytes())
    return [d.size.rows, d.size.cols, int(d.vals.size), h.hexdigest()]


cases = {
    "tridiagonal_50": digest(problems.tridiagonal(50)),
    "tridiagonal_7_zero_upper": digest(problems.tridiagonal(7, lower=-0.5, diag=3.0, upper=0.0)),
    "five_point_poisson_1": digest(problems.five_point_poisson(1)),
    "five_point_poisson_64": digest(problems.five_point_poisson(64)),
    "convection_diffusion_30": digest(problems.convection_diffusion(30)),
    "convection_diffusion_5_c1": digest(problems.convection_diffusion(5, convection=1.0)),
    "random_sparse_30": digest(problems.random_sparse(30, density=0.2, seed=3)),
    "random_sparse_12_nodd": digest(problems.random_sparse(12, density=0.5, seed=1, diag_dominant=False)),
}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "problems.json"), "w") as f:
    json.dump(cases, f, indent=0)
print(len(cases), "cases")
