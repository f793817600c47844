"""The reference's host test-system generators (src/problems.py) restated
in the package: identical raw triples (order included), pinned by SHA-256
of the reference's own output (tests/golden/problems.json)."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

G = json.load(open(os.path.join(GOLDEN, "problems.json")))


def digest(d):
    h = hashlib.sha256()
    for a in (np.asarray(d.rows, np.int64), np.asarray(d.cols, np.int64), np.asarray(d.vals, np.float64)):
        h.update(a.tobytes())
    return [d.size.rows, d.size.cols, int(d.vals.size), h.hexdigest()]


CASES = {
    "tridiagonal_50": lambda p: p.tridiagonal(50),
    "tridiagonal_7_zero_upper": lambda p: p.tridiagonal(7, lower=-0.5, diag=3.0, upper=0.0),
    "five_point_poisson_1": lambda p: p.five_point_poisson(1),
    "five_point_poisson_64": lambda p: p.five_point_poisson(64),
    "convection_diffusion_30": lambda p: p.convection_diffusion(30),
    "convection_diffusion_5_c1": lambda p: p.convection_diffusion(5, convection=1.0),
    "random_sparse_30": lambda p: p.random_sparse(30, density=0.2, seed=3),
    "random_sparse_12_nodd": lambda p: p.random_sparse(12, density=0.5, seed=1, diag_dominant=False),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_generator_matches_reference(name):
    from paper_2006_16852_b200 import problems

    assert digest(CASES[name](problems)) == G[name]
