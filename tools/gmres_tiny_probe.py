"""GMRES(100) on the paper's 1x1 overhead system, for profiling the small-system cycle kernel."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16852_b200 as b2  # noqa: E402

exc = b2.create_executor("cuda")
a = b2.matrix_from_data(exc, b2.MatrixData((1, 1), np.array([0]), np.array([0]), np.array([1.0])), "coo")
s = b2.Gmres(exc, criteria=[b2.Iteration(300)], krylov_dim=100).generate(a)
x = b2.Dense.zeros(exc, 1, 1)
s.apply(b2.Dense(exc, np.full((1, 1), np.nan)), x)
print(s.last_status.iterations)
