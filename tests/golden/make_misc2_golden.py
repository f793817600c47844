"""Golden values for gauss_jordan_inverse and StencilMatrix (reference
src/precond.py:28-46, src/formats.py:268-298), made by running the reference:
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_misc2_golden.py"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import opalg  # noqa: E402
from opalg.precond import gauss_jordan_inverse  # noqa: E402

REF = opalg.ReferenceExecutor()
rng = np.random.default_rng(17)
out = {}
for k, bs in enumerate((1, 2, 5, 17, 32)):
    blk = rng.standard_normal((bs, bs)) + 3.0 * np.eye(bs)
    blk[rng.random((bs, bs)) < 0.3] = 0.0
    np.fill_diagonal(blk, np.diag(blk) + 0.5)
    out[f"gj_{k}_block"] = blk
    out[f"gj_{k}_inv"] = gauss_jordan_inverse(blk)
sing = np.array([[1.0, 2.0], [2.0, 4.0]])
out["gj_singular_block"] = sing
out["gj_singular_is_none"] = np.array(gauss_jordan_inverse(sing) is None)
b = rng.standard_normal((9, 2))
st = opalg.formats.StencilMatrix(REF, 9, -1.3, 2.5, 0.7)
x = opalg.Dense.zeros(REF, 9, 2)
st.apply(opalg.Dense(REF, b), x)
out["stencil_b"] = b
out["stencil_x"] = x.data.copy()
d = st.to_data()
out["stencil_rows"], out["stencil_cols"], out["stencil_vals"] = d.rows, d.cols, d.vals
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "misc2.npz"), **out)
print("ok", len(out))
