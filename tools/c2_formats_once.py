"""One apply (after warm-up) of every C2 SpMV format, fp64 then fp32 -- the
command profiled by ncu for profiles/r03*_ncu_c2_spmv.txt:

    ncu --set full --clock-control none --import-source on \
        -k regex:"csr_classical|csr_lb2|coo_kernel|ell_kernel|sellp_kernel" \
        -o gpurun_out/c2 python tools/c2_formats_once.py
    python tools/ncu_summary.py gpurun_out/c2.ncu-rep
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import problems  # noqa: E402

exc = b2.CudaExecutor(0)
for dt in ("float64", "float32"):
    a = problems.stencil(exc, "27pt", 128, value_dtype=dt)
    n = a.size.rows
    b = b2.Dense(exc, np.random.default_rng(0).standard_normal((n, 1)), value_dtype=dt)
    x = b2.Dense.zeros(exc, n, 1, value_dtype=dt)
    for fmt in ("csr_classical", "csr_lb", "coo", "ell", "sellp", "hybrid"):
        m = b2.convert(a, fmt)
        m.apply(b, x)
        exc.synchronize()
        m.apply(b, x)
    exc.synchronize()
