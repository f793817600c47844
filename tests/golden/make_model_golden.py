"""Golden values of the reference's traffic model (src/model.py:50-123),
produced by running the reference in the build container:
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_model_golden.py"""
import itertools
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from opalg import model  # noqa: E402

out = []
for s in ("cg", "fcg", "cgs", "bicgstab", "gmres"):
    for n, z, it, k, vb in itertools.product((1, 961, 65536, 134217728), (1, 4681, 937951232), (0, 1, 2, 7, 101, 1225),
                                             (1, 30, 100), (8, 4)):
        p = model.predict_traffic(s, model.TrafficParams(n, z, it, vb, 4, k))
        out.append([s, n, z, it, k, vb, p.bytes_read, p.bytes_written])
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "model.json"), "w") as f:
    json.dump(out, f)
print(len(out), "cases")
