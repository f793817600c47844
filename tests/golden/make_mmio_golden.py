"""Golden cases for the Matrix Market reader/writer, produced by running the
REFERENCE (src/mmio.py) in the build container:
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_mmio_golden.py
Writes tests/golden/mmio.json (inputs, the reference's triples or error class
+ message + line, and the reference writer's exact text)."""

import io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from opalg import mmio  # noqa: E402
from opalg.base import Dim2  # noqa: E402
from opalg.formats import MatrixData  # noqa: E402

H = "%%MatrixMarket matrix coordinate real general\n"
HS = "%%MatrixMarket matrix coordinate real symmetric\n"
HA = "%%MatrixMarket matrix array real general\n"
INPUTS = {
    "tri3": H + "3 3 7\n1 1 2\n1 2 -1\n2 1 -1\n2 2 2\n2 3 -1\n3 2 -1\n3 3 2\n",
    "sym": HS + "% comment\n\n4 4 5\n1 1 4.0\n2 1 -1.5e-3\n3 2 1e+300\n4 4 -0.0\n4 1 7\n",
    "dups_unsorted": H + "3 4 5\n3 4 1.0\n1 2 2.0\n3 4 0.5\n1 1 -1\n1 2 1e-20\n",
    "array": HA + "2 3\n1\n2\n3\n4.5\n0\n-6\n",
    "crlf": "%%MatrixMarket Matrix Coordinate REAL General\r\n2 2 2\r\n1 1 1.25\r\n2 2 -2\r\n",
    "cr_only": H.replace("\n", "\r") + "1 1 1\r1 1 3\r",
    "tabs_trailing": H + "  2\t2 1 \n\t 2  1\t 5.5   \n\n% tail comment\n",
    "inf_nan": H + "2 2 2\n1 1 inf\n2 2 -Infinity\n",
    "underscore_int": H + "2 2 1\n1_0 1 1\n",
    "empty": "",
    "blank": "\n",
    "bad_header": "%%MatrixMarket matrix coordinate real\n1 1 0\n",
    "bad_format": "%%MatrixMarket matrix sparse real general\n1 1 0\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 0\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n1 1 0\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n",
    "missing_size": H + "% only comments\n%\n",
    "size_two": H + "2 2\n",
    "size_bad": H + "2 two 1\n",
    "entry_short": H + "2 2 1\n1 1\n",
    "entry_long": H + "2 2 1\n1 1 1 1\n",
    "entry_float_index": H + "2 2 1\n1.0 1 1\n",
    "entry_bad_value": H + "2 2 1\n1 1 one\n",
    "out_of_range": H + "2 2 2\n1 1 1\n0 2 1\n",
    "too_few": H + "2 2 3\n1 1 1\n2 2 1\n",
    "too_many": H + "2 2 1\n1 1 1\n2 2 1\n",
    "array_sym": "%%MatrixMarket matrix array real symmetric\n2 2\n1\n2\n3\n",
    "array_short": HA + "2 2\n1\n2\n3\n",
    "array_bad": HA + "1 2\n1\nx\n",
    "hex_value": H + "1 1 1\n1 1 0x10\n",
    "empty_matrix": H + "3 3 0\n",
}


def run(text):
    try:
        d = mmio.read_matrix_market(io.StringIO(text))
    except Exception as e:  # noqa: BLE001
        return {"error": type(e).__name__, "message": str(e), "line": getattr(e, "line", None)}
    return {"size": [d.size.rows, d.size.cols], "rows": d.rows.tolist(), "cols": d.cols.tolist(),
            "vals": [repr(float(v)) for v in d.vals]}


def written(data):
    s = io.StringIO()
    mmio.write_matrix_market(s, data)
    return s.getvalue()


def main():
    cases = {k: {"input": v, "expect": run(v)} for k, v in INPUTS.items()}
    rng = np.random.default_rng(5)
    r = rng.integers(0, 40, 300)
    c = rng.integers(0, 30, 300)
    v = rng.standard_normal(300) * 10.0 ** rng.integers(-20, 20, 300)
    writes = {
        "random_dups": {"size": [40, 30], "rows": r.tolist(), "cols": c.tolist(), "vals": v.tolist(),
                        "text": written(MatrixData(Dim2(40, 30), r, c, v))},
    }
    s = io.StringIO()
    mmio.write_matrix_market_array(s, np.arange(6.0).reshape(2, 3) / 7)
    writes["array_2x3"] = {"dense": (np.arange(6.0).reshape(2, 3) / 7).tolist(), "text": s.getvalue()}
    with open(os.path.join(HERE, "mmio.json"), "w") as f:
        json.dump({"read": cases, "write": writes}, f, indent=0)
    print(f"wrote {len(cases)} read cases, {len(writes)} write cases")


if __name__ == "__main__":
    main()
