"""The paper's traffic model (src/model.py:50-123) against the reference's
own values (tests/golden/model.json, make_model_golden.py): exact integers."""
import json
import os

import pytest

from conftest import GOLDEN


def test_predict_traffic_matches_reference():
    from paper_2006_16852_b200.model import TrafficParams, predict_traffic

    cases = json.load(open(os.path.join(GOLDEN, "model.json")))
    assert len(cases) > 1000
    for s, n, z, it, k, vb, rd, wr in cases:
        p = predict_traffic(s, TrafficParams(n, z, it, vb, 4, k))
        assert (p.bytes_read, p.bytes_written) == (rd, wr), (s, n, z, it, k, vb)


def test_model_errors_and_per_iteration():
    from paper_2006_16852_b200.errors import OpalgError, Unsupported
    from paper_2006_16852_b200.model import TrafficParams, per_iteration_bytes, predict_traffic

    with pytest.raises(Unsupported):
        predict_traffic("ir", TrafficParams(1, 1, 1))
    with pytest.raises(OpalgError):
        TrafficParams(-1, 1, 1)
    # CG: (15n + 2nnz) VT + 2nnz IT read, (5n + 2) VT written per iteration (src/model.py:50-55)
    n, z = 961, 4681
    assert per_iteration_bytes("cg", n, z, 10) == (15 * n + 2 * z) * 8 + 2 * z * 4 + (5 * n + 2) * 8
