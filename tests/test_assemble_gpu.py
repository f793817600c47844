"""Device assembly of coordinate triples against the
reference's MatrixData.canonicalize run on the same inputs
(tests/golden/assemble.npz): sorted (row, col), duplicates summed in input
order -- bit-exact, -0.0 and exact cancellations included."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden_asm():
    return load_golden("assemble.npz")


@pytest.mark.parametrize("name", ["small", "mid", "wide", "tall", "nodup"])
def test_assembly_bit_exact(cuda, golden_asm, name):
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200.formats import assemble_device

    g = golden_asm[name]
    nr, nc = (int(x) for x in g["size"])
    data = b2.MatrixData((nr, nc), g["rows_in"], g["cols_in"], g["vals_in"])
    r, c, v = assemble_device(cuda, data, np.float64)
    np.testing.assert_array_equal(r.cpu().numpy(), g["rows"])
    np.testing.assert_array_equal(c.cpu().numpy(), g["cols"])
    got = v.cpu().numpy()
    assert got.tobytes() == g["vals"].tobytes()  # bitwise, signed zeros included
    # through the public API: Csr.from_data / Coo.from_data / to_data
    for cls in (b2.Csr, b2.Coo):
        m = cls.from_data(cuda, data)
        back = m.to_data()
        np.testing.assert_array_equal(back.rows, g["rows"])
        assert back.vals.tobytes() == g["vals"].tobytes()


def test_assembly_errors_and_empty(cuda):
    import paper_2006_16852_b200 as b2

    with pytest.raises(b2.DimensionMismatch):
        b2.Csr.from_data(cuda, b2.MatrixData((2, 2), [0, 2], [0, 0], [1.0, 1.0]))
    with pytest.raises(b2.DimensionMismatch):
        b2.Csr.from_data(cuda, b2.MatrixData((2, 2), [0, 1], [0, -1], [1.0, 1.0]))
    m = b2.Csr.from_data(cuda, b2.MatrixData((3, 3)))
    assert m.nnz == 0 and np.asarray(m.row_ptrs).tolist() == [0, 0, 0, 0]


def test_assembly_large_stencil_matches_oracle(cuda):
    """A shuffled 27-point 64^3 stencil (7M triples, two duplicates per
    entry) assembles to the canonical stencil."""
    import paper_2006_16852_b200 as b2
    from oracle import problems as P

    n, r, c, v = P.stencil3d(64, "27pt")
    rng = np.random.default_rng(0)
    order = rng.permutation(r.size)
    half = v / 2
    data = b2.MatrixData((n, n), np.concatenate([r[order], r]), np.concatenate([c[order], c]),
                         np.concatenate([half[order], half]))
    m = b2.Csr.from_data(cuda, data)
    rp, ci, vals = P.to_csr(n, r, c, v)
    assert np.array_equal(np.asarray(m.row_ptrs), rp)
    assert np.array_equal(np.asarray(m.col_idxs), ci)
    assert np.array_equal(np.asarray(m.vals), 0.0 + half + half)
