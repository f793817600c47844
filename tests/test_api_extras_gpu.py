"""Reference API pieces around the hot path: gauss_jordan_inverse (bitwise
vs the reference, via the device generation kernel), the matrix-free
StencilMatrix (apply bitwise, to_data / Csr conversion), Array / StorageMode
ownership semantics (tests/golden/misc2.npz from make_misc2_golden.py)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(GOLDEN, "misc2.npz"))


def test_gauss_jordan_inverse_bitwise(cuda):
    import paper_2006_16852_b200 as b2

    for k in range(5):
        inv = b2.gauss_jordan_inverse(G[f"gj_{k}_block"], cuda)
        assert inv.tobytes() == G[f"gj_{k}_inv"].tobytes(), k
    assert b2.gauss_jordan_inverse(G["gj_singular_block"], cuda) is None


def test_stencil_matrix(cuda):
    import paper_2006_16852_b200 as b2

    st = b2.StencilMatrix(cuda, 9, -1.3, 2.5, 0.7)
    x = b2.Dense.zeros(cuda, 9, 2)
    st.apply(b2.Dense(cuda, G["stencil_b"]), x)
    assert np.asarray(x.data).tobytes() == G["stencil_x"].tobytes()
    d = st.to_data()
    np.testing.assert_array_equal(d.rows, G["stencil_rows"])
    np.testing.assert_array_equal(d.cols, G["stencil_cols"])
    np.testing.assert_array_equal(d.vals, G["stencil_vals"])
    c = st.convert_to("csr")
    y = b2.Dense.zeros(cuda, 9, 2)
    c.apply(b2.Dense(cuda, G["stencil_b"]), y)
    np.testing.assert_allclose(np.asarray(y.data), G["stencil_x"], rtol=1e-14)
    with pytest.raises(b2.Unsupported):
        st.convert_to("coo")
    s2 = st.clone_to(cuda)
    z = b2.Dense.zeros(cuda, 9, 2)
    s2.apply(b2.Dense(cuda, G["stencil_b"]), z)
    np.testing.assert_array_equal(np.asarray(z.data), np.asarray(x.data))


def test_array_ownership(cuda, host):
    import torch

    import paper_2006_16852_b200 as b2

    src = np.arange(6.0)
    a = b2.Array(cuda, data=src)
    assert a.mode is b2.StorageMode.OWNING and len(a) == 6
    src[0] = 99.0
    assert float(a.data[0]) == 0.0  # owning copies
    t = torch.arange(4.0, dtype=torch.float64, device="cuda")
    v = b2.Array.view(cuda, 3, t)
    assert v.mode is b2.StorageMode.VIEW and len(v) == 3
    t[1] = 7.0
    assert float(v.data[1]) == 7.0  # views alias
    with pytest.raises(b2.OpalgError):
        b2.Array.view(cuda, 5, t)
    h = a.copy_to(host)
    np.testing.assert_array_equal(h.data, np.arange(6.0))
    d = h.copy_to(cuda)
    assert torch.equal(d.data.cpu(), torch.arange(6.0, dtype=torch.float64))
