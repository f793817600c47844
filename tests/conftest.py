import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libb200sp.so")


def has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    """{case: {key: array}} from tests/golden/<name>.npz (made by the reference)."""
    raw = np.load(os.path.join(GOLDEN, name))
    out = {}
    for key in raw.files:
        case, field = key.split("__", 1)
        out.setdefault(case, {})[field] = raw[key]
    return out


@pytest.fixture(scope="session")
def golden_spmv():
    return load_golden("spmv.npz")


@pytest.fixture(scope="session")
def golden_solvers():
    return load_golden("solvers.npz")


@pytest.fixture(scope="session")
def golden_jacobi():
    return load_golden("jacobi.npz")


@pytest.fixture(scope="session")
def golden_misc():
    return load_golden("misc.npz")


@pytest.fixture(scope="session")
def cuda():
    import paper_2006_16852_b200 as b2

    return b2.CudaExecutor(0)


@pytest.fixture(scope="session")
def host():
    import paper_2006_16852_b200 as b2

    return b2.HostExecutor()


def random_sparse(n, density=0.1, seed=0, diag_dominant=True):
    """Seeded random test matrix (the reference test-suite recipe,
    src/problems.py:48-58), returned as host MatrixData."""
    from paper_2006_16852_b200 import MatrixData

    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, True)
    dense = np.where(mask, rng.uniform(-1.0, 1.0, (n, n)), 0.0)
    if diag_dominant:
        off = np.abs(dense).sum(axis=1) - np.abs(np.diag(dense))
        np.fill_diagonal(dense, off + 1.0)
    return MatrixData.from_dense_array(dense)


def random_spd(n, density=0.2, seed=0):
    from paper_2006_16852_b200 import MatrixData

    rng = np.random.default_rng(seed)
    mask = np.triu(rng.random((n, n)) < density / 2)
    dense = np.where(mask, rng.uniform(-1.0, 1.0, (n, n)), 0.0)
    dense = dense + dense.T
    off = np.abs(dense).sum(axis=1) - np.abs(np.diag(dense))
    np.fill_diagonal(dense, off + 1.0)
    return MatrixData.from_dense_array(dense)
