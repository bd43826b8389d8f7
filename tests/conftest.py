import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: large configuration")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def random_connected_graph_edges(n, rng, extra_edge_prob=0.15, weighted=False):
    """Random spanning tree plus Bernoulli extra edges (the recipe of the
    reference fixture pkg/tests/conftest.py:7-21).  Returns (u, v, w)."""
    us, vs = [], []
    for v in range(1, n):
        us.append(int(rng.integers(v)))
        vs.append(v)
    iu, iv = np.nonzero(np.triu(rng.random((n, n)) < extra_edge_prob, 1))
    us += iu.tolist()
    vs += iv.tolist()
    w = rng.uniform(0.2, 3.0, size=len(us)) if weighted else np.ones(len(us))
    return np.asarray(us), np.asarray(vs), w


def dense_pinv_resistance(lap_dense):
    p = np.linalg.pinv(lap_dense)
    d = np.diag(p)
    return d[:, None] + d[None, :] - 2.0 * p


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
