import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running (full-size configurations)")


_cache = {}


def golden(name):
    if name not in _cache:
        _cache[name] = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    return _cache[name]


def csr(g, key):
    return sp.csr_matrix((g[key + "_data"], g[key + "_indices"], g[key + "_indptr"]),
                         shape=tuple(g[key + "_shape"]))


def rel_l2(a_u, a_v, b_u, b_v):
    num = np.sqrt(np.sum((a_u - b_u) ** 2) + np.sum((a_v - b_v) ** 2))
    den = np.sqrt(np.sum(b_u ** 2) + np.sum(b_v ** 2))
    return num / den if den > 0 else num


SMALL = ("small_coupled2d", "small_square4", "small_cube2")


@pytest.fixture
def rng():
    return np.random.default_rng(20240901)
