import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: full-size CPU oracle runs (tens of seconds)")


@pytest.fixture(scope="session")
def golden_chunks():
    with open(os.path.join(GOLDEN, "chunks.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_large():
    with open(os.path.join(GOLDEN, "large.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_dwt():
    return dict(np.load(os.path.join(GOLDEN, "dwt.npz")))


@pytest.fixture(scope="session")
def golden_spiht():
    return dict(np.load(os.path.join(GOLDEN, "spiht.npz")))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.build()
    return o
