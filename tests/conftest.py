"""Shared fixtures.  `gpu`-marked tests need a B200 (run via gpurun); the rest
run on CPU.  The checkers (oracle/) are imported only from tests."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "energies.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_merged():
    with open(os.path.join(GOLDEN, "merged.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_buckets():
    with open(os.path.join(GOLDEN, "buckets.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_schedule_c1():
    with open(os.path.join(GOLDEN, "schedule_C1.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def q():
    import paper_2204_06045_b200 as q
    return q


@pytest.fixture(scope="session")
def ctx(q):
    return q.Context(0)


def reorder(data, vars_from, vars_to):
    """Tensor data with axes `vars_from` re-laid out with axes `vars_to`."""
    import numpy as np
    r = len(vars_from)
    if list(vars_from) == list(vars_to) or r == 0:
        return np.asarray(data)
    a = np.asarray(data).reshape([2] * r)
    return a.transpose([list(vars_from).index(v) for v in vars_to]).reshape(-1)
