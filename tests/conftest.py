import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLD = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs via gpurun")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference itself (oracle/_ref), only where it was built."""
    from pyoracle import REF_SO, Ref
    if not os.path.exists(REF_SO) and not os.path.isdir("/root/reference/proj"):
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return Ref()


@pytest.fixture(scope="session")
def small_golden():
    with open(os.path.join(GOLD, "small.json")) as f:
        return json.load(f)


def load_golden(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def prl():
    """The product package (GPU tests only)."""
    import paper_2108_02997_b200 as p
    return p
