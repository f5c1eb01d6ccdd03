import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")
    config.addinivalue_line("markers", "slow: long-running case")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden():
    return load_golden("reference_goldens.json")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def sieve():
    import paper_2310_17746_b200 as ws
    s = ws.Sieve()
    yield s
    s.close()


@pytest.fixture(scope="session")
def sieve12():
    import paper_2310_17746_b200 as ws
    s = ws.Sieve(segment_slots=1 << 12)
    yield s
    s.close()
