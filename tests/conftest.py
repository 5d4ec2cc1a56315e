import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libgeoheat_b200.so")
    config.addinivalue_line("markers", "slow: full-size parity runs")


@pytest.fixture(scope="session")
def port_oracle():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def gpu():
    """The CUDA path; a GPU test fails (never skips to a CPU path) if it is unusable."""
    import paper_1812_06060_b200 as gh
    n = gh.geoheat.device_count()
    assert n > 0, "no CUDA device visible to libgeoheat_b200.so"
    return gh


@pytest.fixture
def zero_skipping(gpu):
    """The opt-in exact-zero skipping on for one test; off again afterwards (the default)."""
    gpu.set_zero_level_truncation(True)
    yield gpu
    gpu.set_zero_level_truncation(False)
