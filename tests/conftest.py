import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test (minutes); runs with HELM_SLOW=1")


def pytest_collection_modifyitems(config, items):
    """Tests marked slow (the h = 2^-9 FD5 paper tables, minutes of splu work)
    run only with HELM_SLOW=1, so the default CPU suite stays a few minutes."""
    if os.environ.get("HELM_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow paper-table pin: set HELM_SLOW=1")
    for item in items:
        if "slow" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def root():
    return ROOT
