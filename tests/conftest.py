import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large inputs (seconds to minutes)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure every native artefact is compiled (cheap when up to date)."""
    import __graft_entry__

    __graft_entry__.build()
