import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large instances")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref) — the parity checker."""
    from oracle import ref as r
    r.lib()
    return r
