import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# featlsq (the host framework the drop-in plugs into) from sys.path or baseline/_ref
import paper_2506_17626_b200._featlsq  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (still CPU-only unless also gpu)")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
