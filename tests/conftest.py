import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long CPU-reference runs")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle checkers and the CUDA engine once (nvcc cross-compiles)."""
    import __graft_entry__ as g
    g.build_all(quiet=True)
