import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the native libraries in-tree once per session (no-op when up to date)."""
    from paper_1912_10024_b200.build import build
    only = None if os.environ.get("QT_SKIP_CUDA_BUILD") is None else ["qtgen_host", "oracle"]
    build(only=only)
    yield
