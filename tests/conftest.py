import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: long-running stress test")


@pytest.fixture(scope="session")
def reference():
    """The live reference package, only in the build container (never on the GPU box)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not present on this machine")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import persistkern  # noqa: F401
    from persistkern import native, protocol
    return {"native": native, "protocol": protocol}
