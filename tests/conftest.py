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


REF_INSTALL = ROOT / "baseline" / "_ref"   # pip-installed reference (git-ignored; travels to the GPU box)


def reference_sys_path():
    """Directory holding the unmodified reference package: the build
    container's source tree, else the installed copy under baseline/_ref
    (the GPU box has only the latter).  None when neither exists."""
    for p in (REFERENCE_SRC, REF_INSTALL):
        if (p / "persistkern" / "__init__.py").exists():
            return p
    return None


@pytest.fixture(scope="session")
def refpkg():
    """The unmodified reference package from wherever it is available here."""
    p = reference_sys_path()
    if p is None:
        pytest.skip("reference package not available")
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))
    import persistkern  # noqa: F401
    from persistkern import bench, cli
    return {"bench": bench, "cli": cli, "path": p}
