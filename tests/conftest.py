import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "embquant"))


@pytest.fixture(scope="session")
def ref():
    """The real reference package, importable only in the build container."""
    if not reference_available():
        pytest.skip("reference not present (GPU box); golden fixtures cover this")
    sys.dont_write_bytecode = True
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import embquant

    return embquant
