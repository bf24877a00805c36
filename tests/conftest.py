import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libsmoe.so")
    config.addinivalue_line("markers", "reference: imports the read-only reference (CPU box only)")


@pytest.fixture(scope="session")
def moesched():
    """The reference package, imported read-only (absent on the GPU box)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not mounted")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import moesched as m
    return m
