import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly when selected without a device; never skip silently
    # on a GPU box. Here (no GPU) they are deselected by `-m "not gpu"`.
    pass


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the in-tree library and the oracle once per session."""
    from paper_2005_05826_b200 import build
    build.build_all()
    yield
