import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "reference: needs the read-only reference checkout (build container only)")
    config.addinivalue_line("markers", "slow: long-running")


def has_reference() -> bool:
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture(scope="session")
def ref_pipesched():
    """The reference package, imported read-only (skips when absent, e.g. on the GPU box)."""
    if not has_reference():
        pytest.skip("reference checkout not present")
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import importlib
    return importlib.import_module("pipesched")
