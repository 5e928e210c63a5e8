"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def built():
    """Builds the checkers (and the product library if stale) once per session."""
    from paper_1510_03560_b200 import build
    build.build_oracle()
    return True


def have_ref() -> bool:
    from paper_1510_03560_b200 import capi
    return os.path.exists(capi.REF_LIB)
