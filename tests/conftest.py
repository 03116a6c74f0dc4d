import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtidq.so")


@pytest.fixture(scope="session")
def golden():
    from helpers import load_golden

    return load_golden()


@pytest.fixture(scope="session")
def gpu():
    """The libtidq context on cuda:0; GPU tests fail loudly without it."""
    from paper_1807_01409_b200 import _lib

    return _lib.context(0)
