import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    """The CPU oracle (test infrastructure): built on demand, loaded with ctypes."""
    from tests import oracle_lib

    return oracle_lib.load()


@pytest.fixture(scope="session")
def solver():
    """One device context shared by the GPU tests."""
    import paper_2605_08793_b200 as rg

    s = rg.Solver(0)
    yield s
    s.close()
