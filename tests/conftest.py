import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through the C-ABI library")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure the oracle and the product library exist (build is cheap when up to date)."""
    import subprocess
    for d in ("oracle", "paper_1612_09447_b200"):
        path = os.path.join(ROOT, d)
        lib = "liboracle.so" if d == "oracle" else "libeqs_b200.so"
        if not os.path.exists(os.path.join(path, lib)):
            subprocess.run(["make", "-C", path, "-j8"], check=True, stdout=subprocess.DEVNULL)
    yield
