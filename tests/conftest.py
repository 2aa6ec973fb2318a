import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    import pyoracle
    return pyoracle.restatement()


@pytest.fixture(scope="session")
def reference():
    import pyoracle
    if not pyoracle.reference_available():
        pytest.skip("oracle/_ref/libccwref.so not built")
    return pyoracle.reference()
