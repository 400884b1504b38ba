import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as r
    if not r.available():
        pytest.skip("reference oracle library not built (make -C oracle ref)")
    return r


@pytest.fixture(scope="session")
def dev():
    from paper_2501_07904_b200 import api
    from paper_2501_07904_b200._native import lib
    if lib().ttg_device_count() < 1:
        pytest.fail("GPU test collected but no CUDA device is visible")
    return api
