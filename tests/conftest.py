import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "ref: needs the compiled reference (oracle/_ref)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    return oracle.oracle()


@pytest.fixture(scope="session")
def ref_lib():
    import oracle
    if not oracle.ref_available():
        pytest.skip("reference library not built and /root/reference absent")
    return oracle.ref()
