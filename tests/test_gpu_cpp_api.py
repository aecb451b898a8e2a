"""The reference's engine test cases through the C++ host API (tests/cpp)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
EXE = Path(__file__).resolve().parent / "cpp" / "test_engine_cpp"


def test_cpp_engine_cases():
    assert EXE.exists(), "run __graft_entry__.build() first"
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
