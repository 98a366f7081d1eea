"""The reference-facing C++ host API (include/ballmatch_b200.hpp): compiles and
links against libballmatch_b200 + the oracle here; on a GPU the C++ parity
program (tests/cpp/test_shim.cpp) must pass against the oracle's C++ API."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CPP = ROOT / "tests" / "cpp"


def _build():
    subprocess.run(["make", "-C", str(ROOT / "oracle")], check=True, capture_output=True)
    r = subprocess.run(["make", "-C", str(CPP)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return CPP / "_build" / "test_shim"


def test_cpp_shim_compiles_and_links():
    exe = _build()
    assert exe.exists()


@pytest.mark.gpu
def test_cpp_shim_parity_on_device(cuda_device):
    exe = _build()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
