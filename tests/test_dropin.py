"""The C++ drop-in header (include/geodock_b200/geodock.hpp).

Compiling tests/cpp/test_dropin.cpp against the header and the in-tree
library is a CPU test; running it (the reference's own test cases through
the GPU) is a GPU test.
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "cpp" / "test_dropin.cpp"
OUT = ROOT / "tests" / "_build" / "test_dropin"
LIBDIR = ROOT / "paper_1901_06363_b200"


def _compile():
    OUT.parent.mkdir(exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", str(ROOT / "include"), str(SRC), "-o", str(OUT),
           "-L", str(LIBDIR), "-lgeodock_b200", f"-Wl,-rpath,{LIBDIR}", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return OUT


def test_dropin_header_compiles_and_links():
    _compile()
    assert OUT.exists()


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu(docker):
    exe = _compile()
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "FAIL" not in res.stdout
