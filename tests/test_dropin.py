"""The C++ drop-in headers (include/geodock_b200/{geodock,analysis,formats}.hpp).

Compiling tests/cpp/test_dropin.cpp against the headers and the in-tree
library is a CPU test; running it (the reference's own test cases through
the GPU) is a GPU test.  tests/cpp/test_formats.cpp (file formats, reports,
ligand graph helpers) and tests/cpp/test_planner.cpp (cost model, config
selection, planner files) need no GPU and run in the CPU suite.
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIBDIR = ROOT / "paper_1901_06363_b200"


def _compile(name="test_dropin"):
    src = ROOT / "tests" / "cpp" / f"{name}.cpp"
    out = ROOT / "tests" / "_build" / name
    out.parent.mkdir(exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", str(ROOT / "include"), str(src), "-o", str(out),
           "-L", str(LIBDIR), "-lgeodock_b200", f"-Wl,-rpath,{LIBDIR}", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return out


def test_dropin_header_compiles_and_links():
    assert _compile().exists()


@pytest.mark.parametrize("name", ["test_formats", "test_planner"])
def test_dropin_host_parts_on_cpu(name):
    """File formats, ligand graph helpers and the planner need no GPU."""
    exe = _compile(name)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "FAIL" not in res.stdout


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu(docker):
    exe = _compile()
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "FAIL" not in res.stdout
