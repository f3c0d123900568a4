"""The C++ shim (include/polydg_b200.hpp) compiles against the C-ABI and runs
a reference-style caller (tests/cpp/shim_demo.cpp)."""
import pathlib
import subprocess

import pytest

from tests.conftest import ROOT, gpu_available

LIBDIR = ROOT / "paper_2512_19536_b200"
EXE = ROOT / "build" / "shim_demo"


def _compile():
    EXE.parent.mkdir(exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "shim_demo.cpp"), "-L", str(LIBDIR), "-lpolydg_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(EXE)], check=True, capture_output=True, text=True)


def test_shim_compiles_and_links():
    _compile()
    assert EXE.exists()


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_shim_runs_reference_style_caller():
    _compile()
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "converged 1" in out.stdout
