"""The reference-facing C++ API (include/fastfca/*.hpp, csrc/shim.cpp) built
and exercised as a C++ program, like the reference's doctest binary."""
import subprocess

import pytest

from conftest import ROOT

BIN = ROOT / "build" / "test_api_gpu"


def compile_test() -> None:
    cmd = ["g++", "-O2", "-std=c++20", "-Wno-class-memaccess",
           "-I", str(ROOT / "include"), "-I", str(ROOT / "oracle"),
           str(ROOT / "tests" / "cpp" / "test_api_gpu.cpp"), str(ROOT / "oracle" / "oracle.cpp"),
           "-L", str(ROOT / "paper_2101_08563_b200"), "-lffca",
           "-Wl,-rpath," + str(ROOT / "paper_2101_08563_b200"), "-pthread", "-o", str(BIN)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_cpp_api_compiles_against_the_library(built):
    BIN.parent.mkdir(exist_ok=True)
    compile_test()
    assert BIN.exists()


@pytest.mark.gpu
def test_cpp_api_on_gpu(built):
    BIN.parent.mkdir(exist_ok=True)
    compile_test()
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout
