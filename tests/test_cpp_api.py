"""The reference-facing C++ API (include/fastfca/*.hpp, csrc/shim.cpp) built
and exercised as a C++ program, like the reference's doctest binary."""
import subprocess

import pytest

from conftest import ROOT

BIN = ROOT / "build" / "test_api_gpu"
STEPS = ROOT / "build" / "test_steps_gpu"


def compile_test(src: str = "test_api_gpu.cpp", out=BIN) -> None:
    cmd = ["g++", "-O2", "-std=c++20", "-Wno-class-memaccess",
           "-I", str(ROOT / "include"), "-I", str(ROOT / "oracle"),
           str(ROOT / "tests" / "cpp" / src), str(ROOT / "oracle" / "oracle.cpp"),
           "-L", str(ROOT / "paper_2101_08563_b200"), "-lffca",
           "-Wl,-rpath," + str(ROOT / "paper_2101_08563_b200"), "-pthread", "-o", str(out)]
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


def test_cpp_step_tests_compile_against_the_library(built):
    """The reference's per-step unit tests (test_fastfca.cpp:82-228), re-stated
    against include/fastfca, compile and link against libffca.so."""
    STEPS.parent.mkdir(exist_ok=True)
    compile_test("test_steps_gpu.cpp", STEPS)
    assert STEPS.exists()


@pytest.mark.gpu
def test_cpp_step_tests_on_gpu(built):
    STEPS.parent.mkdir(exist_ok=True)
    compile_test("test_steps_gpu.cpp", STEPS)
    r = subprocess.run([str(STEPS)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout
