"""Runs the C++ drop-in program (tests/cpp/dropin_test.cpp): the reference's own C++ types and
encoder feed libmacko_cuda.so through include/macko/macko_cuda.hpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "dropin_test")


@pytest.mark.gpu
def test_cpp_dropin(cuda):
    assert os.path.exists(BIN), "tests/cpp/dropin_test not built (make cpptest)"
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "dropin ok" in out.stdout


def test_cpp_dropin_is_built_and_links_the_library():
    assert os.path.exists(BIN)
    ldd = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libmacko_cuda.so" in ldd and "libmacko_ref.so" in ldd
