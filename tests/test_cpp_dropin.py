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


REF_BIN = os.path.join(ROOT, "tests", "cpp", "dropin_ref_test")


@pytest.mark.gpu
def test_cpp_reference_caller_on_libmacko(cuda):
    # the reference's headers + libmacko.so only: fp16 / bitpack / convert / SPEC executors, the
    # worked examples, roundtrips, integer-mode exactness and the reference's exception types
    assert os.path.exists(REF_BIN), "tests/cpp/dropin_ref_test not built (make cpptest)"
    out = subprocess.run([REF_BIN], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "dropin_ref ok" in out.stdout


def test_reference_caller_links_libmacko_without_reference_code():
    assert os.path.exists(REF_BIN)
    ldd = subprocess.run(["ldd", REF_BIN], capture_output=True, text=True).stdout
    assert "libmacko.so" in ldd and "libmacko_cuda.so" in ldd
    assert "libmacko_ref" not in ldd and "oracle" not in ldd
    # libmacko.so defines the reference's API itself (fp16.cpp / bitpack.cpp / convert.cpp surface)
    nm = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(ROOT, "paper_2511_13061_b200", "libmacko.so")],
                        capture_output=True, text=True).stdout
    for sym in ("macko::float_to_half(float)", "macko::half_to_float(macko::Half)", "macko::half_table()",
                "macko::pack_deltas(", "macko::unpack_deltas(", "macko::pack_delta_at(", "macko::is_valid_delta_bits(",
                "macko::csr_from_dense(", "macko::macko_from_csr(", "macko::dense_from_macko(",
                "macko::padding_count(", "macko::validate_csr(", "macko::validate_macko(",
                "macko::reference_spmv(", "macko::dense_mv("):
        assert sym in nm, sym
