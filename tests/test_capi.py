"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/macko_cuda.h
declares, and the host-only entry points behave like the reference (error taxonomy, shard
arithmetic, density threshold).  No kernel is launched here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2511_13061_b200 import _lib
from paper_2511_13061_b200 import macko as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "macko_cuda.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(macko_[a-z_]+)\s*\(", hdr)))


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 16
    for s in syms:
        assert hasattr(L, s), f"libmacko_cuda.so does not export {s}"
    assert set(syms) == set(_lib.EXPORTS)
    assert "sm_100a" in M.version()


def test_library_is_sm100a_cubin():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_density_threshold_matches_oracle():
    from oracle import oracle as O

    for d in (0.0, 0.05, 0.3, 0.5, 0.7, 0.9, 0.123456, 1.0, 1.5, -1.0):
        assert M.density_threshold(d) == O.density_threshold(d)


def test_shard_rows():
    for R in (4096, 36864, 131072, 7):
        for n in (1, 2, 4, 8):
            bounds = [M.shard_rows(R, n, g) for g in range(n)]
            assert bounds[0][0] == 0 and bounds[-1][1] == R
            assert all(bounds[i][1] == bounds[i + 1][0] for i in range(n - 1))
    with pytest.raises(ValueError):
        M.shard_rows(10, 0, 0)
    with pytest.raises(ValueError):
        M.shard_rows(10, 2, 2)


def test_upload_rejects_bad_arguments_before_touching_the_device():
    L = _lib.load()
    h = C.c_void_p()
    rp = np.array([0, 2], np.uint32)
    v = np.zeros(8, np.uint16)
    d = np.zeros(16, np.uint8)
    # b_delta not in {1,2,4,8}: std::invalid_argument (bitpack.cpp:14-15)
    with pytest.raises(ValueError, match="delta width"):
        _lib.check(L.macko_dev_upload(0, 1, 4, 3, v.ctypes.data, 8, d.ctypes.data, 16, rp.ctypes.data, None, C.byref(h)))
    # non-monotone row pointers: FormatError
    bad = np.array([0, 5, 3], np.uint32)
    with pytest.raises(M.FormatError):
        _lib.check(L.macko_dev_upload(0, 2, 4, 4, v.ctypes.data, 8, d.ctypes.data, 16, bad.ctypes.data, None, C.byref(h)))
    # payload shorter than pad_nnz: FormatError
    with pytest.raises(M.FormatError):
        _lib.check(L.macko_dev_upload(0, 1, 4, 4, v.ctypes.data, 1, d.ctypes.data, 16, rp.ctypes.data, None, C.byref(h)))
    # empty shape
    with pytest.raises(ValueError):
        _lib.check(L.macko_dev_upload(0, 0, 4, 4, v.ctypes.data, 8, d.ctypes.data, 16, rp.ctypes.data, None, C.byref(h)))


def test_null_handles_are_einval():
    L = _lib.load()
    assert L.macko_dev_spmv(None, None, None, None) == _lib.MACKO_EINVAL
    assert L.macko_dev_free(None) == _lib.MACKO_OK
    with pytest.raises(ValueError):
        _lib.check(L.macko_dev_get_info(None, None))


def test_package_has_no_cpu_fallback_or_oracle_import():
    pkg = os.path.join(ROOT, "paper_2511_13061_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(from|import)\s+oracle|libmacko_oracle|libmacko_ref|_ref/", src), f


def test_unit_steps_is_the_documented_reduction_unit():
    # the oracle's unit_steps for the kernel's fixed summation order (csrc/common.cuh kUnitSteps)
    from paper_2511_13061_b200 import macko as M

    assert M.unit_steps() == 16
