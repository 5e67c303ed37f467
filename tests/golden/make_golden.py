"""Generate tests/golden/*.npz from the REFERENCE's own code (oracle/_ref/libmacko_ref.so:
/root/reference/proj/src fp16.cpp + bitpack.cpp + headers, plus the SPEC-restated bodies in
oracle/ref_shim.cpp).  Run here, where /root/reference exists; the fixtures are committed so
the GPU box (no /root/reference) can check against them.

Inputs are drawn with numpy's PCG64 (independent of our counter-hash generator) and rounded
to fp16 by the reference float_to_half.  Each case stores: dense, bits, values, deltas,
row_ptrs (reference encoder), x, y_ref (reference reference_spmv), y_dense (dense_mv).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402


def ref_f2h(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float32)
    out = np.zeros(max(a.size, 1), np.uint16)
    O.ref().ref_float_to_half_array(a.reshape(-1), a.size, out)
    return out[: a.size].reshape(a.shape)


def random_dense(rng, R, C, d, int_mode):
    mask = rng.random((R, C)) < d
    if int_mode:
        v = rng.integers(1, 9, (R, C)) * rng.choice([-1, 1], (R, C))
        vals = v.astype(np.float32)
    else:
        vals = rng.normal(0.0, 0.05, (R, C)).astype(np.float32)
        vals[vals == 0] = 1e-3
    dense = ref_f2h(np.where(mask, vals, 0.0))
    # keep "nonzero" entries that rounded to fp16 zero as zeros (csr_from_dense drops them)
    return dense


def random_x(rng, C, int_mode):
    if int_mode:
        return ref_f2h(rng.integers(-8, 9, C).astype(np.float32))
    return ref_f2h(rng.normal(0.0, 1.0, C).astype(np.float32))


def case(name, dense, bits, x, out):
    R, C = dense.shape
    rm = O.RefMatrix.encode(dense, bits)
    m = rm.to_macko(R, C, bits)
    y_ref = rm.spmv(x, R) if bits else None
    y_dense = np.zeros(max(R, 1), np.uint16)
    O.ref().ref_dense_mv(np.ascontiguousarray(dense.reshape(-1)), R, C, x, y_dense)
    out[name] = dict(dense=dense, bits=np.uint32(bits), values=m.values, deltas=m.deltas, row_ptrs=m.row_ptrs,
                     x=x, y_ref=y_ref, y_dense=y_dense[:R])


def main():
    rng = np.random.default_rng(20251113)
    cases = {}
    # SPEC.md:62,70 / PAPER.md:256-258 — Fig. 3 (0-based cols 1,4,11,12), b_delta = 2
    fig3 = np.zeros((1, 14), np.uint16)
    fig3[0, [1, 4, 11, 12]] = ref_f2h(np.array([1, 2, 3, 4], np.float32))
    case("fig3_b2", fig3, 2, ref_f2h(np.ones(14, np.float32)), cases)
    # diagonal and all-zero
    diag = np.zeros((2, 2), np.uint16)
    diag[0, 0], diag[1, 1] = ref_f2h(np.array([1, 2], np.float32))
    case("diag", diag, 4, ref_f2h(np.array([3, 5], np.float32)), cases)
    case("zeros3", np.zeros((3, 3), np.uint16), 4, ref_f2h(np.ones(3, np.float32)), cases)
    # dense row of 16; single nonzero at column 31 of a 1x32 row
    case("dense16", ref_f2h(np.arange(1, 17, dtype=np.float32)[None, :]), 4, random_x(rng, 16, True), cases)
    one31 = np.zeros((1, 32), np.uint16)
    one31[0, 31] = ref_f2h(np.array([7], np.float32))[0]
    case("single31", one31, 4, random_x(rng, 32, True), cases)
    # worst case 1x32: 16 zeros then 16 ones
    wc = np.zeros((1, 32), np.uint16)
    wc[0, 16:] = ref_f2h(np.ones(16, np.float32))
    case("worst1x32", wc, 4, random_x(rng, 32, True), cases)
    # random cases: shapes incl. ragged columns, empty rows, every b_delta, both modes
    specs = [
        ("r17x100_d30", 17, 100, 0.3), ("r64x700_d50", 64, 700, 0.5), ("r33x257_d10", 33, 257, 0.1),
        ("r4x2048_d05", 4, 2048, 0.05), ("r5x37_d100", 5, 37, 1.0), ("r24x600_d90", 24, 600, 0.9),
        ("r3x5_d50", 3, 5, 0.5), ("r1x3000_d02", 1, 3000, 0.02),
    ]
    for name, R, C, d in specs:
        for bits in (1, 2, 4, 8):
            for im in ((False, True) if bits == 4 else (False,)):
                dense = random_dense(rng, R, C, d, im)
                if name == "r24x600_d90":
                    dense[[3, 17, 18, 23], :] = 0  # empty rows
                case(f"{name}_b{bits}_{'int' if im else 'f16'}", dense, bits, random_x(rng, C, im), cases)
    flat = {}
    for k, v in cases.items():
        for f, a in v.items():
            if a is not None:
                flat[f"{k}/{f}"] = np.asarray(a)
    path = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(path, **flat)
    print(f"wrote {len(cases)} cases to {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
