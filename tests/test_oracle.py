"""Pinning the CPU oracle (oracle/macko_oracle.c) against the reference.

* fp16 / bit packing: against the reference's own fp16.cpp / bitpack.cpp (oracle/_ref) and
  numpy's IEEE conversion;
* encoder / decoder / SpMV: against the golden vectors produced by the reference code path
  (tests/golden/make_golden.py) and SPEC.md's worked examples and acceptance criteria.
"""
import itertools

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


# ------------------------------------------------------------------------------------ fp16
def test_half_to_float_all_codes_match_reference():
    codes = np.arange(65536, dtype=np.uint16)
    mine = O.half_to_float_array(codes).view(np.uint32)
    ref = np.zeros(65536, np.float32)
    O.ref().ref_half_to_float_array(codes, 65536, ref)  # array form: no sNaN quieting via ctypes
    ref = ref.view(np.uint32)
    assert np.array_equal(mine, ref)
    finite = (codes & 0x7C00) != 0x7C00
    assert np.array_equal(mine[finite], codes[finite].view(np.float16).astype(np.float32).view(np.uint32))


def _ref_f2h(x):
    out = np.zeros(x.size, np.uint16)
    O.ref().ref_float_to_half_array(np.ascontiguousarray(x, np.float32), x.size, out)
    return out


def test_float_to_half_matches_reference_on_2pow24_patterns():
    # every 256th bit pattern over all 2^32 (exponent/sign/NaN/subnormal ranges all covered),
    # plus the exact neighbourhood of every rounding boundary class
    rng = np.random.default_rng(1)
    pats = (np.arange(1 << 24, dtype=np.uint64) << 8).astype(np.uint32) | rng.integers(0, 256, 1 << 24, dtype=np.uint32)
    x = pats.view(np.float32)
    assert np.array_equal(O.float_to_half_array(x), _ref_f2h(x))


def test_float_to_half_rounding_boundaries():
    # halfway points between consecutive fp16 values (ties-to-even) and one ulp either side
    h = np.arange(0, 0x7C00, dtype=np.uint16)
    lo = h[:-1].view(np.float16).astype(np.float64)
    hi = h[1:].view(np.float16).astype(np.float64)
    mid = ((lo + hi) / 2).astype(np.float32)
    cand = np.concatenate([mid, np.nextafter(mid, np.float32(0)), np.nextafter(mid, np.float32(np.inf))])
    cand = np.concatenate([cand, -cand, np.float32([65504, 65519.996, 65520, 65536, 2.0**-24, 2.0**-25, 2.0**-26])])
    mine = O.float_to_half_array(cand)
    assert np.array_equal(mine, _ref_f2h(cand))
    assert np.array_equal(mine, cand.astype(np.float16).view(np.uint16))  # IEEE RNE witness


# ------------------------------------------------------------------------------------ bitpack
def test_pack_known_answers():
    # SPEC.md:91-92
    assert O.pack_deltas([2, 3], 4).tolist() == [0x21]
    assert O.pack_deltas([16], 8).tolist() == [0x0F]
    # Fig. 3, b_delta = 2
    assert O.pack_deltas([2, 3, 4, 3, 1], 2).tolist() == [0xB9, 0x00]


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_pack_unpack_match_reference(bits):
    rng = np.random.default_rng(bits)
    for n in (0, 1, 7, 8, 9, 33, 1000):
        d = rng.integers(1, (1 << bits) + 1, n).astype(np.uint32)
        mine = O.pack_deltas(d, bits)
        ref = np.zeros(max(len(mine), 1), np.uint8)
        assert O.ref().ref_pack_deltas(np.ascontiguousarray(d), n, bits, ref, len(ref)) == 0
        assert np.array_equal(mine, ref[: len(mine)])
        assert np.array_equal(O.unpack_deltas(mine, n, bits), d)


def test_pack_rejects_bad_input_like_reference():
    for bad_bits in (0, 3, 5, 16):
        with pytest.raises(O.OracleError):
            O.pack_deltas([1], bad_bits)
        assert O.ref().ref_pack_deltas(np.ones(1, np.uint32), 1, bad_bits, np.zeros(4, np.uint8), 4) == 1
    for bad in ([0], [17]):
        with pytest.raises(O.OracleError):
            O.pack_deltas(bad, 4)
        assert O.ref().ref_pack_deltas(np.array(bad, np.uint32), 1, 4, np.zeros(4, np.uint8), 4) == 1


# ------------------------------------------------------------------------------------ golden vectors
def test_golden_vectors_encoder_and_spmv(golden):
    assert len(golden) >= 40
    for name, c in golden.items():
        bits = int(c["bits"])
        m = O.encode_dense(c["dense"], bits)
        assert np.array_equal(m.row_ptrs, c["row_ptrs"]), name
        assert np.array_equal(m.values, c["values"]), name
        assert np.array_equal(m.deltas, c["deltas"]), name
        assert np.array_equal(O.dense_from_macko(m), c["dense"]), name
        O.validate_macko(m)
        assert np.array_equal(O.reference_spmv(m, c["x"]), c["y_ref"]), name
        assert np.array_equal(O.dense_mv(c["dense"], c["x"]), c["y_dense"]), name
        if name.endswith("_int"):
            # integer mode is order independent -> every executor bit-exact
            assert np.array_equal(c["y_ref"], c["y_dense"]), name
            assert np.array_equal(O.warp_spmv(m, c["x"]), c["y_ref"]), name
            assert np.array_equal(O.b200_order_spmv(m, c["x"], 4), c["y_ref"]), name


def test_fig3_worked_example(golden):
    c = golden["fig3_b2"]
    m = O.encode_dense(c["dense"], 2)
    assert m.pad_nnz == 5 and O.padding_count(m) == 1
    assert [O.half_to_float(int(v)) for v in m.values[:5]] == [1.0, 2.0, 0.0, 3.0, 4.0]
    assert O.unpack_deltas(m.deltas, 5, 2).tolist() == [2, 3, 4, 3, 1]
    assert O.half_to_float(int(O.reference_spmv(m, c["x"])[0])) == 10.0


def test_spec_examples():
    one = O.float_to_half(1.0)
    # csr_from_dense
    d = np.array([[one, 0], [0, O.float_to_half(2.0)]], np.uint16)
    vals, cols, rp = O.csr_from_dense(d)
    assert cols.tolist() == [0, 1] and rp.tolist() == [0, 1, 2]
    vals, cols, rp = O.csr_from_dense(np.zeros((3, 3), np.uint16))
    assert len(vals) == 0 and rp.tolist() == [0, 0, 0, 0]
    # -0 is dropped as zero
    assert O.encode_dense(np.array([[0x8000, one]], np.uint16)).pad_nnz == 1
    # dense row of 16 -> no pads, all deltas 1
    m = O.encode_dense(np.full((1, 16), one, np.uint16), 4)
    assert O.padding_count(m) == 0 and O.unpack_deltas(m.deltas, 16, 4).tolist() == [1] * 16
    # 1x32 single nonzero at 31 -> one pad at 15, then delta 16
    row = np.zeros((1, 32), np.uint16)
    row[0, 31] = one
    m = O.encode_dense(row, 4)
    assert m.pad_nnz == 2 and O.unpack_deltas(m.deltas, 2, 4).tolist() == [16, 16]
    # macko_from_csr rejects out-of-range / non-increasing columns
    with pytest.raises(O.OracleError):
        O.macko_from_csr(1, 4, [one, one], [2, 1], [0, 2], 4)
    with pytest.raises(O.OracleError):
        O.macko_from_csr(1, 4, [one], [4], [0, 1], 4)
    # payload sizes with 16-byte tails (matrix.hpp:77-81)
    assert O.values_bytes(5) == 16 and O.delta_bytes(5, 2) == 16 and O.delta_bytes(33, 4) == 32


def test_worst_case_eq9_exact():
    # SPEC.md:171-179, acceptance 4: padding_count = R*C*(1-d)/2^b for zero runs of 2^b
    for bits in (1, 2, 4):
        run = 1 << bits
        for R, reps in ((1, 1), (64, 16), (7, 5)):
            C = reps * (run + 1)
            m = O.encode_dense(O.gen_worst_case(R, C, run), bits)
            assert O.padding_count(m) == R * reps
    m = O.encode_dense(O.gen_worst_case(64, 4096 * 17 // 16, 16), 4)
    assert O.padding_count(m) == 64 * 256


def _min_pads_bruteforce(cols_nz, maxd):
    """Fewest padding entries over ALL valid encodings: enumerate every subset of
    zero columns before the last nonzero, keep those whose entry sequence (from the virtual
    column -1) has all gaps in [1, maxd]."""
    last = cols_nz[-1]
    zeros = [c for c in range(last) if c not in cols_nz]
    best = None
    for k in range(len(zeros) + 1):
        for pads in itertools.combinations(zeros, k):
            seq = sorted(cols_nz + list(pads))
            prev, ok = -1, True
            for c in seq:
                if c - prev > maxd:
                    ok = False
                    break
                prev = c
            if ok:
                return k
    return best


def test_greedy_padding_is_minimal_exhaustive():
    one = O.float_to_half(1.0)
    for bits in (1, 2):
        maxd = 1 << bits
        for C in range(1, 11):
            for mask in range(1, 1 << C):
                cols_nz = [c for c in range(C) if mask >> c & 1]
                row = np.zeros((1, C), np.uint16)
                row[0, cols_nz] = one
                m = O.encode_dense(row, bits)
                assert O.padding_count(m) == _min_pads_bruteforce(cols_nz, maxd)


def test_random_roundtrip_and_reference_equivalence():
    # acceptance 2 (losslessness) at reduced count, and bit-equality with the reference path
    rng = np.random.default_rng(7)
    for i in range(150):
        R, C = int(rng.integers(1, 40)), int(rng.integers(1, 300))
        d = float(rng.choice([0.0, 0.05, 0.3, 0.5, 0.7, 0.95, 1.0]))
        bits = int(rng.choice([1, 2, 4, 8]))
        A = O.gen_dense(R, C, d, i, bool(i & 1))
        m = O.encode_dense(A, bits)
        r = O.RefMatrix.encode(A, bits).to_macko(R, C, bits)
        assert np.array_equal(m.values, r.values) and np.array_equal(m.deltas, r.deltas)
        assert np.array_equal(m.row_ptrs, r.row_ptrs)
        assert np.array_equal(O.dense_from_macko(m), A)
        vals, cols, rp = O.csr_from_dense(A)
        m2 = O.macko_from_csr(R, C, vals, cols, rp, bits)
        assert np.array_equal(m2.values, m.values) and np.array_equal(m2.deltas, m.deltas)


def test_integer_mode_executors_bit_exact():
    # acceptance 3 (reduced count): warp_spmv = reference_spmv = dense_mv in integer mode
    for i in range(60):
        rng = np.random.default_rng(100 + i)
        R, C = int(rng.integers(1, 30)), int(rng.integers(1, 2000))
        A = O.gen_dense(R, C, float(rng.choice([0.02, 0.2, 0.5, 1.0])), i, True)
        if i % 5 == 0:
            A[::3] = 0
        x = O.gen_vector(C, 1000 + i, True)
        m = O.encode_dense(A, 4)
        y = O.dense_mv(A, x)
        assert np.array_equal(O.reference_spmv(m, x), y)
        assert np.array_equal(O.warp_spmv(m, x), y)
        assert np.array_equal(O.b200_order_spmv(m, x, 4), y)
        assert np.array_equal(O.reference_spmv(m, x, 4), y)


def test_warp_prefix_sum_algorithm1():
    # acceptance 8
    rng = np.random.default_rng(3)
    assert O.warp_prefix_sum(np.ones(32)).tolist() == list(range(32))
    for _ in range(10000 // 50):
        v = rng.integers(0, 200, 32).astype(np.uint32)
        ex = O.warp_prefix_sum(v)
        assert np.array_equal(ex, np.concatenate([[0], np.cumsum(v)[:-1]]).astype(np.uint32))
        assert ex[31] + v[31] == v.sum()


def tol_bound(A, x, y_ref):
    """|dy| <= ulp16(|y_ref|) + 2*n*2^-24*sum|a_i x_i|."""
    a = A.view(np.float16).astype(np.float64)
    xf = x.view(np.float16).astype(np.float64)
    s = np.abs(a) @ np.abs(xf)
    n = (A & 0x7FFF != 0).sum(axis=1)
    yr = y_ref.view(np.float16).astype(np.float64)
    ulp = np.spacing(np.abs(y_ref.view(np.float16))).astype(np.float64)
    return ulp + 2 * n * 2.0**-24 * s, yr


def test_float_mode_error_budget_4096():
    # acceptance 9: B200 order vs sequential reference within the stated bound
    A = O.gen_dense(4096, 4096, 0.5, 11)
    x = O.gen_vector(4096, 12)
    m = O.encode_dense(A)
    y_seq = O.reference_spmv(m, x, 8)
    y_b200 = O.b200_order_spmv(m, x, 4)
    y_warp = O.warp_spmv(m, x)
    bound, yr = tol_bound(A, x, y_seq)
    for y in (y_b200, y_warp):
        dy = np.abs(y.view(np.float16).astype(np.float64) - yr)
        assert (dy <= bound).all()
    assert np.array_equal(O.b200_order_spmv(m, x, 0), y_warp)


def _b200_py(m, x, unit_steps=8):
    """Pure-Python restatement of the kernel's summation order (small cases): the
    row's walk starts at its 8-aligned element al (ROMA); element i goes to lane
    ((i - al) mod 256) / 8 of step (i - al) / 256; steps form units of unit_steps (the row's last
    unit absorbs a shorter remainder); per unit the 32 lane sums are reduced by the xor butterfly
    and the unit totals are added in order (+0 start); one RNE at the end."""
    h = lambda a: np.float32(np.uint16(a).view(np.float16))
    codes = O.unpack_deltas(m.deltas, m.pad_nnz, m.b_delta)
    y = np.zeros(m.rows, np.uint16)
    for r in range(m.rows):
        s, e = int(m.row_ptrs[r]), int(m.row_ptrs[r + 1])
        al = s & ~7
        T = (e - al + 255) // 256 if e > s else 0
        n_r = T // unit_steps if T >= unit_steps else 1
        col, tot = -1, np.float32(0)
        for j in range(n_r if T else 0):
            lo_step, hi_step = j * unit_steps, (T if j == n_r - 1 else (j + 1) * unit_steps)
            acc = [np.float32(0)] * 32
            for i in range(max(s, al + 256 * lo_step), min(e, al + 256 * hi_step)):
                col += int(codes[i])
                ln = ((i - al) % 256) // 8
                acc[ln] = np.float32(acc[ln] + h(m.values[i]) * h(x[col]))
            for k in (16, 8, 4, 2, 1):
                acc = [np.float32(acc[q] + acc[q ^ k]) for q in range(32)]
            tot = np.float32(tot + acc[0])
        y[r] = np.float16(tot).view(np.uint16)
    return y


def test_b200_order_restatement():
    # the C restatement of the kernel's summation order (mo_b200_order_spmv) == the Python one, on
    # rows that start at every alignment mod 8, span several units, and are empty
    for seed, (R, C, d) in enumerate(((3, 9000, 0.6), (40, 700, 0.5), (5, 5000, 1.0), (9, 64, 0.3), (2, 20000, 0.2))):
        A = O.gen_dense(R, C, d, 300 + seed)
        A[R // 2] = 0
        x = O.gen_vector(C, 400 + seed)
        m = O.encode_dense(A)
        assert np.array_equal(O.b200_order_spmv(m, x, 8), _b200_py(m, x, 8)), (R, C, d)
        assert np.array_equal(O.b200_order_spmv(m, x, 2), _b200_py(m, x, 2)), (R, C, d)
        assert np.array_equal(O.b200_order_spmv(m, x, 16), _b200_py(m, x, 16)), (R, C, d)


def test_slab_encoding_equals_global_slice():
    # encoding rows [r0, r1) standalone = global encoding sliced
    A = O.gen_dense(64, 333, 0.4, 5)
    g = O.encode_dense(A, 4)
    for r0, r1 in ((0, 32), (32, 64), (5, 17)):
        s = O.encode_dense(A[r0:r1], 4)
        base = int(g.row_ptrs[r0])
        assert np.array_equal(s.row_ptrs, g.row_ptrs[r0 : r1 + 1] - base)
        n = s.pad_nnz
        assert np.array_equal(s.values[:n], g.values[base : base + n])
        gd = O.unpack_deltas(g.deltas, g.pad_nnz, 4)[base : base + n]
        assert np.array_equal(O.unpack_deltas(s.deltas, n, 4), gd)


def test_generator_density_and_determinism():
    A = O.gen_dense(1024, 4096, 0.5, 99)
    d = (A & 0x7FFF != 0).mean()
    assert abs(d - 0.5) < 3 * np.sqrt(0.25 / A.size)
    assert np.array_equal(A, O.gen_dense(1024, 4096, 0.5, 99))
    assert (O.gen_dense(8, 8, 0.0, 1) == 0).all() and (O.gen_dense(8, 8, 1.0, 1) != 0).all()


def test_traffic_definition():
    # SPEC.md:339 and :447
    assert O.dense_traffic_bytes(12288, 12288) - 2 * 12288 * 2 == 301989888
    m = O.encode_dense(O.gen_dense(64, 512, 0.5, 1))
    assert O.spmv_traffic_bytes(64, 512, m.pad_nnz, 4) == len(m.values) * 2 + len(m.deltas) + 4 * 65 + 2 * 512 + 2 * 64
