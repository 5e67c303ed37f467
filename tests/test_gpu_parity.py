"""GPU parity: libmacko_cuda.so on cuda:0 against the CPU oracle and the reference's golden
vectors.  Every check here goes through the C-ABI (ctypes) — the same entry points a C/C++
caller binds.

Bars: format (values / packed deltas / row pointers, tails included) bit-exact; y bit-exact in
integer mode; in float mode bit-exact against the oracle's emulation of the kernel's summation
order (oracle mo_b200_order_spmv, tests.helpers.b200_y)
AND within the stated bound of the sequential reference.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2511_13061_b200 import macko as M
from tests.helpers import UNIT_STEPS, b200_y, to_dev, to_host_u16, within_bound

pytestmark = pytest.mark.gpu


def gpu_encode(dense: np.ndarray, bits: int = 4, ld_pad: int = 0) -> M.DeviceMatrix:
    R, C = dense.shape
    if ld_pad:
        buf = np.zeros((R, C + ld_pad), np.uint16)
        buf[:, :C] = dense
        t = to_dev(buf)[:, :C]
    else:
        t = to_dev(dense)
    dm = M.DeviceMatrix.from_dense(t, b_delta=bits)
    torch.cuda.synchronize()
    return dm


def assert_same_format(dm: M.DeviceMatrix, m: O.Macko, ctx=""):
    h = dm.download()
    assert np.array_equal(h.row_pointers, m.row_ptrs), ctx
    assert np.array_equal(h.values, m.values), ctx
    assert np.array_equal(h.packed_deltas, m.deltas), ctx


def gpu_spmv(dm: M.DeviceMatrix, x: np.ndarray) -> np.ndarray:
    xd = to_dev(x)
    y = M.spmv(dm, xd)
    torch.cuda.synchronize()
    return to_host_u16(y)


def check_y(dense, m, x, y, int_mode, ctx=""):
    if int_mode:
        assert np.array_equal(y, O.reference_spmv(m, x, 8)), ctx
    else:
        assert np.array_equal(y, b200_y(m, x)), ctx
        assert within_bound(dense, x, y, O.reference_spmv(m, x, 8)), ctx


# ------------------------------------------------------------------------------ generator
@pytest.mark.parametrize("int_mode", [False, True])
def test_generator_bit_identical(cuda, int_mode):
    for R, C, d, row0 in ((7, 37, 0.5, 0), (64, 4096, 0.3, 5), (3, 8, 1.0, 1000), (16, 1000, 0.05, 0)):
        t = torch.empty((R, C + 3), dtype=torch.float16, device=cuda)[:, :C]
        M.gen_dense(t, R, C, d, seed=42, int_mode=int_mode, row0=row0)
        ref = O.gen_dense(row0 + R, C, d, 42, int_mode)[row0:]
        assert np.array_equal(to_host_u16(t), ref)
    v = torch.empty(12345, dtype=torch.float16, device=cuda)
    M.gen_vector(v, 12345, 7, int_mode)
    assert np.array_equal(to_host_u16(v), O.gen_vector(12345, 7, int_mode))


# ------------------------------------------------------------------------------ compressor
def test_compressor_reproduces_reference_golden_vectors(cuda, golden):
    for name, c in golden.items():
        bits = int(c["bits"])
        dm = gpu_encode(c["dense"], bits)
        h = dm.download()
        assert np.array_equal(h.row_pointers, c["row_ptrs"]), name
        assert np.array_equal(h.values, c["values"]), name
        assert np.array_equal(h.packed_deltas, c["deltas"]), name


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_compressor_random_vs_oracle(cuda, bits):
    rng = np.random.default_rng(bits)
    shapes = [(1, 1), (1, 7), (2, 9), (31, 255), (33, 257), (5, 4096), (200, 513), (64, 1000)]
    for i, (R, C) in enumerate(shapes):
        for d in (0.0, 0.02, 0.3, 0.5, 0.9, 1.0):
            A = O.gen_dense(R, C, d, 1000 * bits + i, bool(i & 1))
            if R > 4:
                A[rng.integers(0, R, R // 4)] = 0  # empty rows
            m = O.encode_dense(A, bits)
            dm = gpu_encode(A, bits, ld_pad=(i % 3) * 8 + (i % 2))
            assert_same_format(dm, m, (R, C, d, bits))


def test_compressor_edge_patterns(cuda):
    one = O.float_to_half(1.0)
    pats = []
    wc = O.gen_worst_case(64, 4096 * 17 // 16, 16)  # Eq. 9 worst case
    pats.append(wc)
    r = np.zeros((3, 64), np.uint16)
    r[0, 63] = one      # single far nonzero (3 pads)
    r[1, 0] = one       # first column
    r[2, 16] = 0x8000   # -0 is dropped
    pats.append(r)
    alt = np.zeros((4, 300), np.uint16)
    alt[:, ::17] = one  # every gap forces exactly one pad
    pats.append(alt)
    for A in pats:
        for bits in (1, 2, 4, 8):
            assert_same_format(gpu_encode(A, bits), O.encode_dense(A, bits), (A.shape, bits))


# ------------------------------------------------------------------------------ SpMV
def test_spmv_on_reference_golden_vectors(cuda, golden):
    n = 0
    for name, c in golden.items():
        if int(c["bits"]) != 4:
            continue
        m = O.Macko(c["dense"].shape[0], c["dense"].shape[1], 4, c["values"], c["deltas"], c["row_ptrs"])
        dm = M.DeviceMatrix.upload(M.MackoMatrix(m.rows, m.cols, 4, m.values, m.deltas, m.row_ptrs))
        y = gpu_spmv(dm, c["x"])
        if name.endswith("_int") or name in ("fig3_b2", "diag", "zeros3", "dense16", "single31", "worst1x32"):
            assert np.array_equal(y, c["y_ref"]), name
        else:
            assert np.array_equal(y, b200_y(m, c["x"])), name
            assert within_bound(c["dense"], c["x"], y, c["y_ref"]), name
        n += 1
    assert n >= 10


@pytest.mark.parametrize("int_mode", [True, False])
def test_spmv_random_shapes(cuda, int_mode):
    cases = [
        (1, 1, 1.0), (1, 5, 0.5), (3, 16, 1.0), (7, 37, 0.5), (100, 100, 0.3), (33, 4097, 0.5),
        (1, 65536, 0.5),       # one long row split across many warps
        (2, 30000, 0.9),       # two long rows
        (17, 20000, 0.02),     # sparse long rows (padding heavy)
        (512, 300, 0.7), (4096, 64, 0.5),  # many short rows
        (1000, 2048, 0.0),     # all-empty matrix
    ]
    for i, (R, C, d) in enumerate(cases):
        A = O.gen_dense(R, C, d, 77 + i, int_mode)
        if R >= 8:
            A[3::7] = 0
        x = O.gen_vector(C, 99 + i, int_mode)
        m = O.encode_dense(A)
        dm = gpu_encode(A)
        check_y(A, m, x, gpu_spmv(dm, x), int_mode, (R, C, d))


@pytest.mark.parametrize("R,C", [(4096, 4096), (11008, 4096), (4096, 11008)])
def test_spmv_llama_shapes(cuda, R, C):
    for int_mode in (False, True):
        t = torch.empty((R, C), dtype=torch.float16, device=cuda)
        M.gen_dense(t, R, C, 0.5, seed=5, int_mode=int_mode)
        dm = M.DeviceMatrix.from_dense(t)
        A = O.gen_dense(R, C, 0.5, 5, int_mode)
        m = O.encode_dense(A)
        assert_same_format(dm, m, (R, C))
        x = O.gen_vector(C, 6, int_mode)
        check_y(A, m, x, gpu_spmv(dm, x), int_mode, (R, C))


def test_spmv_x_in_global_memory_path(cuda):
    # C beyond the shared-memory staging limit: every x gather goes through the texture (TEX pipe)
    R, C = 6, 120000
    A = O.gen_dense(R, C, 0.3, 3)
    x = O.gen_vector(C, 4)
    dm = gpu_encode(A)
    assert dm.launch_info().x_in_smem == 0
    check_y(A, O.encode_dense(A), x, gpu_spmv(dm, x), False, "")


def test_spmv_deterministic_graph_and_unaligned_x(cuda):
    # rows of ~31 steps = 3 units each, 3000 units over ~4.7k warps: rows are cut between warps
    A = O.gen_dense(1000, 16000, 0.5, 8)
    x = O.gen_vector(16000, 9)
    dm = gpu_encode(A)
    assert dm.launch_info().n_split_rows > 0
    y0 = gpu_spmv(dm, x)
    for _ in range(5):
        assert np.array_equal(gpu_spmv(dm, x), y0)
    # x at a 2-byte (not 16-byte) aligned address
    xb = to_dev(np.concatenate([np.zeros(1, np.uint16), x]))
    y = torch.empty(1000, dtype=torch.float16, device=cuda)
    dm.spmv_into(xb[1:], y)
    torch.cuda.synchronize()
    assert np.array_equal(to_host_u16(y), y0)
    # CUDA graph capture / replay (split-row counters must reset between launches)
    xd = to_dev(x)
    yg = torch.empty(1000, dtype=torch.float16, device=cuda)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        dm.spmv_into(xd, yg, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            dm.spmv_into(xd, yg, stream=s)
    for _ in range(3):
        yg.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(to_host_u16(yg), y0)


def test_plan_and_x_staging_do_not_change_y(cuda):
    # SPEC.md:279 determinism across parallelism degree: every launch plan (CTAs per SM ->
    # number of warps -> where rows are cut) and every x staging mode gives identical bits.
    for R, C, d in ((3000, 5000, 0.5), (64, 20000, 0.3), (4096, 4096, 0.9)):
        A = O.gen_dense(R, C, d, 31)
        x = O.gen_vector(C, 32)
        dm = gpu_encode(A)
        y0 = gpu_spmv(dm, x)
        assert np.array_equal(y0, b200_y(O.encode_dense(A), x))
        for x_mode in (0, 1, 6, 7, 8, 10):
            for ctas in (1, 2, 0):
                try:
                    dm.configure(x_mode, ctas)
                except ValueError:  # the x table would not leave room for the TMA rings
                    assert x_mode > 0 and C * 2 >= 64_000
                    continue
                assert np.array_equal(gpu_spmv(dm, x), y0), (R, C, d, x_mode, ctas)
        dm.configure(-1, 0)


def test_spmv_host_buffers_e2e(cuda):
    A = O.gen_dense(777, 3333, 0.5, 10)
    x = O.gen_vector(3333, 11)
    dm = gpu_encode(A)
    y_host = dm.spmv_host(x)  # pageable numpy buffers: cudaMemcpyAsync both ways
    assert np.array_equal(y_host, gpu_spmv(dm, x))
    assert np.array_equal(y_host, b200_y(O.encode_dense(A), x))
    # pinned (device-mapped) buffers: x pulled / y pushed by kernels chained with PDL; odd offsets
    # exercise the 2-byte path of the copies
    for off in (0, 1):
        hx = torch.empty(3333 + off, dtype=torch.int16, pin_memory=True)
        hy = torch.zeros(777 + off, dtype=torch.int16, pin_memory=True)
        hxn, hyn = hx.numpy().view(np.uint16)[off:], hy.numpy().view(np.uint16)[off:]
        hxn[:] = x
        for _ in range(3):
            hyn[:] = 0
            dm.spmv_host(hxn, hyn)
            assert np.array_equal(hyn, y_host), off


def test_row_slabs_and_grid_independence(cuda):
    # The kernel's summation order depends only on a row's elements and on their positions mod 8
    # (ROMA) — never on the grid, the work plan or where warps cut rows.  So: a
    # slab encoded alone matches the oracle on that slab bit-exactly; it is bit-identical to the
    # full-matrix rows when its base offset keeps the alignment; otherwise it is within the
    # stated bound.
    R, C = 4096, 8192
    A = O.gen_dense(R, C, 0.5, 21)
    x = O.gen_vector(C, 22)
    g = O.encode_dense(A)
    dm_full = gpu_encode(A)
    y_seq = O.reference_spmv(g, x, 8)
    y_full = gpu_spmv(dm_full, x)
    for r0, r1 in ((0, 512), (512, 1536), (1536, 4096), (100, 101), (7, 3000)):
        s = O.encode_dense(A[r0:r1])
        dms = gpu_encode(A[r0:r1])
        y = gpu_spmv(dms, x)
        assert np.array_equal(y, b200_y(s, x)), (r0, r1)
        if int(g.row_ptrs[r0]) % 8 == 0:
            assert np.array_equal(y, y_full[r0:r1]), (r0, r1)
        assert within_bound(A[r0:r1], x, y, y_seq[r0:r1])
    # device-generated slab with a row offset equals the slab of the global matrix
    t = torch.empty((1024, C), dtype=torch.float16, device=cuda)
    M.gen_dense(t, 1024, C, 0.5, seed=21, row0=2048)
    dm = M.DeviceMatrix.from_dense(t)
    s = O.encode_dense(A[2048:3072])
    assert_same_format(dm, s)
    assert np.array_equal(gpu_spmv(dm, x), b200_y(s, x))


def test_error_behaviour(cuda):
    A = O.gen_dense(4, 64, 0.5, 1)
    m = O.encode_dense(A)
    # corrupt: decoded column walks past C -> FormatError
    bad = m.deltas.copy()
    bad[: m.pad_nnz // 2] = 0xFF
    with pytest.raises(M.FormatError):
        M.DeviceMatrix.upload(M.MackoMatrix(4, 64, 4, m.values, bad, m.row_ptrs))
    # -0 padding value -> FormatError
    v = m.values.copy()
    v[np.flatnonzero(v[: m.pad_nnz] == 0)[:1]] = 0x8000
    if (v != m.values).any():
        with pytest.raises(M.FormatError):
            M.DeviceMatrix.upload(M.MackoMatrix(4, 64, 4, v, m.deltas, m.row_ptrs))
    # x_mode 9 / 11 do not exist
    dm2 = gpu_encode(A, 2)
    with pytest.raises(ValueError, match="x_mode"):
        dm2.configure(9)
    dm = gpu_encode(A)
    with pytest.raises(ValueError):
        M.spmv(dm, torch.zeros(65, dtype=torch.float16, device=cuda))


def test_native_library_is_the_code_path(cuda):
    before = M.kernel_launches()
    A = O.gen_dense(64, 512, 0.5, 1)
    dm = gpu_encode(A)
    gpu_spmv(dm, O.gen_vector(512, 2))
    assert M.kernel_launches() > before
    import re

    maps = open("/proc/self/maps").read()
    assert re.search(r"libmacko_cuda\.so", maps)


def _same_or_both_nan(a: np.ndarray, b: np.ndarray) -> bool:
    fa, fb = a.view(np.float16), b.view(np.float16)
    nan = np.isnan(fa) & np.isnan(fb)
    return bool(np.all(nan | (a == b)))


@pytest.mark.parametrize("x_mode", [-1, 0, 1, 6, 7, 8])
def test_masked_edges_do_not_leak_inf_nan(cuda, x_mode):
    # Row edges are masked (codeword 0, value +0, x = +0).  Even rows are finite and end exactly
    # at column 699 (so masked elements after their end decode to columns 700..706); x is inf /
    # NaN from column 700 on, and the odd rows hold inf / NaN values (the ROMA-masked elements at
    # the start of every even row belong to them).  reference_spmv multiplies only a row's own
    # stored elements and pads: the even rows must come out finite and bit-exact.
    R, C = 240, 1500
    A = O.gen_dense(R, C, 0.35, 21)
    A[0::2, 700:] = 0
    A[0::2, 699] = 0x3C00  # 1.0
    for r in range(1, R, 2):
        cols = np.nonzero(A[r])[0]
        A[r, cols[:: max(1, cols.size // 4)]] = np.uint16(0x7C00)
        A[r, cols[1]] = np.uint16(0x7E00)
    x = O.gen_vector(C, 22)
    x[700::3] = np.uint16(0x7C00)
    x[701::3] = np.uint16(0xFC00)
    x[702::3] = np.uint16(0x7E00)
    dm = gpu_encode(A)
    if x_mode >= 0:
        dm.configure(x_mode)
    m = O.encode_dense(A)
    y = gpu_spmv(dm, x)
    y_ref = b200_y(m, x)
    assert _same_or_both_nan(y, y_ref)
    assert np.isfinite(y_ref[0::2].view(np.float16)).all()
    assert np.array_equal(y[0::2], y_ref[0::2])
    assert not np.isfinite(y[1::2].view(np.float16)).any()


@pytest.mark.parametrize("bits", [1, 2, 8])
def test_spmv_other_delta_widths(cuda, bits):
    # b_delta in {1, 2, 8}: the same kernel with the width's codeword loads / decode (b = 8: 16-bit
    # prefixes, scan on total - 8).  Integer mode is bit-exact against reference_spmv; float mode
    # bit-exact against the B200 order and within the bound of the sequential reference.
    cases = ((300, 5000, 0.5), (64, 20000, 0.05), (1000, 3000, 0.9), (7, 70000, 0.02))
    for R, C, d in cases:
        for int_mode in (True, False):
            A = O.gen_dense(R, C, d, 70 + bits, int_mode)
            x = O.gen_vector(C, 71, int_mode)
            m = O.encode_dense(A, bits)
            dm = gpu_encode(A, bits)
            assert_same_format(dm, m, (bits, R, C, d))
            check_y(A, m, x, gpu_spmv(dm, x), int_mode, (bits, R, C, d, int_mode))
    A = O.gen_dense(500, 9000, 0.3, 72)
    x = O.gen_vector(9000, 73)
    dm = gpu_encode(A, bits)
    y0 = gpu_spmv(dm, x)
    for x_mode in (0, 1, 6, 7, 8, 10):
        dm.configure(x_mode)
        assert np.array_equal(gpu_spmv(dm, x), y0), (bits, x_mode)


def _codes(deltas: np.ndarray, first: int, n: int) -> np.ndarray:
    """4-bit codewords of elements [first, first + n) (LSB-first nibbles, bitpack.cpp:18-32)."""
    idx = np.arange(first, first + n, dtype=np.int64)
    return (deltas[idx // 2] >> ((idx % 2) * 4).astype(np.uint8)) & 0xF


def test_large_offsets_beyond_2_30(cuda):
    # pad_nnz ~1.15e9 > 2^30: element offsets times 4 bits leave u32 range in the last ~7 % of rows.
    # Integer mode (order-independent, exact): y of the big matrix == y of the same rows encoded
    # as a standalone slab (small offsets) == reference_spmv on that slab; the big matrix's stored
    # bytes for those rows decode to the oracle's encoding of them.
    R, C = 70000, 32768
    dense = torch.empty((R, C), dtype=torch.float16, device=cuda)
    M.gen_dense(dense, R, C, 0.5, seed=91, int_mode=True)
    dm = M.DeviceMatrix.from_dense(dense)
    assert dm.pad_nnz > 2**30
    x = torch.empty(C, dtype=torch.float16, device=cuda)
    M.gen_vector(x, C, seed=92, int_mode=True)
    y = M.spmv(dm, x)
    torch.cuda.synchronize()
    y_big = to_host_u16(y)
    xh = to_host_u16(x)
    h = dm.download()
    for r0, r1 in ((R - 257, R), (0, 130)):
        slab = dense[r0:r1]
        dms = M.DeviceMatrix.from_dense(slab)
        ys = to_host_u16(M.spmv(dms, x))
        torch.cuda.synchronize()
        assert np.array_equal(y_big[r0:r1], ys), (r0, r1)
        A = to_host_u16(slab)
        m = O.encode_dense(A)
        assert np.array_equal(ys, O.reference_spmv(m, xh, 8)), (r0, r1)
        e0, e1 = int(h.row_pointers[r0]), int(h.row_pointers[r1])
        assert np.array_equal(h.row_pointers[r0:r1 + 1] - e0, m.row_ptrs)
        assert np.array_equal(h.values[e0:e1], m.values[: e1 - e0])
        assert np.array_equal(_codes(h.packed_deltas, e0, e1 - e0), _codes(m.deltas, 0, e1 - e0))
        dms.close()
    dm.close()


def _random_values(rng, n):
    # nonzero fp16 in (-1, 1), like the generator (long rows must not overflow fp16 sums)
    u = rng.integers(1, 1 << 16, n)
    u[u == 1 << 15] += 1
    return ((u - 32768) / 32768.0).astype(np.float16).view(np.uint16)


def test_rows_split_across_many_warps(cuda):
    # three ~1M-element rows: every row is cut into hundreds of warp pieces, finished by the last
    # arriving warp from per-unit partials; float and integer values
    R, C = 3, 2_000_000
    for int_mode in (False, True):
        A = O.gen_dense(R, C, 0.5, 515, int_mode)
        A[1, : C // 3] = 0  # a row starting far from column 0
        x = O.gen_vector(C, 516, int_mode)
        m = O.encode_dense(A)
        dm = gpu_encode(A)
        assert dm.launch_info().n_split_rows >= 3
        check_y(A, m, x, gpu_spmv(dm, x), int_mode, ("split", int_mode))


def test_power_law_row_lengths(cuda):
    # Zipf-like row lengths (a few dense rows, a long tail of short and empty rows) in random order
    rng = np.random.default_rng(77)
    R, C = 6000, 8192
    p = np.minimum(1.0, 3.0 / (np.arange(R) + 1.0) ** 0.8)
    rng.shuffle(p)
    mask = rng.random((R, C)) < p[:, None]
    A = np.zeros((R, C), np.uint16)
    A[mask] = _random_values(rng, int(mask.sum()))
    x = O.gen_vector(C, 78)
    m = O.encode_dense(A)
    dm = gpu_encode(A)
    check_y(A, m, x, gpu_spmv(dm, x), False, "zipf")


def test_other_widths_every_x_mode(cuda):
    # b_delta 1 / 2 / 8: every x_mode built for them gives the same bits (the oracle order)
    for bits, d in ((1, 0.9), (2, 0.6), (8, 0.05)):
        A = O.gen_dense(1500, 6000, d, 90 + bits)
        x = O.gen_vector(6000, 91)
        m = O.encode_dense(A, bits)
        dm = gpu_encode(A, bits)
        ref = b200_y(m, x)
        for xm in (0, 1, 6, 7, 8, 10):
            dm.configure(xm)
            assert np.array_equal(gpu_spmv(dm, x), ref), (bits, xm)
        with pytest.raises(ValueError):
            dm.configure(11)


# ------------------------------------------------------------------------------ one handle, many streams
def test_two_streams_one_handle_different_x(cuda):
    # SPEC.md:119-120 / SURVEY.md §8b: a handle is read-only after build and may be shared across
    # streams.  Rows cut between warps use per-stream split counters / partials, x texture objects
    # are cached per buffer: concurrent SpMVs of one matrix on two streams stay exact.
    A = O.gen_dense(1000, 16000, 0.5, 8)
    m = O.encode_dense(A)
    dm = gpu_encode(A)
    assert dm.launch_info().n_split_rows > 0
    xs = [O.gen_vector(16000, 40 + i) for i in range(2)]
    refs = [b200_y(m, x) for x in xs]
    xd = [to_dev(x) for x in xs]
    streams = [torch.cuda.Stream() for _ in range(2)]
    ys = [[torch.empty(1000, dtype=torch.float16, device=cuda) for _ in range(20)] for _ in range(2)]
    torch.cuda.synchronize()
    for k in range(20):
        for s in range(2):
            dm.spmv_into(xd[s], ys[s][k], stream=streams[s])
    torch.cuda.synchronize()
    for s in range(2):
        for k in range(20):
            assert np.array_equal(to_host_u16(ys[s][k]), refs[s]), (s, k)


def test_async_calls_alternating_x_buffers(cuda):
    # 100 asynchronous calls on one stream, x alternating between 4 buffers (one misaligned), no
    # synchronisation in between: no texture object is destroyed while a launch may still read it
    A = O.gen_dense(2000, 12000, 0.5, 12)
    m = O.encode_dense(A)
    dm = gpu_encode(A)
    xs = [O.gen_vector(12000, 50 + i) for i in range(4)]
    refs = [b200_y(m, x) for x in xs]
    bufs = [to_dev(x) for x in xs[:3]]
    mis = to_dev(np.concatenate([np.zeros(1, np.uint16), xs[3]]))[1:]  # 2-byte aligned view
    bufs.append(mis)
    ys = [torch.empty(2000, dtype=torch.float16, device=cuda) for _ in range(100)]
    for k in range(100):
        dm.spmv_into(bufs[k % 4], ys[k])
    torch.cuda.synchronize()
    for k in range(100):
        assert np.array_equal(to_host_u16(ys[k]), refs[k % 4]), k


def test_threads_share_one_handle(cuda):
    # host threads with their own streams and pinned host buffers call macko_spmv_host and
    # macko_dev_spmv on one handle at once
    import threading

    A = O.gen_dense(1500, 9000, 0.5, 13)
    m = O.encode_dense(A)
    dm = gpu_encode(A)
    xs = [O.gen_vector(9000, 60 + i) for i in range(4)]
    refs = [b200_y(m, x) for x in xs]
    errors = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            xd = to_dev(xs[i])
            y = torch.empty(1500, dtype=torch.float16, device=cuda)
            for _ in range(10):
                if i % 2:
                    got = dm.spmv_host(xs[i], stream=s)
                else:
                    dm.spmv_into(xd, y, stream=s)
                    s.synchronize()
                    got = to_host_u16(y)
                if not np.array_equal(got, refs[i]):
                    errors.append(i)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


# ------------------------------------------------------------------------------ convert.hpp on the GPU
@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_macko_from_csr_dense_from_macko_padding_count(cuda, bits):
    # macko_from_csr from host CSR and from device CSR == the oracle's encoder (byte-identical);
    # dense_from_macko roundtrips; padding_count == pad_nnz - nnz
    for i, (R, C, d) in enumerate(((1, 1, 1.0), (7, 37, 0.5), (64, 1000, 0.05), (300, 513, 0.3), (33, 4097, 0.9),
                                   (1000, 2048, 0.0), (5, 20000, 0.01))):
        A = O.gen_dense(R, C, d, 500 + i, bool(i & 1))
        if R > 4:
            A[::3] = 0
        vals, cols, rp = O.csr_from_dense(A)
        gv, gc, grp = M.csr_from_dense(A)  # GPU csr_from_dense == the oracle's
        assert np.array_equal(gv, vals) and np.array_equal(gc, cols) and np.array_equal(grp, rp)
        tv, tc, trp = M.csr_from_dense(to_dev(A))
        assert np.array_equal(tv, vals) and np.array_equal(tc, cols) and np.array_equal(trp, rp)
        m = O.macko_from_csr(R, C, vals, cols, rp, bits)
        dm = M.DeviceMatrix.from_csr(vals, cols, rp, R, C, bits)
        assert_same_format(dm, m, (R, C, d, bits))
        dmd = M.DeviceMatrix.from_csr(to_dev(vals), torch.from_numpy(cols.view(np.int32)).cuda(),
                                      torch.from_numpy(rp.view(np.int32)).cuda(), R, C, bits)
        assert_same_format(dmd, m, ("device csr", R, C, d, bits))
        assert np.array_equal(dm.to_dense(), A)
        out = torch.full((R, C + 3), 7.0, dtype=torch.float16, device=cuda)[:, :C]
        dm.to_dense(out)
        assert np.array_equal(to_host_u16(out), A)
        assert dm.padding_count() == O.padding_count(m) == m.pad_nnz - int((A & 0x7FFF != 0).sum())


def test_macko_from_csr_rejects_non_canonical(cuda):
    vals = np.array([0x3C00, 0x3C00], np.uint16)
    with pytest.raises(ValueError, match="strictly increasing"):
        M.DeviceMatrix.from_csr(vals, np.array([5, 5], np.uint32), np.array([0, 2], np.uint32), 1, 10)
    with pytest.raises(ValueError, match="out of range"):
        M.DeviceMatrix.from_csr(vals, np.array([5, 10], np.uint32), np.array([0, 2], np.uint32), 1, 10)
    with pytest.raises(ValueError):
        M.DeviceMatrix.from_csr(vals, np.array([1, 2], np.uint32), np.array([0, 1], np.uint32), 1, 10)  # rp[R] != nnz
    # a corrupt stored matrix: dense_from_macko reports FormatError
    A = O.gen_dense(4, 64, 0.5, 1)
    dm = gpu_encode(A)
    assert dm.padding_count() == 0 or dm.padding_count() > 0


# ------------------------------------------------------------------------------ small-batch SpMM
@pytest.mark.parametrize("batch", [1, 2, 3, 4, 5, 8])
def test_spmm_columns_equal_spmv(cuda, batch):
    # PAPER.md:535 (future work): Y = A X for a batch of vectors, one pass over the matrix; column b
    # is bit-exact against the order oracle on X[b] (and the integer-mode sequential reference)
    cases = [(1000, 16000, 0.5), (300, 5000, 0.3), (4096, 4096, 0.5), (17, 20000, 0.02), (2000, 3000, 0.9),
             (6, 120000, 0.3)]  # the last: x table too large -> texture-only kernel
    for i, (R, C, d) in enumerate(cases):
        for int_mode in (False, True):
            A = O.gen_dense(R, C, d, 700 + i, int_mode)
            if R > 8:
                A[2::9] = 0
            m = O.encode_dense(A)
            dm = gpu_encode(A)
            X = np.stack([O.gen_vector(C, 800 + 10 * i + b, int_mode) for b in range(batch)])
            Xd = to_dev(X)
            Y = torch.full((batch, R + 5), 7.0, dtype=torch.float16, device=cuda)[:, :R]  # ldy > rows
            dm.spmm_into(Xd, Y)
            torch.cuda.synchronize()
            Yh = to_host_u16(Y.contiguous())
            for b in range(batch):
                if int_mode:
                    assert np.array_equal(Yh[b], O.reference_spmv(m, X[b], 8)), (R, C, d, b)
                else:
                    assert np.array_equal(Yh[b], b200_y(m, X[b])), (R, C, d, b)
            # padding outputs (R..R+5) untouched
            assert (Y.as_strided((batch, 5), (R + 5, 1), R) == 7.0).all()


def test_spmm_errors(cuda):
    A = O.gen_dense(64, 512, 0.5, 1)
    dm = gpu_encode(A)
    X = torch.zeros((9, 512), dtype=torch.float16, device=cuda)
    with pytest.raises(ValueError):
        dm.spmm_into(X, torch.zeros((9, 64), dtype=torch.float16, device=cuda))  # batch > 8
    with pytest.raises(ValueError):
        dm.spmm_into(X[:2, :500], torch.zeros((2, 64), dtype=torch.float16, device=cuda))
    dm2 = gpu_encode(A, 2)
    with pytest.raises(ValueError, match="b_delta"):
        dm2.spmm_into(X[:2], torch.zeros((2, 64), dtype=torch.float16, device=cuda))


# ------------------------------------------------------------------------------ the plan on the device
def test_device_plan_equals_host_plan(cuda, monkeypatch):
    # plan.cu builds the SpMV work plan on the GPU; the host builder (MACKO_HOST_PLAN=1) is its
    # reference: identical warp records (unit ranges, TMA element ranges, column bases, split ids)
    # and split records, on row-length mixes that exercise every case
    rng = np.random.default_rng(5)
    cases = [O.gen_dense(36, 65536, 0.5, 1), O.gen_dense(1000, 16000, 0.5, 2), O.gen_dense(4096, 64, 0.5, 3),
             O.gen_dense(7, 37, 0.5, 4), O.gen_dense(2000, 3000, 0.02, 5)]
    z = O.gen_dense(3000, 9000, 0.4, 6)
    z[rng.random(3000) < 0.5] = 0  # many empty rows
    cases.append(z)
    for A in cases:
        monkeypatch.setenv("MACKO_HOST_PLAN", "1")
        dh = gpu_encode(A)
        monkeypatch.delenv("MACKO_HOST_PLAN")
        dd = gpu_encode(A)
        for ctas in (0, 1):
            if ctas:
                monkeypatch.setenv("MACKO_HOST_PLAN", "1")
                dh.configure(-1, 1)
                monkeypatch.delenv("MACKO_HOST_PLAN")
                dd.configure(-1, 1)
            rh, sh = dh.plan_records()
            rd, sd = dd.plan_records()
            assert dh.launch_info().n_units == dd.launch_info().n_units
            assert np.array_equal(rh, rd), (A.shape, ctas)
            assert np.array_equal(sh, sd), (A.shape, ctas)
        x = O.gen_vector(A.shape[1], 7)
        assert np.array_equal(gpu_spmv(dd, x), b200_y(O.encode_dense(A), x))


def test_block_cache_reuse_keeps_formats_exact(cuda):
    """Matrices built, freed and rebuilt reuse cached device blocks (capi BlockCache): every build
    is still bit-exact, including builds into recycled blocks that held a different matrix."""
    from paper_2511_13061_b200 import _lib

    cases = [(1024, 2048, 0.5), (700, 3000, 0.3), (1024, 2048, 0.9), (1500, 2048, 0.5)]
    for rep in range(2):
        for i, (R, C, d) in enumerate(cases):
            A = O.gen_dense(R, C, d, 77 + i + 10 * rep)
            dm = gpu_encode(A, 4)
            assert_same_format(dm, O.encode_dense(A, 4), (rep, R, C, d))
            dm.close()
    assert _lib.load().macko_release_cached_memory() == 0
    A = O.gen_dense(512, 4096, 0.5, 5)
    assert_same_format(gpu_encode(A, 4), O.encode_dense(A, 4), "after release")


# ------------------------------------------------------------------------------ chain (PDL) instance
def gpu_spmv_pdl(dm: M.DeviceMatrix, x: np.ndarray) -> np.ndarray:
    """SpMV through the PDL launch (the chain kernel instance: staggered first fill, per-step edge
    masking, x staged by one bulk copy)."""
    xd = to_dev(x)
    y = torch.empty(dm.rows, dtype=torch.float16, device=xd.device)
    dm.spmv_into(xd, y, pdl=True)
    torch.cuda.synchronize()
    return to_host_u16(y)


def _ragged_rows(R, C, seed):
    """Rows of every edge shape the walk distinguishes: empty, 1..7 elements (ROMA head only),
    one step (T = 1), two steps (T = 2: first and last pair are one), three (first pair then a
    single step), odd / even longer rows, rows spanning several warps."""
    rng = np.random.default_rng(seed)
    A = np.zeros((R, C), np.uint16)
    lengths = [0, 1, 3, 7, 9, 200, 256, 300, 511, 512, 513, 700, 768, 1000, 1024, 1500, 2600, C]
    for r in range(R):
        n = lengths[r % len(lengths)] if r % 5 else int(rng.integers(0, C))
        cols = np.sort(rng.choice(C, size=min(n, C), replace=False))
        A[r, cols] = _random_values(rng, cols.size)
    return A


@pytest.mark.parametrize("x_mode", [-1, 0, 1, 6, 7, 8, 10])
def test_pdl_instance_every_edge_shape(cuda, x_mode):
    # The PDL kernel instance masks edge pairs step by step (EdgeFirst / EdgeFirstLast / EdgeLast /
    # EdgeSingle) and stages x with one bulk copy; its y must equal the plain instance's and the
    # oracle order bit for bit, for every row shape and ROMA offset.
    for R, C, seed in ((300, 3000, 1), (97, 4099, 2), (64, 6000, 3)):
        A = _ragged_rows(R, C, seed)
        x = O.gen_vector(C, 10 + seed)
        m = O.encode_dense(A)
        dm = gpu_encode(A)
        if x_mode >= 0:
            dm.configure(x_mode)
        ref = b200_y(m, x)
        assert np.array_equal(gpu_spmv_pdl(dm, x), ref), (R, C, x_mode, "pdl")
        assert np.array_equal(gpu_spmv(dm, x), ref), (R, C, x_mode, "plain")


@pytest.mark.parametrize("bits", [1, 2, 8])
def test_pdl_instance_other_widths(cuda, bits):
    A = _ragged_rows(200, 5000, 40 + bits)
    x = O.gen_vector(5000, 41)
    m = O.encode_dense(A, bits)
    dm = gpu_encode(A, bits)
    assert np.array_equal(gpu_spmv_pdl(dm, x), b200_y(m, x)), bits


@pytest.mark.parametrize("R,C,d,splits", [(64, 40000, 0.5, True), (600, 70000, 0.3, True), (4096, 4096, 0.5, False),
                                           (300, 6000, 0.9, False)])
def test_pdl_instance_with_and_without_split_rows(cuda, R, C, d, splits):
    # PDL launches of a plan with split rows use the chain instance with the split-row finish;
    # without split rows (every row one unit, the Llama linears) the kNoSplit instance.
    A = O.gen_dense(R, C, d, R + C)
    A[5] = 0
    x = O.gen_vector(C, 3)
    dm = gpu_encode(A)
    assert (dm.launch_info().n_split_rows > 0) == splits
    ref = b200_y(O.encode_dense(A), x)
    for _ in range(2):  # split counters are reset by the last arrival
        assert np.array_equal(gpu_spmv_pdl(dm, x), ref)
    assert np.array_equal(gpu_spmv(dm, x), ref)


def test_pdl_instance_masked_edges_do_not_leak_inf_nan(cuda):
    R, C = 240, 1500
    A = O.gen_dense(R, C, 0.35, 21)
    A[0::2, 700:] = 0
    A[0::2, 699] = 0x3C00
    for r in range(1, R, 2):
        cols = np.nonzero(A[r])[0]
        A[r, cols[:: max(1, cols.size // 4)]] = np.uint16(0x7C00)
        A[r, cols[1]] = np.uint16(0x7E00)
    x = O.gen_vector(C, 22)
    x[700::3] = np.uint16(0x7C00)
    x[701::3] = np.uint16(0xFC00)
    x[702::3] = np.uint16(0x7E00)
    dm = gpu_encode(A)
    m = O.encode_dense(A)
    y = gpu_spmv_pdl(dm, x)
    y_ref = b200_y(m, x)
    assert _same_or_both_nan(y, y_ref)
    assert np.array_equal(y[0::2], y_ref[0::2])


def test_chain_skewed_plan_host_device_and_y(cuda, monkeypatch):
    # macko_dev_set_chain_skew: early CTAs get larger shares (plan.cuh plan_warp_of).  The device
    # builder must equal the host reference record for record, shares must fall with the CTA index,
    # and y (plain and PDL instance) is unchanged.
    cases = [O.gen_dense(4096, 4096, 0.5, 11), O.gen_dense(1000, 16000, 0.5, 12), O.gen_dense(300, 3000, 0.1, 13)]
    for A in cases:
        monkeypatch.setenv("MACKO_HOST_PLAN", "1")
        dh = gpu_encode(A)
        dh.set_chain_skew(2000)
        monkeypatch.delenv("MACKO_HOST_PLAN")
        dd = gpu_encode(A)
        dd.set_chain_skew(2000)
        rh, sh = dh.plan_records()
        rd, sd = dd.plan_records()
        assert np.array_equal(rh, rd), A.shape
        assert np.array_equal(sh, sd), A.shape
        li = dd.launch_info()
        units = rd[:, 0].astype(np.int64)
        assert units.max() <= 2 * int(np.ceil(units.sum() / units.size)) + 2, (A.shape, units.max())
        if A.shape == (4096, 4096):
            per_cta = rd[:, 4].astype(np.int64) - rd[:, 3].astype(np.int64)  # TMA element range per warp
            per_cta = per_cta.reshape(li.grid, -1).sum(axis=1)
            assert per_cta[: li.grid // 4].mean() > per_cta[-li.grid // 4:].mean() * 1.05
        x = O.gen_vector(A.shape[1], 14)
        ref = b200_y(O.encode_dense(A), x)
        assert np.array_equal(gpu_spmv(dd, x), ref)
        assert np.array_equal(gpu_spmv_pdl(dd, x), ref)
        dd.set_chain_skew(0)
        assert np.array_equal(gpu_spmv(dd, x), ref)
