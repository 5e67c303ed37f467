"""Parity at every configuration bench.py times, at full size (BASELINE.json configs[1], [4]).

The matrices are generated on the GPU (the counter-hash generator, bit-identical to the oracle's:
test_gpu_parity.py::test_generator_bit_identical) and compressed by the GPU compressor.  Then:

  * format: the downloaded values / packed deltas / row pointers equal the CPU oracle's encoding
    of the same dense rows, slab by slab (rows are independent: a slab's standalone
    encoding is the global encoding sliced), so host memory stays bounded;
  * y: bit-exact against the oracle's emulation of the kernel order (mo_b200_order_spmv) run on
    the verified arrays, in float mode; bit-exact against the sequential reference_spmv in integer
    mode; within the stated bound of the sequential reference on a sample of rows.

The oracle runs threaded (row partitions, byte-identical to the single-threaded restatement).
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2511_13061_b200 import macko as M
from tests.helpers import UNIT_STEPS, to_host_u16, within_bound

pytestmark = pytest.mark.gpu
THREADS = max(1, min(64, len(os.sched_getaffinity(0))))
SEED_A, SEED_X = 1234, 4321  # bench.py's seeds


def _codes(deltas: np.ndarray, first: int, n: int, bits: int) -> np.ndarray:
    """Codewords of elements [first, first + n) (LSB-first, bitpack.cpp:18-32)."""
    per = 8 // bits
    idx = np.arange(first, first + n, dtype=np.int64)
    shift = ((idx % per) * bits).astype(np.uint8)
    return (deltas[idx // per] >> shift) & ((1 << bits) - 1)


def verify_format(h: M.MackoMatrix, dense: torch.Tensor, bits: int = 4, slab: int = 8192) -> None:
    """h (downloaded GPU arrays of the whole matrix) == the oracle's encoding of `dense`, slab by slab."""
    R = dense.shape[0]
    assert h.row_pointers[0] == 0
    for r0 in range(0, R, slab):
        r1 = min(R, r0 + slab)
        m = O.encode_dense(to_host_u16(dense[r0:r1]), bits, THREADS)
        e0, e1 = int(h.row_pointers[r0]), int(h.row_pointers[r1])
        assert np.array_equal(h.row_pointers[r0:r1 + 1] - np.uint32(e0), m.row_ptrs), (r0, r1)
        assert np.array_equal(h.values[e0:e1], m.values[: e1 - e0]), (r0, r1)
        if (e0 * bits) % 8 == 0 and (e1 * bits) % 8 == 0:
            assert np.array_equal(h.packed_deltas[e0 * bits // 8:e1 * bits // 8], m.deltas[: (e1 - e0) * bits // 8])
        else:
            assert np.array_equal(_codes(h.packed_deltas, e0, e1 - e0, bits), _codes(m.deltas, 0, e1 - e0, bits))
    pad_nnz = int(h.row_pointers[-1])
    # tails: values / deltas zero past pad_nnz up to the 16-byte multiple (matrix.hpp:57-59)
    assert len(h.values) == M.values_bytes(pad_nnz) // 2 and not h.values[pad_nnz:].any()
    last = (pad_nnz * bits + 7) // 8
    assert len(h.packed_deltas) == M.delta_bytes(pad_nnz, bits) and not h.packed_deltas[last:].any()


def as_oracle(h: M.MackoMatrix) -> O.Macko:
    return O.Macko(h.rows, h.cols, h.b_delta, h.values, h.packed_deltas, h.row_pointers)


def build(R, C, d, int_mode=False, row0=0, bits=4):
    dense = torch.empty((R, C), dtype=torch.float16, device="cuda")
    M.gen_dense(dense, R, C, d, seed=SEED_A, int_mode=int_mode, row0=row0)
    dm = M.DeviceMatrix.from_dense(dense, b_delta=bits)
    x = torch.empty(C, dtype=torch.float16, device="cuda")
    M.gen_vector(x, C, seed=SEED_X, int_mode=int_mode)
    torch.cuda.synchronize()
    return dense, dm, x


def check_y(dm, dense, x, int_mode, sample_rows=1024):
    y = to_host_u16(M.spmv(dm, x))
    # the PDL (decode-chain) kernel instance: staggered fills, per-step edges, bulk-copied x
    y_pdl = torch.empty(dm.rows, dtype=torch.float16, device=x.device)
    dm.spmv_into(x, y_pdl, pdl=True)
    torch.cuda.synchronize()
    assert np.array_equal(to_host_u16(y_pdl), y)
    h = dm.download()
    m = as_oracle(h)
    xh = to_host_u16(x)
    if int_mode:
        assert np.array_equal(y, O.reference_spmv(m, xh, THREADS))
    else:
        y_ord = O.b200_order_spmv(m, xh, UNIT_STEPS, THREADS)
        assert np.array_equal(y, y_ord)
        # the bound against the sequential reference on a sample of rows
        rows = np.unique(np.linspace(0, dm.rows - 1, sample_rows).astype(np.int64))
        A = to_host_u16(dense[torch.from_numpy(rows).to(dense.device)])
        ms = O.encode_dense(A, dm.b_delta, THREADS)
        assert within_bound(A, xh, y[rows], O.reference_spmv(ms, xh, THREADS))
    return h, y


@pytest.mark.timeout(900)
@pytest.mark.parametrize("density", [0.7, 0.5, 0.3, 0.1])
def test_headline_36864x12288_full(cuda, density):
    """configs[1]: the sparsity sweep 30/50/70/90 % of the bench, whole matrix."""
    dense, dm, x = build(36864, 12288, density)
    h, _ = check_y(dm, dense, x, False)
    verify_format(h, dense)
    dm.close()


@pytest.mark.timeout(900)
def test_headline_36864x12288_int_mode(cuda):
    dense, dm, x = build(36864, 12288, 0.5, int_mode=True)
    h, _ = check_y(dm, dense, x, True)
    verify_format(h, dense)
    dm.close()


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("density", [0.5, 0.1])
def test_config5_131072x32768_whole_and_slabs(cuda, density):
    """configs[4]: 131072x32768 @50 / 90 % — the whole matrix on one GPU, and the row slabs the
    N = 2 / 4 / 8 ranks own (first, middle and last slab of each N): a slab built on its own from
    the generator (row0 offset) is the global encoding sliced, and its y is the kernel order on
    its own encoding."""
    R, C = 131072, 32768
    dense, dm, x = build(R, C, density)
    h, y_full = check_y(dm, dense, x, False)
    verify_format(h, dense, slab=16384)
    xh = to_host_u16(x)
    del dense
    dm.close()
    torch.cuda.empty_cache()
    for n in (2, 4, 8):
        for g in sorted({0, n // 2, n - 1}):
            r0, r1 = M.shard_rows(R, n, g)
            ds, dms, _ = build(r1 - r0, C, density, row0=r0)
            hs = dms.download()
            e0, e1 = int(h.row_pointers[r0]), int(h.row_pointers[r1])
            assert np.array_equal(hs.row_pointers, h.row_pointers[r0:r1 + 1] - np.uint32(e0)), (n, g)
            assert np.array_equal(hs.values[: e1 - e0], h.values[e0:e1]), (n, g)
            assert np.array_equal(_codes(hs.packed_deltas, 0, e1 - e0, 4), _codes(h.packed_deltas, e0, e1 - e0, 4))
            ys = to_host_u16(M.spmv(dms, x))
            torch.cuda.synchronize()
            assert np.array_equal(ys, O.b200_order_spmv(as_oracle(hs), xh, UNIT_STEPS, THREADS)), (n, g)
            if e0 % 8 == 0:  # same ROMA alignment as in the whole matrix: bit-identical rows
                assert np.array_equal(ys, y_full[r0:r1]), (n, g)
            del ds
            dms.close()
            torch.cuda.empty_cache()
