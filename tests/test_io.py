"""MCKO container and Matrix Market reader (reference io.cpp is absent).

Host paths (no GPU needed): write_macko / read_macko through libmacko_cuda's C-ABI, checked
byte for byte against the oracle's restatement of the file layout (oracle.mcko_bytes) on every
golden matrix (all b_delta), plus SPEC's examples and error cases.  GPU paths: device matrix ->
file -> device matrix, streamed through pinned buffers, and an SpMV on the loaded matrix.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_13061_b200 import macko as M
from tests.helpers import b200_y, to_dev, to_host_u16


def _host(c) -> M.MackoMatrix:
    R, C = c["dense"].shape
    return M.MackoMatrix(R, C, int(c["bits"]), c["values"], c["deltas"], c["row_ptrs"])


def _oracle(c) -> O.Macko:
    R, C = c["dense"].shape
    return O.Macko(R, C, int(c["bits"]), c["values"], c["deltas"], c["row_ptrs"])


def test_golden_roundtrip_bytes(golden, tmp_path):
    for name, c in golden.items():
        p = tmp_path / f"{name}.mcko"
        M.write_mcko(_host(c), p)
        data = p.read_bytes()
        assert data == O.mcko_bytes(_oracle(c)), name
        back = M.read_mcko_host(p)
        assert np.array_equal(back.row_pointers, c["row_ptrs"]), name
        assert np.array_equal(back.values[: c["values"].size], c["values"]), name
        assert np.array_equal(back.packed_deltas[: c["deltas"].size], c["deltas"]), name
        q = tmp_path / f"{name}.again.mcko"
        M.write_mcko(back, q)
        assert q.read_bytes() == data, name  # identical bytes on rewrite


def test_fig3_and_header(golden, tmp_path):
    c = golden["fig3_b2"]
    p = tmp_path / "fig3.mcko"
    M.write_mcko(_host(c), p)
    data = p.read_bytes()
    assert data[:4] == b"MCKO" and data[4:6] == b"\x01\x00" and data[6] == 16 and data[7] == 2
    info = M.mcko_info(p)
    assert (info.rows, info.cols, info.pad_nnz, info.b_delta) == (1, c["dense"].shape[1], 5, 2)
    assert len(data) == 32 + 4 * 2 + info.delta_bytes + info.values_bytes


def test_empty_1x1_roundtrip(tmp_path):
    m = O.encode_dense(np.zeros((1, 1), np.uint16))
    p = tmp_path / "z.mcko"
    M.write_mcko(M.MackoMatrix(1, 1, 4, m.values, m.deltas, m.row_ptrs), p)
    back = M.read_mcko_host(p)
    assert back.pad_nnz() == 0 and back.rows == 1 and back.cols == 1
    assert p.read_bytes() == O.mcko_bytes(m)


def _corrupt(tmp_path, golden, fn):
    c = golden["r17x100_d30_b4_f16"]
    p = tmp_path / "c.mcko"
    M.write_mcko(_host(c), p)
    b = bytearray(p.read_bytes())
    fn(b)
    p.write_bytes(bytes(b))
    return p


def test_errors(golden, tmp_path):
    with pytest.raises(M.IoError):  # corrupted magic -> distinct error
        M.read_mcko_host(_corrupt(tmp_path, golden, lambda b: b.__setitem__(0, ord("X"))))
    with pytest.raises(M.IoError):  # version
        M.read_mcko_host(_corrupt(tmp_path, golden, lambda b: b.__setitem__(4, 2)))
    with pytest.raises(M.IoError):  # truncated values section
        M.read_mcko_host(_corrupt(tmp_path, golden, lambda b: b.__delitem__(slice(len(b) - 20, len(b)))))
    with pytest.raises(M.FormatError):  # row_pointers[R] != pad_nnz
        M.read_mcko_host(_corrupt(tmp_path, golden, lambda b: b.__setitem__(24, b[24] ^ 1)))
    with pytest.raises(M.FormatError):  # b_delta outside {1,2,4,8}
        M.read_mcko_host(_corrupt(tmp_path, golden, lambda b: b.__setitem__(7, 3)))
    with pytest.raises(M.FormatError):  # decoded column past C: every codeword all-ones

        def all_ones(b):
            R = 17
            d0 = 32 + 4 * (R + 1)
            pad = int.from_bytes(b[24:32], "little")
            for i in range(d0, d0 + (pad * 4 + 7) // 8):
                b[i] = 0xFF

        M.read_mcko_host(_corrupt(tmp_path, golden, all_ones))
    with pytest.raises(M.IoError):
        M.read_mcko_host(tmp_path / "missing.mcko")


MM3 = """%%MatrixMarket matrix coordinate real general
% three entries
3 4 3
1 1 1.5
2 4 -2
3 2 0.1
"""


def test_matrix_market(tmp_path):
    p = tmp_path / "a.mtx"
    p.write_text(MM3)
    A = M.read_matrix_market(p)
    assert A.shape == (3, 4)
    F = A.view(np.float16).astype(np.float32)
    assert F[0, 0] == 1.5 and F[1, 3] == -2 and F[2, 1] == np.float32(np.float16(0.1))  # 1-based -> 0-based
    assert (A != 0).sum() == 3
    p.write_text(MM3.replace("3 2 0.1", "2 4 1"))
    with pytest.raises(M.FormatError):  # duplicate coordinate
        M.read_matrix_market(p)
    p.write_text(MM3.replace("3 2 0.1", "4 2 1"))
    with pytest.raises(M.FormatError):  # index out of range
        M.read_matrix_market(p)
    p.write_text(MM3.replace("coordinate", "array"))
    with pytest.raises(M.IoError):  # unsupported kind
        M.read_matrix_market(p)
    # through the encoder: the file's matrix encodes like the oracle's
    p.write_text(MM3)
    m = O.encode_dense(M.read_matrix_market(p), 4)
    assert m.pad_nnz == 3


@pytest.mark.gpu
def test_device_write_read_spmv(cuda, tmp_path):
    import torch

    for R, C, d in ((777, 3333, 0.5), (8192, 12288, 0.5)):  # the second spans several 32-MiB blocks
        A = O.gen_dense(R, C, d, 41)
        dm = M.DeviceMatrix.from_dense(to_dev(A))
        p = tmp_path / "dev.mcko"
        M.write_mcko(dm, p)
        m = O.encode_dense(A)
        assert p.read_bytes() == O.mcko_bytes(m)
        dm2 = M.read_mcko(p)
        h = dm2.download()
        assert np.array_equal(h.values, m.values) and np.array_equal(h.packed_deltas, m.deltas)
        assert np.array_equal(h.row_pointers, m.row_ptrs)
        x = O.gen_vector(C, 42)
        y = M.spmv(dm2, to_dev(x))
        torch.cuda.synchronize()
        assert np.array_equal(to_host_u16(y), b200_y(m, x))
        dm.close()
        dm2.close()
