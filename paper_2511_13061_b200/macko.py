"""Host-side mirror of the reference MACKO interface over the B200 C-ABI.

Reference operation (file:line)                     -> here (runs on the GPU through libmacko_cuda)
  csr_from_dense + macko_from_csr (convert.hpp:8-16) -> macko_from_dense(dense)        [GPU compressor]
  csr_from_dense (convert.hpp:8-10)                  -> csr_from_dense(dense)          [GPU]
  macko_from_csr (convert.hpp:12-16)                 -> macko_from_csr(values, cols, row_ptrs, ...) [GPU]
  dense_from_macko (convert.hpp:18-20)               -> DeviceMatrix.to_dense()        [GPU decode]
  padding_count (convert.hpp:22-23)                  -> DeviceMatrix.padding_count()   [GPU]
  MackoMatrix (matrix.hpp:57-81)                     -> MackoMatrix (host arrays, same bytes)
  host MackoMatrix as SpMV operand                   -> DeviceMatrix.upload(MackoMatrix)
  reference_spmv / warp_spmv       -> spmv(dm, x)                    [sm_100a kernel]
  validate_macko (convert.hpp:25-27)                 -> DeviceMatrix.validate()
  macko_values_bytes / macko_delta_bytes (matrix.hpp:77-81) -> values_bytes / delta_bytes
  spmv_traffic                     -> DeviceMatrix.traffic_bytes
  write_macko / read_macko          -> write_mcko / read_mcko_host / read_mcko (-> device)
  read_matrix_market                -> read_matrix_market

Arguments follow the reference's meaning (fp16 payloads as raw uint16 bits, b_delta in
{1,2,4,8}, row pointers as u32 element offsets) and its error behaviour (ValueError for
std::invalid_argument, FormatError / IoError / InfeasibleError for the reference exceptions).
Device tensors may be torch CUDA tensors; streams default to torch's current stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import CudaError, FormatError, InfeasibleError, IoError, check  # noqa: F401


def values_bytes(pad_nnz: int) -> int:
    """macko_values_bytes (matrix.hpp:77)."""
    return (pad_nnz * 2 + 15) // 16 * 16


def delta_bytes(pad_nnz: int, b_delta: int) -> int:
    """macko_delta_bytes (matrix.hpp:78-81)."""
    return ((pad_nnz * b_delta + 7) // 8 + 15) // 16 * 16


@dataclass
class MackoMatrix:
    """Host copy of the reference MackoMatrix (matrix.hpp:57-67): identical byte layout."""

    rows: int
    cols: int
    b_delta: int
    values: np.ndarray      # uint16 fp16 bits, >= pad_nnz (16-byte zero tail)
    packed_deltas: np.ndarray  # uint8, >= ceil(pad_nnz*b_delta/8) (16-byte zero tail)
    row_pointers: np.ndarray   # uint32, rows+1

    def pad_nnz(self) -> int:
        return int(self.row_pointers[-1]) if len(self.row_pointers) else 0


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        try:
            import torch

            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:  # pragma: no cover - torch absent
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


def _ptr(t) -> int:
    """Device pointer of a torch tensor (or an int pointer)."""
    if isinstance(t, int):
        return t
    return t.data_ptr()


class DeviceMatrix:
    """A MACKO matrix resident in HBM (opaque macko_dev_matrix handle)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        info = _lib.DevInfo()
        check(_lib.load().macko_dev_get_info(self._h, C.byref(info)))
        self.info = info

    @property
    def handle(self) -> int:
        """The C-ABI handle (torch.ops.macko.spmv, foreign bindings); valid until close()."""
        if not getattr(self, "_h", None) or not self._h.value:
            raise ValueError("matrix is closed")
        return self._h.value

    # -- construction -----------------------------------------------------------------------
    @classmethod
    def upload(cls, m: MackoMatrix, device: int = 0, stream=None) -> "DeviceMatrix":
        vals = np.ascontiguousarray(m.values, np.uint16)
        dl = np.ascontiguousarray(m.packed_deltas, np.uint8)
        rp = np.ascontiguousarray(m.row_pointers, np.uint32)
        h = C.c_void_p()
        check(_lib.load().macko_dev_upload(device, m.rows, m.cols, m.b_delta, vals.ctypes.data, len(vals),
                                           dl.ctypes.data, len(dl), rp.ctypes.data, _stream_ptr(stream), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_dense(cls, dense, rows: int | None = None, cols: int | None = None, ld: int | None = None,
                   b_delta: int = 4, device: int | None = None, stream=None) -> "DeviceMatrix":
        """GPU compressor from a dense fp16 device tensor (torch, row-major) or device pointer."""
        if not isinstance(dense, int):
            rows, cols = dense.shape
            ld = dense.stride(0)
            if device is None:
                device = dense.device.index
        if device is None:
            device = 0
        h = C.c_void_p()
        check(_lib.load().macko_dev_from_dense(device, _ptr(dense), rows, cols, ld if ld is not None else cols, b_delta,
                                               _stream_ptr(stream), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_csr(cls, values, col_idx, row_ptrs, rows: int, cols: int, b_delta: int = 4, device: int | None = None,
                 stream=None) -> "DeviceMatrix":
        """macko_from_csr on the GPU from a canonical CSR: numpy host arrays (uint16 fp16 bits,
        uint32 columns, uint32 row pointers) or torch CUDA tensors (int16/float16, int32, int32)."""
        L = _lib.load()
        h = C.c_void_p()
        if isinstance(values, np.ndarray):
            v = np.ascontiguousarray(values, np.uint16)
            ci = np.ascontiguousarray(col_idx, np.uint32)
            rp = np.ascontiguousarray(row_ptrs, np.uint32)
            if rp.shape != (rows + 1,):
                raise ValueError("row_ptrs must have rows + 1 entries")
            nnz = int(v.size)
            if ci.size != nnz:
                raise ValueError("values and col_idx lengths differ")
            check(L.macko_dev_from_csr(0 if device is None else device, rows, cols, b_delta,
                                       v.ctypes.data if nnz else None, ci.ctypes.data if nnz else None,
                                       rp.ctypes.data, nnz, 0, _stream_ptr(stream), C.byref(h)))
        else:
            nnz = int(values.numel())
            if device is None:
                device = values.device.index
            check(L.macko_dev_from_csr(device, rows, cols, b_delta, values.data_ptr() if nnz else None,
                                       col_idx.data_ptr() if nnz else None, row_ptrs.data_ptr(), nnz, 1,
                                       _stream_ptr(stream), C.byref(h)))
        return cls(h.value)

    def to_dense(self, out=None, stream=None):
        """dense_from_macko on the GPU: into a torch CUDA tensor `out` (rows x cols fp16) or, with
        out=None, a host numpy uint16 array."""
        L = _lib.load()
        if out is None:
            host = np.zeros((self.rows, self.cols), np.uint16)
            check(L.macko_dev_to_dense(self._h, host.ctypes.data, self.cols, 0, _stream_ptr(stream)))
            return host
        check(L.macko_dev_to_dense(self._h, out.data_ptr(), out.stride(0), 1, _stream_ptr(stream)))
        return out

    def padding_count(self, stream=None) -> int:
        """padding_count: zero-valued stored entries (pad_nnz - nnz of the source)."""
        n = C.c_uint64()
        check(_lib.load().macko_dev_padding_count(self._h, C.byref(n), _stream_ptr(stream)))
        return n.value

    # -- properties -------------------------------------------------------------------------
    @property
    def rows(self) -> int:
        return self.info.rows

    @property
    def cols(self) -> int:
        return self.info.cols

    @property
    def pad_nnz(self) -> int:
        return self.info.pad_nnz

    @property
    def b_delta(self) -> int:
        return self.info.b_delta

    @property
    def traffic_bytes(self) -> int:
        """Algorithmic bytes of one SpMV (spmv_traffic)."""
        return self.info.traffic_bytes

    def launch_info(self) -> _lib.LaunchInfo:
        li = _lib.LaunchInfo()
        check(_lib.load().macko_dev_launch_info(self._h, C.byref(li)))
        return li

    def plan_records(self):
        """(warp records as an (W, 12) uint32 array, split records as (S, 4) uint32) — introspection."""
        li = self.launch_info()
        recs = np.zeros((li.warps, 12), np.uint32)
        splits = np.zeros((max(li.n_split_rows, 1), 4), np.uint32)
        check(_lib.load().macko_dev_plan_records(self._h, recs.ctypes.data, recs.nbytes, splits.ctypes.data,
                                                 splits.nbytes, None))
        return recs, splits[: li.n_split_rows]

    def configure(self, x_mode: int = -1, ctas_per_sm: int = 0, stream=None) -> None:
        """Re-plan the launch (x_mode: -1 auto, 0 texture only, 1 shared table only, 6 / 7 / 8 / 10
        split; CTA cap k/4 or 0 = auto).  y is bit-identical for every setting."""
        check(_lib.load().macko_dev_configure(self._h, x_mode, ctas_per_sm, _stream_ptr(stream)))

    def set_chain_skew(self, start_spread_ns: int = 2000, stream=None) -> None:
        """Re-plan for PDL-chained launches: later CTAs, which start up to start_spread_ns after
        the first one in a chain, get proportionally less work (0: equal split).  y unchanged."""
        check(_lib.load().macko_dev_set_chain_skew(self._h, int(start_spread_ns), _stream_ptr(stream)))

    # -- operations -------------------------------------------------------------------------
    def download(self, stream=None) -> MackoMatrix:
        i = self.info
        vals = np.zeros(i.values_bytes // 2, np.uint16)
        dl = np.zeros(i.delta_bytes, np.uint8)
        rp = np.zeros(i.rows + 1, np.uint32)
        check(_lib.load().macko_dev_download(self._h, vals.ctypes.data if vals.size else None,
                                             dl.ctypes.data if dl.size else None, rp.ctypes.data, _stream_ptr(stream)))
        return MackoMatrix(i.rows, i.cols, i.b_delta, vals, dl, rp)

    def validate(self, stream=None) -> None:
        check(_lib.load().macko_dev_validate(self._h, _stream_ptr(stream)))

    def spmv_into(self, x, y, stream=None, pdl: bool = False, peers: bool = False, bank: int = 0) -> None:
        """y = A*x with device tensors / pointers (stream-ordered, asynchronous).  pdl: launch as
        a programmatic dependent of the previous kernel on the stream (SpMV chains).  peers: also
        store y into the peer buffers of set_peers (bank 0) or set_peer_bank(1, ...) (bank 1) and
        signal their flags (fused all-gather)."""
        flags = (1 if pdl else 0) | (2 if peers else 0) | (4 if (peers and bank) else 0)
        if flags:
            check(_lib.load().macko_dev_spmv_ex(self._h, _ptr(x), _ptr(y), _stream_ptr(stream), flags))
        else:
            check(_lib.load().macko_dev_spmv(self._h, _ptr(x), _ptr(y), _stream_ptr(stream)))

    def spmm_into(self, X, Y, stream=None) -> None:
        """Y = A X^T for a small batch: X (batch x cols) and Y (batch x rows) fp16 CUDA tensors with
        unit column stride, 1 <= batch <= 8; the matrix streams once (macko_dev_spmm).  Row b of Y
        is bit-identical to spmv_into(X[b])."""
        if X.dim() != 2 or Y.dim() != 2 or X.shape[0] != Y.shape[0]:
            raise ValueError("X and Y must be (batch x cols) and (batch x rows)")
        if X.shape[1] != self.cols or Y.shape[1] != self.rows:
            raise ValueError("dimension mismatch")
        if X.stride(1) != 1 or Y.stride(1) != 1:
            raise ValueError("X and Y rows must be contiguous")
        check(_lib.load().macko_dev_spmm(self._h, _ptr(X), X.stride(0), _ptr(Y), Y.stride(0), X.shape[0],
                                         _stream_ptr(stream)))

    def set_peers(self, peer_y: Sequence[int], peer_flags: Sequence[int], stream=None) -> None:
        """Fused all-gather destinations (device / IPC-mapped addresses; see macko_dev_set_peers)."""
        n = len(peer_y)
        ys = (C.c_void_p * max(n, 1))(*peer_y)
        fs = (C.c_void_p * max(n, 1))(*peer_flags)
        check(_lib.load().macko_dev_set_peers(self._h, ys, fs, n, _stream_ptr(stream)))

    def set_peer_bank(self, bank: int, peer_y: Sequence[int], stream=None) -> None:
        """Second set of y destinations (double-buffered fused all-gather)."""
        n = len(peer_y)
        ys = (C.c_void_p * max(n, 1))(*peer_y)
        check(_lib.load().macko_dev_set_peer_bank(self._h, bank, ys, n, _stream_ptr(stream)))

    def spmv_host(self, x: np.ndarray, y: np.ndarray | None = None, stream=None) -> np.ndarray:
        """End-to-end call with host buffers (H2D x, kernel, D2H y, synchronise)."""
        x = np.ascontiguousarray(x, np.uint16)
        if x.shape != (self.cols,):
            raise ValueError("dimension mismatch: x must have cols entries")
        if y is None:
            y = np.zeros(self.rows, np.uint16)
        elif not (isinstance(y, np.ndarray) and y.dtype == np.uint16 and y.shape == (self.rows,)
                  and y.flags.c_contiguous and y.flags.writeable):
            raise ValueError("y must be a writeable C-contiguous uint16 array of rows entries")
        check(_lib.load().macko_spmv_host(self._h, x.ctypes.data, y.ctypes.data, _stream_ptr(stream)))
        return y

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.load().macko_dev_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def unit_steps() -> int:
    """Steps per reduction unit of the SpMV's summation order (oracle b200_order_spmv's unit_steps)."""
    return int(_lib.load().macko_unit_steps())


def macko_from_dense(dense, b_delta: int = 4, stream=None) -> DeviceMatrix:
    """csr_from_dense + macko_from_csr (convert.hpp:8-16) on the GPU."""
    return DeviceMatrix.from_dense(dense, b_delta=b_delta, stream=stream)


def csr_from_dense(dense, device: int = 0, stream=None):
    """csr_from_dense (convert.hpp:8-10) on the GPU: (values uint16, col_idx uint32, row_ptrs uint32)
    host arrays from a host numpy (rows x cols uint16) or CUDA torch fp16 matrix."""
    L = _lib.load()
    if isinstance(dense, np.ndarray):
        d = np.ascontiguousarray(dense, np.uint16)
        rows, cols = d.shape
        ptr, ld, on_dev = d.ctypes.data, cols, 0
    else:
        rows, cols = dense.shape
        ptr, ld, on_dev = dense.data_ptr(), dense.stride(0), 1
        device = dense.device.index
    rp = np.zeros(rows + 1, np.uint32)
    n = C.c_uint64()
    check(L.macko_csr_from_dense(device, ptr, rows, cols, ld, on_dev, rp.ctypes.data, None, None, C.byref(n),
                                 _stream_ptr(stream)))
    vals = np.zeros(max(n.value, 1), np.uint16)
    ci = np.zeros(max(n.value, 1), np.uint32)
    check(L.macko_csr_from_dense(device, ptr, rows, cols, ld, on_dev, rp.ctypes.data, vals.ctypes.data,
                                 ci.ctypes.data, C.byref(n), _stream_ptr(stream)))
    return vals[: n.value], ci[: n.value], rp


def macko_from_csr(values, col_idx, row_ptrs, rows: int, cols: int, b_delta: int = 4, stream=None) -> DeviceMatrix:
    """macko_from_csr (convert.hpp:12-16) on the GPU."""
    return DeviceMatrix.from_csr(values, col_idx, row_ptrs, rows, cols, b_delta, stream=stream)


def spmv(m: DeviceMatrix, x, y=None, stream=None):
    """reference_spmv on the GPU for a torch CUDA fp16/uint16 vector x."""
    import torch

    if x.shape[-1] != m.cols:
        raise ValueError("dimension mismatch: x must have cols entries")
    if y is None:
        y = torch.empty(m.rows, dtype=x.dtype, device=x.device)
    m.spmv_into(x, y, stream)
    return y


def _path(path) -> bytes:
    import os

    return os.fsencode(path)


def write_mcko(m, path) -> None:
    """write_macko: a DeviceMatrix (streamed from HBM) or a host MackoMatrix."""
    L = _lib.load()
    if isinstance(m, DeviceMatrix):
        check(L.macko_mcko_write_dev(m._h, _path(path), None))
        return
    vals = np.ascontiguousarray(m.values, np.uint16)
    dl = np.ascontiguousarray(m.packed_deltas, np.uint8)
    rp = np.ascontiguousarray(m.row_pointers, np.uint32)
    check(L.macko_mcko_write(_path(path), m.rows, m.cols, m.b_delta, vals.ctypes.data if vals.size else None, len(vals),
                             dl.ctypes.data if dl.size else None, len(dl), rp.ctypes.data))


def mcko_info(path) -> _lib.DevInfo:
    info = _lib.DevInfo()
    check(_lib.load().macko_mcko_read_info(_path(path), C.byref(info)))
    return info


def read_mcko_host(path) -> MackoMatrix:
    """read_macko into host arrays (validated like validate_macko)."""
    i = mcko_info(path)
    vals = np.zeros(i.values_bytes // 2, np.uint16)
    dl = np.zeros(i.delta_bytes, np.uint8)
    rp = np.zeros(i.rows + 1, np.uint32)
    check(_lib.load().macko_mcko_read(_path(path), vals.ctypes.data if vals.size else None,
                                      dl.ctypes.data if dl.size else None, rp.ctypes.data))
    return MackoMatrix(i.rows, i.cols, i.b_delta, vals, dl, rp)


def read_mcko(path, device: int = 0, stream=None) -> DeviceMatrix:
    """MCKO file -> device matrix (sections streamed through pinned buffers, validated on the GPU)."""
    h = C.c_void_p()
    check(_lib.load().macko_mcko_read_dev(device, _path(path), _stream_ptr(stream), C.byref(h)))
    return DeviceMatrix(h.value)


def read_matrix_market(path) -> np.ndarray:
    """read_matrix_market -> dense fp16 bits (rows x cols uint16)."""
    L = _lib.load()
    r, c = C.c_uint64(), C.c_uint64()
    check(L.macko_mm_read_dense(_path(path), C.byref(r), C.byref(c), None))
    out = np.zeros((r.value, c.value), np.uint16)
    check(L.macko_mm_read_dense(_path(path), C.byref(r), C.byref(c), out.ctypes.data))
    return out


def density_threshold(d: float) -> int:
    return _lib.load().macko_density_threshold(d)


def gen_dense(out, rows: int, cols: int, density: float, seed: int, int_mode: bool = False, row0: int = 0,
              device: int | None = None, stream=None) -> None:
    """Fill a device fp16 matrix with the counter-hash generator (bit-identical to the oracle)."""
    ld = out.stride(0) if not isinstance(out, int) else cols
    if device is None:
        device = out.device.index if not isinstance(out, int) else 0
    check(_lib.load().macko_gen_dense(device, _ptr(out), rows, cols, ld, row0, density_threshold(density), seed,
                                      int(int_mode), _stream_ptr(stream)))


def gen_vector(out, n: int, seed: int, int_mode: bool = False, device: int | None = None, stream=None) -> None:
    if device is None:
        device = out.device.index if not isinstance(out, int) else 0
    check(_lib.load().macko_gen_vector(device, _ptr(out), n, seed, int(int_mode), _stream_ptr(stream)))


def shard_rows(rows: int, n_shards: int, shard: int) -> tuple[int, int]:
    """Contiguous equal-row slab [r0, r1) of shard `shard`."""
    r0, r1 = C.c_uint64(), C.c_uint64()
    check(_lib.load().macko_shard_rows(rows, n_shards, shard, C.byref(r0), C.byref(r1)))
    return r0.value, r1.value


def kernel_launches() -> int:
    return _lib.load().macko_kernel_launches()


def version() -> str:
    return _lib.load().macko_version().decode()


def wait_flags(flags, n: int, target: int, stream=None) -> None:
    """Stream-ordered wait until flags[i] >= target for i < n (macko_wait_flags)."""
    check(_lib.load().macko_wait_flags(_ptr(flags), n, target & 0xFFFFFFFF, _stream_ptr(stream)))


def ipc_handle(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding t, t's byte offset in it)."""
    buf = C.create_string_buffer(64)
    off = C.c_uint64()
    check(_lib.load().macko_ipc_get_handle(_ptr(t), buf, C.byref(off)))
    return buf.raw, off.value


def ipc_open(handle: bytes, device: int) -> int:
    """Map a peer allocation; returns its base address (close with ipc_close)."""
    p = C.c_void_p()
    check(_lib.load().macko_ipc_open(handle, device, C.byref(p)))
    return p.value


def ipc_close(ptr: int) -> None:
    check(_lib.load().macko_ipc_close(ptr))
