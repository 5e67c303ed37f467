"""ctypes bindings for the CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs
may import this module, and only as the checker or the CPU baseline.  The product package
``paper_2511_13061_b200`` never imports it.

Two libraries:
  * ``libmacko_oracle.so`` — plain-C restatement of the reference algorithm (macko_oracle.c);
  * ``_ref/libmacko_ref.so`` — the reference's own fp16.cpp / bitpack.cpp / headers compiled
    from /root/reference plus ref_shim.cpp (restated absent bodies).  Built in this container
    and shipped prebuilt to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u64 = C.c_uint64


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise OSError(f"oracle library missing: {path} (run `make -C oracle`)")
    return C.CDLL(path)


_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        L = _load(os.path.join(HERE, "libmacko_oracle.so"))
        L.mo_last_error.restype = C.c_char_p
        L.mo_float_to_half.restype = C.c_uint16
        L.mo_float_to_half.argtypes = [C.c_float]
        L.mo_half_to_float.restype = C.c_float
        L.mo_half_to_float.argtypes = [C.c_uint16]
        L.mo_float_to_half_array.argtypes = [_f32p, _u64, _u16p]
        L.mo_half_to_float_array.argtypes = [_u16p, _u64, _f32p]
        L.mo_pack_deltas.argtypes = [_u32p, _u64, C.c_uint, _u8p]
        L.mo_unpack_deltas.argtypes = [_u8p, _u64, C.c_uint, _u32p]
        for f in ("mo_values_bytes",):
            getattr(L, f).restype = _u64
            getattr(L, f).argtypes = [_u64]
        L.mo_delta_bytes.restype = _u64
        L.mo_delta_bytes.argtypes = [_u64, C.c_uint]
        L.mo_csr_count.restype = _u64
        L.mo_csr_count.argtypes = [_u16p, _u64, _u64, _u32p]
        L.mo_csr_fill.argtypes = [_u16p, _u64, _u64, _u32p, _u16p, _u32p]
        L.mo_macko_count.argtypes = [_u64, _u64, _u32p, _u32p, C.c_uint, _u32p, C.POINTER(_u64)]
        L.mo_macko_fill.argtypes = [_u64, _u64, _u32p, _u32p, _u16p, C.c_uint, _u32p, _u16p, _u8p]
        L.mo_encode_dense_count.argtypes = [_u16p, _u64, _u64, C.c_uint, _u32p, C.POINTER(_u64)]
        L.mo_encode_dense_fill.argtypes = [_u16p, _u64, _u64, C.c_uint, _u32p, _u16p, _u8p]
        L.mo_dense_from_macko.argtypes = [_u64, _u64, C.c_uint, _u16p, _u8p, _u32p, _u16p]
        L.mo_validate_macko.argtypes = [_u64, _u64, C.c_uint, _u16p, _u64, _u8p, _u64, _u32p]
        L.mo_padding_count.restype = _u64
        L.mo_padding_count.argtypes = [_u64, _u16p, _u32p]
        L.mo_dense_mv.argtypes = [_u16p, _u64, _u64, _u16p, _u16p]
        L.mo_reference_spmv.argtypes = [_u64, _u64, C.c_uint, _u16p, _u8p, _u32p, _u16p, _u16p, C.c_int]
        L.mo_warp_prefix_sum.argtypes = [_u32p, _u32p]
        L.mo_warp_spmv.argtypes = [_u64, _u64, C.c_uint, _u16p, _u8p, _u32p, _u16p, _u16p]
        L.mo_b200_order_spmv.argtypes = [_u64, _u64, C.c_uint, _u16p, _u8p, _u32p, _u16p, _u16p, C.c_uint]
        L.mo_b200_order_spmv_mt.argtypes = [_u64, _u64, C.c_uint, _u16p, _u8p, _u32p, _u16p, _u16p, C.c_uint, C.c_int]
        L.mo_gen_dense_rows_mt.argtypes = [_u64, _u64, _u64, C.c_uint32, _u64, C.c_int, _u16p, C.c_int]
        L.mo_encode_dense_count_mt.argtypes = [_u16p, _u64, _u64, C.c_uint, _u32p, C.POINTER(_u64), C.c_int]
        L.mo_encode_dense_fill_mt.argtypes = [_u16p, _u64, _u64, C.c_uint, _u32p, _u16p, _u8p, C.c_int]
        L.mo_density_threshold.restype = C.c_uint32
        L.mo_density_threshold.argtypes = [C.c_double]
        L.mo_gen_dense.argtypes = [_u64, _u64, C.c_uint32, _u64, C.c_int, _u16p]
        L.mo_gen_vector.argtypes = [_u64, _u64, C.c_int, _u16p]
        L.mo_gen_worst_case.argtypes = [_u64, _u64, _u64, _u16p]
        L.mo_spmv_traffic_bytes.restype = _u64
        L.mo_spmv_traffic_bytes.argtypes = [_u64, _u64, _u64, C.c_uint]
        L.mo_dense_traffic_bytes.restype = _u64
        L.mo_dense_traffic_bytes.argtypes = [_u64, _u64]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libmacko_ref.so"))


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        R = _load(os.path.join(HERE, "_ref", "libmacko_ref.so"))
        R.ref_last_error.restype = C.c_char_p
        R.ref_float_to_half.restype = C.c_uint16
        R.ref_float_to_half.argtypes = [C.c_float]
        R.ref_half_to_float.restype = C.c_float
        R.ref_half_to_float.argtypes = [C.c_uint16]
        R.ref_float_to_half_array.argtypes = [_f32p, _u64, _u16p]
        R.ref_half_to_float_array.argtypes = [_u16p, _u64, _f32p]
        R.ref_pack_deltas.argtypes = [_u32p, _u64, C.c_uint, _u8p, _u64]
        R.ref_unpack_deltas.argtypes = [_u8p, _u64, C.c_uint, _u32p]
        R.ref_encode_dense.argtypes = [_u16p, _u64, _u64, C.c_uint, C.POINTER(C.c_void_p)]
        R.ref_from_arrays.argtypes = [_u64, _u64, C.c_uint, _u16p, _u64, _u8p, _u64, _u32p, C.POINTER(C.c_void_p)]
        R.ref_matrix_info.argtypes = [C.c_void_p, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]
        R.ref_matrix_copy.argtypes = [C.c_void_p, _u16p, _u8p, _u32p]
        R.ref_matrix_free.argtypes = [C.c_void_p]
        R.ref_dense_from_macko.argtypes = [C.c_void_p, _u16p]
        R.ref_validate.argtypes = [C.c_void_p]
        R.ref_padding_count.restype = _u64
        R.ref_padding_count.argtypes = [C.c_void_p]
        R.ref_spmv.argtypes = [C.c_void_p, _u16p, _u16p, C.c_int]
        R.ref_dense_mv.argtypes = [_u16p, _u64, _u64, _u16p, _u16p]
        _ref = R
    return _ref


def _check(code: int, which: str = "oracle") -> None:
    if code != 0:
        msg = (lib().mo_last_error() if which == "oracle" else ref().ref_last_error()).decode()
        raise OracleError(code, msg)


@dataclass
class Macko:
    """Host MACKO arrays (bit layout of reference matrix.hpp:57-81)."""

    rows: int
    cols: int
    b_delta: int
    values: np.ndarray  # uint16, values_bytes/2 entries (tail zero-padded)
    deltas: np.ndarray  # uint8, delta_bytes (tail zero-padded)
    row_ptrs: np.ndarray  # uint32, rows+1

    @property
    def pad_nnz(self) -> int:
        return int(self.row_ptrs[-1]) if len(self.row_ptrs) else 0


# ---------------------------------------------------------------- restatement (macko_oracle.c)
def float_to_half(x: float) -> int:
    return lib().mo_float_to_half(x)


def half_to_float(h: int) -> float:
    return lib().mo_half_to_float(h)


def float_to_half_array(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros(max(x.size, 1), np.uint16)
    lib().mo_float_to_half_array(x.reshape(-1), x.size, out)
    return out[: x.size].reshape(x.shape)


def half_to_float_array(h: np.ndarray) -> np.ndarray:
    h = np.ascontiguousarray(h, np.uint16)
    out = np.zeros(max(h.size, 1), np.float32)
    lib().mo_half_to_float_array(h.reshape(-1), h.size, out)
    return out[: h.size].reshape(h.shape)


def pack_deltas(deltas, bits: int) -> np.ndarray:
    d = np.ascontiguousarray(deltas, dtype=np.uint32)
    per = 8 // bits if bits in (1, 2, 4, 8) else 1
    out = np.zeros(max(1, (len(d) + per - 1) // per), np.uint8)
    _check(lib().mo_pack_deltas(d, len(d), bits, out))
    return out[: (len(d) + per - 1) // per]


def unpack_deltas(b: np.ndarray, n: int, bits: int) -> np.ndarray:
    out = np.zeros(max(n, 1), np.uint32)
    _check(lib().mo_unpack_deltas(np.ascontiguousarray(b, np.uint8), n, bits, out))
    return out[:n]


def values_bytes(pad_nnz: int) -> int:
    return lib().mo_values_bytes(pad_nnz)


def delta_bytes(pad_nnz: int, bits: int) -> int:
    return lib().mo_delta_bytes(pad_nnz, bits)


def csr_from_dense(dense: np.ndarray):
    d = np.ascontiguousarray(dense, np.uint16)
    R, Cc = d.shape
    rp = np.zeros(R + 1, np.uint32)
    nnz = lib().mo_csr_count(d, R, Cc, rp)
    vals = np.zeros(max(nnz, 1), np.uint16)
    cols = np.zeros(max(nnz, 1), np.uint32)
    lib().mo_csr_fill(d, R, Cc, rp, vals, cols)
    return vals[:nnz], cols[:nnz], rp


def macko_from_csr(rows: int, cols: int, vals, col_idx, rp, bits: int = 4) -> Macko:
    v = np.ascontiguousarray(vals, np.uint16)
    ci = np.ascontiguousarray(col_idx, np.uint32)
    crp = np.ascontiguousarray(rp, np.uint32)
    if len(v) == 0:
        v = np.zeros(1, np.uint16)
        ci = np.zeros(1, np.uint32)
    mrp = np.zeros(rows + 1, np.uint32)
    pn = _u64(0)
    _check(lib().mo_macko_count(rows, cols, crp, ci, bits, mrp, C.byref(pn)))
    values = np.zeros(values_bytes(pn.value) // 2, np.uint16)
    deltas = np.zeros(delta_bytes(pn.value, bits), np.uint8)
    _check(lib().mo_macko_fill(rows, cols, crp, ci, v, bits, mrp, _nz(values), _nz(deltas)))
    return Macko(rows, cols, bits, values, deltas, mrp)


def _nz(a: np.ndarray) -> np.ndarray:
    """ctypes ndpointer rejects empty arrays' null data only sometimes; keep a 1-elt buffer."""
    return a if a.size else np.zeros(1, a.dtype)


def encode_dense(dense: np.ndarray, bits: int = 4, nthreads: int = 1) -> Macko:
    d = np.ascontiguousarray(dense, np.uint16)
    R, Cc = d.shape
    rp = np.zeros(R + 1, np.uint32)
    pn = _u64(0)
    if nthreads > 1:
        _check(lib().mo_encode_dense_count_mt(_nz(d.reshape(-1)), R, Cc, bits, rp, C.byref(pn), nthreads))
    else:
        _check(lib().mo_encode_dense_count(_nz(d.reshape(-1)), R, Cc, bits, rp, C.byref(pn)))
    values = np.zeros(values_bytes(pn.value) // 2, np.uint16)
    deltas = np.zeros(delta_bytes(pn.value, bits), np.uint8)
    if pn.value:
        if nthreads > 1:
            _check(lib().mo_encode_dense_fill_mt(_nz(d.reshape(-1)), R, Cc, bits, rp, values, deltas, nthreads))
        else:
            _check(lib().mo_encode_dense_fill(_nz(d.reshape(-1)), R, Cc, bits, rp, values, deltas))
    return Macko(R, Cc, bits, values, deltas, rp)


def dense_from_macko(m: Macko) -> np.ndarray:
    out = np.zeros(max(m.rows * m.cols, 1), np.uint16)
    _check(lib().mo_dense_from_macko(m.rows, m.cols, m.b_delta, _nz(m.values), _nz(m.deltas), m.row_ptrs, out))
    return out[: m.rows * m.cols].reshape(m.rows, m.cols)


def validate_macko(m: Macko) -> None:
    _check(lib().mo_validate_macko(m.rows, m.cols, m.b_delta, _nz(m.values), len(m.values),
                                   _nz(m.deltas), len(m.deltas), m.row_ptrs))


def padding_count(m: Macko) -> int:
    return lib().mo_padding_count(m.rows, _nz(m.values), m.row_ptrs)


def dense_mv(dense: np.ndarray, x: np.ndarray) -> np.ndarray:
    d = np.ascontiguousarray(dense, np.uint16)
    y = np.zeros(max(d.shape[0], 1), np.uint16)
    lib().mo_dense_mv(_nz(d.reshape(-1)), d.shape[0], d.shape[1], np.ascontiguousarray(x, np.uint16), y)
    return y[: d.shape[0]]


def reference_spmv(m: Macko, x: np.ndarray, nthreads: int = 1) -> np.ndarray:
    y = np.zeros(max(m.rows, 1), np.uint16)
    _check(lib().mo_reference_spmv(m.rows, m.cols, m.b_delta, _nz(m.values), _nz(m.deltas), m.row_ptrs,
                                   _nz(np.ascontiguousarray(x, np.uint16)), y, nthreads))
    return y[: m.rows]


def warp_prefix_sum(local) -> np.ndarray:
    out = np.zeros(32, np.uint32)
    lib().mo_warp_prefix_sum(np.ascontiguousarray(local, np.uint32), out)
    return out


def warp_spmv(m: Macko, x: np.ndarray) -> np.ndarray:
    y = np.zeros(max(m.rows, 1), np.uint16)
    _check(lib().mo_warp_spmv(m.rows, m.cols, m.b_delta, _nz(m.values), _nz(m.deltas), m.row_ptrs,
                              _nz(np.ascontiguousarray(x, np.uint16)), y))
    return y[: m.rows]


def b200_order_spmv(m: Macko, x: np.ndarray, unit_steps: int, nthreads: int = 1) -> np.ndarray:
    y = np.zeros(max(m.rows, 1), np.uint16)
    xx = _nz(np.ascontiguousarray(x, np.uint16))
    rp = np.ascontiguousarray(m.row_ptrs, np.uint32)
    if nthreads > 1:
        _check(lib().mo_b200_order_spmv_mt(m.rows, m.cols, m.b_delta, _nz(m.values), _nz(m.deltas), rp, xx, y,
                                           unit_steps, nthreads))
    else:
        _check(lib().mo_b200_order_spmv(m.rows, m.cols, m.b_delta, _nz(m.values), _nz(m.deltas), rp, xx, y,
                                        unit_steps))
    return y[: m.rows]


def density_threshold(d: float) -> int:
    return lib().mo_density_threshold(d)


def gen_dense_rows(row0: int, rows: int, cols: int, density: float, seed: int, int_mode: bool = False,
                   nthreads: int = 1) -> np.ndarray:
    """Rows [row0, row0 + rows) of the generator's conceptual matrix (threaded)."""
    out = np.zeros(max(rows * cols, 1), np.uint16)
    lib().mo_gen_dense_rows_mt(row0, rows, cols, density_threshold(density), seed, int(int_mode), out, nthreads)
    return out[: rows * cols].reshape(rows, cols)


def gen_dense(rows: int, cols: int, density: float, seed: int, int_mode: bool = False) -> np.ndarray:
    out = np.zeros(max(rows * cols, 1), np.uint16)
    lib().mo_gen_dense(rows, cols, density_threshold(density), seed, int(int_mode), out)
    return out[: rows * cols].reshape(rows, cols)


def gen_vector(n: int, seed: int, int_mode: bool = False) -> np.ndarray:
    out = np.zeros(max(n, 1), np.uint16)
    lib().mo_gen_vector(n, seed, int(int_mode), out)
    return out[:n]


def gen_worst_case(rows: int, cols: int, zero_run: int) -> np.ndarray:
    out = np.zeros(max(rows * cols, 1), np.uint16)
    lib().mo_gen_worst_case(rows, cols, zero_run, out)
    return out[: rows * cols].reshape(rows, cols)


def spmv_traffic_bytes(rows: int, cols: int, pad_nnz: int, bits: int = 4) -> int:
    return lib().mo_spmv_traffic_bytes(rows, cols, pad_nnz, bits)


def dense_traffic_bytes(rows: int, cols: int) -> int:
    return lib().mo_dense_traffic_bytes(rows, cols)


# ---------------------------------------------------------------- reference sources (_ref)
class RefMatrix:
    """A reference ``macko::MackoMatrix`` built by the reference's own code path."""

    def __init__(self, handle: int):
        self.h = C.c_void_p(handle)

    @classmethod
    def encode(cls, dense: np.ndarray, bits: int = 4) -> "RefMatrix":
        d = np.ascontiguousarray(dense, np.uint16)
        h = C.c_void_p()
        _check(ref().ref_encode_dense(_nz(d.reshape(-1)), d.shape[0], d.shape[1], bits, C.byref(h)), "ref")
        return cls(h.value)

    @classmethod
    def from_macko(cls, m: Macko) -> "RefMatrix":
        h = C.c_void_p()
        _check(ref().ref_from_arrays(m.rows, m.cols, m.b_delta, _nz(m.values), len(m.values), _nz(m.deltas),
                                     len(m.deltas), m.row_ptrs, C.byref(h)), "ref")
        return cls(h.value)

    def to_macko(self, rows: int, cols: int, bits: int) -> Macko:
        pn, nv, nd = _u64(), _u64(), _u64()
        ref().ref_matrix_info(self.h, C.byref(pn), C.byref(nv), C.byref(nd))
        v = np.zeros(max(nv.value, 1), np.uint16)
        d = np.zeros(max(nd.value, 1), np.uint8)
        rp = np.zeros(rows + 1, np.uint32)
        ref().ref_matrix_copy(self.h, v, d, rp)
        return Macko(rows, cols, bits, v[: nv.value], d[: nd.value], rp)

    def spmv(self, x: np.ndarray, rows: int, nthreads: int = 1) -> np.ndarray:
        y = np.zeros(max(rows, 1), np.uint16)
        _check(ref().ref_spmv(self.h, _nz(np.ascontiguousarray(x, np.uint16)), y, nthreads), "ref")
        return y[:rows]

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value and _ref is not None:
            _ref.ref_matrix_free(self.h)
            self.h = None


# ---------------------------------------------------------------- MCKO container
def mcko_bytes(m: Macko) -> bytes:
    """write_macko restated from SPEC.md:376-386 (io.cpp is absent): 32-byte LE header "MCKO",
    u16 version 1, u8 b_val 16, u8 b_delta, u64 R, u64 C, u64 pad_nnz; then row_pointers
    ((R+1) x u32 LE), packed_deltas (tail-padded to 16 B), values (u16 LE, tail-padded to 16 B)."""
    import struct

    pad_nnz = m.pad_nnz
    db, vb = delta_bytes(pad_nnz, m.b_delta), values_bytes(pad_nnz)
    d = np.zeros(db, np.uint8)
    d[: min(db, m.deltas.size)] = m.deltas[:db]
    v = np.zeros(vb // 2, np.uint16)
    v[: min(vb // 2, m.values.size)] = m.values[: vb // 2]
    head = b"MCKO" + struct.pack("<HBBQQQ", 1, 16, m.b_delta, m.rows, m.cols, pad_nnz)
    return head + np.asarray(m.row_ptrs, "<u4").tobytes() + d.tobytes() + v.astype("<u2").tobytes()
