"""ctypes binding of libmacko_cuda.so (the C-ABI in include/macko_cuda.h).

The library is built in-tree (``make lib`` / ``__graft_entry__.build()``).  There is no CPU
fallback: if the shared object is missing or fails to load, importing the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MACKO_LIB overrides the library path (the opt-in trace build, `make trace`); default in-tree .so
LIB_PATH = os.environ.get("MACKO_LIB") or os.path.join(HERE, "libmacko_cuda.so")

MACKO_OK, MACKO_EINVAL, MACKO_EFORMAT, MACKO_EIO, MACKO_EINFEASIBLE, MACKO_ECUDA, MACKO_ENCCL, MACKO_ENOMEM = range(8)

# Every symbol include/macko_cuda.h declares (tests check the library exports all of them).
EXPORTS = (
    "macko_last_error", "macko_version", "macko_unit_steps", "macko_dev_upload", "macko_dev_from_dense", "macko_dev_from_csr", "macko_csr_from_dense",
    "macko_dev_to_dense", "macko_dev_padding_count", "macko_dev_get_info",
    "macko_dev_download", "macko_dev_spmv", "macko_dev_spmv_ex", "macko_dev_spmm", "macko_spmv_host", "macko_dev_validate", "macko_dev_free", "macko_release_cached_memory", "macko_dev_set_chain_skew",
    "macko_density_threshold", "macko_gen_dense", "macko_gen_vector", "macko_shard_rows",
    "macko_dev_launch_info", "macko_dev_plan_records", "macko_dev_configure", "macko_kernel_launches",
    "macko_mcko_write", "macko_mcko_read_info", "macko_mcko_read", "macko_mcko_write_dev", "macko_mcko_read_dev",
    "macko_mm_read_dense", "macko_sharded_spmv",
    "macko_dev_set_peers", "macko_dev_set_peer_bank", "macko_wait_flags", "macko_ipc_get_handle", "macko_ipc_open", "macko_ipc_close",
)


class FormatError(RuntimeError):
    """macko::FormatError (reference errors.hpp:9-11)."""


class IoError(RuntimeError):
    """macko::IoError (reference errors.hpp:14-16)."""


class InfeasibleError(RuntimeError):
    """macko::InfeasibleError (reference errors.hpp:19-21)."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside libmacko_cuda."""


_ERRORS = {
    MACKO_EINVAL: ValueError,  # std::invalid_argument
    MACKO_EFORMAT: FormatError,
    MACKO_EIO: IoError,
    MACKO_EINFEASIBLE: InfeasibleError,
    MACKO_ECUDA: CudaError,
    MACKO_ENCCL: CudaError,
    MACKO_ENOMEM: MemoryError,
}


class DevInfo(C.Structure):
    _fields_ = [
        ("rows", C.c_uint64), ("cols", C.c_uint64), ("pad_nnz", C.c_uint64),
        ("values_bytes", C.c_uint64), ("delta_bytes", C.c_uint64), ("row_ptr_bytes", C.c_uint64),
        ("traffic_bytes", C.c_uint64), ("b_delta", C.c_uint32), ("device", C.c_int32),
        ("d_values", C.c_void_p), ("d_deltas", C.c_void_p), ("d_row_ptrs", C.c_void_p),
    ]


class LaunchInfo(C.Structure):
    _fields_ = [
        ("grid", C.c_uint32), ("block", C.c_uint32), ("warps", C.c_uint32), ("ctas_per_sm", C.c_uint32),
        ("n_split_rows", C.c_uint32), ("x_in_smem", C.c_uint32), ("n_units", C.c_uint64), ("smem_bytes", C.c_uint64),
        ("reserved0", C.c_uint32), ("reserved", C.c_uint32),
    ]


_lib = None


def load() -> C.CDLL:
    """Load libmacko_cuda.so (raises OSError if it is not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"libmacko_cuda.so not built at {LIB_PATH}; run `make lib` (or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, u64, u32, i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
    st = C.c_int
    L.macko_last_error.restype = C.c_char_p
    L.macko_version.restype = C.c_char_p
    L.macko_dev_upload.restype = st
    L.macko_dev_upload.argtypes = [i32, u64, u64, u32, vp, u64, vp, u64, vp, vp, C.POINTER(vp)]
    L.macko_dev_from_dense.restype = st
    L.macko_dev_from_dense.argtypes = [i32, vp, u64, u64, u64, u32, vp, C.POINTER(vp)]
    L.macko_dev_from_csr.restype = st
    L.macko_dev_from_csr.argtypes = [i32, u64, u64, u32, vp, vp, vp, u64, i32, vp, C.POINTER(vp)]
    L.macko_csr_from_dense.restype = st
    L.macko_csr_from_dense.argtypes = [i32, vp, u64, u64, u64, i32, vp, vp, vp, C.POINTER(u64), vp]
    L.macko_dev_to_dense.restype = st
    L.macko_dev_to_dense.argtypes = [vp, vp, u64, i32, vp]
    L.macko_dev_padding_count.restype = st
    L.macko_dev_padding_count.argtypes = [vp, C.POINTER(u64), vp]
    L.macko_dev_get_info.restype = st
    L.macko_dev_get_info.argtypes = [vp, C.POINTER(DevInfo)]
    L.macko_dev_download.restype = st
    L.macko_dev_download.argtypes = [vp, vp, vp, vp, vp]
    L.macko_dev_spmv.restype = st
    L.macko_dev_spmv.argtypes = [vp, vp, vp, vp]
    L.macko_dev_spmv_ex.restype = st
    L.macko_dev_spmv_ex.argtypes = [vp, vp, vp, vp, C.c_uint32]
    L.macko_dev_spmm.restype = st
    L.macko_dev_spmm.argtypes = [vp, vp, u64, vp, u64, u32, vp]
    L.macko_spmv_host.restype = st
    L.macko_spmv_host.argtypes = [vp, vp, vp, vp]
    L.macko_dev_validate.restype = st
    L.macko_dev_validate.argtypes = [vp, vp]
    L.macko_unit_steps.restype = C.c_uint32
    L.macko_unit_steps.argtypes = []
    L.macko_dev_free.restype = st
    L.macko_dev_free.argtypes = [vp]
    L.macko_release_cached_memory.restype = st
    L.macko_release_cached_memory.argtypes = []
    L.macko_dev_set_chain_skew.restype = st
    L.macko_dev_set_chain_skew.argtypes = [vp, C.c_uint32, vp]
    L.macko_density_threshold.restype = u32
    L.macko_density_threshold.argtypes = [C.c_double]
    L.macko_gen_dense.restype = st
    L.macko_gen_dense.argtypes = [i32, vp, u64, u64, u64, u64, u32, u64, i32, vp]
    L.macko_gen_vector.restype = st
    L.macko_gen_vector.argtypes = [i32, vp, u64, u64, i32, vp]
    L.macko_shard_rows.restype = st
    L.macko_shard_rows.argtypes = [u64, u32, u32, C.POINTER(u64), C.POINTER(u64)]
    cp = C.c_char_p
    L.macko_mcko_write.restype = st
    L.macko_mcko_write.argtypes = [cp, u64, u64, u32, vp, u64, vp, u64, vp]
    L.macko_mcko_read_info.restype = st
    L.macko_mcko_read_info.argtypes = [cp, C.POINTER(DevInfo)]
    L.macko_mcko_read.restype = st
    L.macko_mcko_read.argtypes = [cp, vp, vp, vp]
    L.macko_mcko_write_dev.restype = st
    L.macko_mcko_write_dev.argtypes = [vp, cp, vp]
    L.macko_mcko_read_dev.restype = st
    L.macko_mcko_read_dev.argtypes = [C.c_int, cp, vp, C.POINTER(vp)]
    L.macko_sharded_spmv.restype = st
    L.macko_sharded_spmv.argtypes = [vp, vp, C.c_int, vp, vp, C.c_uint64, vp]
    L.macko_dev_set_peers.restype = st
    L.macko_dev_set_peers.argtypes = [vp, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_uint32, vp]
    L.macko_dev_set_peer_bank.restype = st
    L.macko_dev_set_peer_bank.argtypes = [vp, C.c_uint32, C.POINTER(C.c_void_p), C.c_uint32, vp]
    L.macko_wait_flags.restype = st
    L.macko_wait_flags.argtypes = [vp, C.c_uint32, C.c_uint32, vp]
    L.macko_ipc_get_handle.restype = st
    L.macko_ipc_get_handle.argtypes = [vp, C.c_char_p, C.POINTER(C.c_uint64)]
    L.macko_ipc_open.restype = st
    L.macko_ipc_open.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
    L.macko_ipc_close.restype = st
    L.macko_ipc_close.argtypes = [vp]
    L.macko_mm_read_dense.restype = st
    L.macko_mm_read_dense.argtypes = [cp, C.POINTER(u64), C.POINTER(u64), vp]
    L.macko_dev_launch_info.restype = st
    L.macko_dev_launch_info.argtypes = [vp, C.POINTER(LaunchInfo)]
    L.macko_dev_plan_records.restype = st
    L.macko_dev_plan_records.argtypes = [vp, vp, u64, vp, u64, vp]
    L.macko_dev_configure.restype = st
    L.macko_dev_configure.argtypes = [vp, i32, i32, vp]
    L.macko_kernel_launches.restype = u64
    _lib = L
    return L


def check(code: int) -> None:
    if code != MACKO_OK:
        msg = load().macko_last_error().decode(errors="replace")
        raise _ERRORS.get(code, CudaError)(msg)
