"""B200-native MACKO-SpMV (arxiv 2511.13061): GPU compressor + sm_100a SpMV behind a C-ABI.

The product is libmacko_cuda.so (include/macko_cuda.h).  This package is the thin host-side
mirror of the reference interface used by tests and bench.py; it never falls back to CPU.
"""
from .macko import (  # noqa: F401
    CudaError,
    DeviceMatrix,
    FormatError,
    InfeasibleError,
    IoError,
    MackoMatrix,
    delta_bytes,
    density_threshold,
    gen_dense,
    gen_vector,
    kernel_launches,
    csr_from_dense,
    macko_from_csr,
    macko_from_dense,
    mcko_info,
    read_matrix_market,
    read_mcko,
    read_mcko_host,
    shard_rows,
    spmv,
    values_bytes,
    version,
    wait_flags,
    write_mcko,
)
