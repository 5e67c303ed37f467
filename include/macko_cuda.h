/*
 * macko_cuda.h — the C-ABI drop-in boundary of the B200-native MACKO-SpMV library
 * (libmacko_cuda.so, built from paper_2511_13061_b200/csrc/).
 *
 * The reference declares a shared library `macko` exposing "the extern-C surface declared in
 * include/macko/macko.h" (proj/src/CMakeLists.txt:16-19) but ships neither capi.cpp nor the
 * header.  The entry points below are what that surface has to bind for
 * the hot path; each cites the reference C++ operation it replaces.  Plain pointers and sizes
 * only.  `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All
 * device calls are stream-ordered and asynchronous unless stated.  Errors are returned as
 * macko_status; no C++ exception crosses this boundary; macko_last_error() gives the
 * thread-local message.  Status codes map onto the reference's exception taxonomy
 * (errors.hpp:7-21, std::invalid_argument in bitpack.cpp:14-15,26-27,45-46).
 *
 * Matrix byte layout on the device is exactly the reference MackoMatrix (matrix.hpp:57-81):
 * values = pad_nnz fp16 (+0 at padding entries) zero-padded to a 16-byte multiple;
 * packed_deltas = codeword (delta-1) in b_delta bits, LSB-first, zero-padded to 16 bytes;
 * row_pointers = rows+1 u32 element offsets.
 */
#ifndef MACKO_CUDA_H
#define MACKO_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum macko_status {
    MACKO_OK = 0,
    MACKO_EINVAL = 1,      /* std::invalid_argument (bitpack.cpp:14-15; convert.hpp:25) */
    MACKO_EFORMAT = 2,     /* macko::FormatError (errors.hpp:9-11) */
    MACKO_EIO = 3,         /* macko::IoError (errors.hpp:14-16) */
    MACKO_EINFEASIBLE = 4, /* macko::InfeasibleError (errors.hpp:19-21) */
    MACKO_ECUDA = 5,       /* CUDA runtime failure (no reference counterpart) */
    MACKO_ENCCL = 6,       /* NCCL failure (macko_sharded_spmv; no reference counterpart) */
    MACKO_ENOMEM = 7       /* device allocation failure */
} macko_status;

/* Opaque device-resident MACKO matrix (owns its values / deltas / row_pointers buffers and
 * the SpMV work plan).  Immutable after construction: one handle may be used
 * from any number of host threads and streams of its device at once.  Everything a launch
 * mutates besides y (split-row counters and partial sums, the aligned copy of a misaligned x,
 * macko_spmv_host's device buffers) lives in a per-stream workspace, so launches on different
 * streams never share state; x texture objects are cached per x buffer and destroyed only with
 * the handle.  Workspaces are created on a stream's first SpMV, which must not be inside a
 * stream capture (run one SpMV on the capture stream first); a captured CUDA graph uses the
 * workspace of its capture stream.  macko_dev_configure / macko_dev_free must not run
 * concurrently with SpMVs of the same handle. */
typedef struct macko_dev_matrix macko_dev_matrix;

typedef struct macko_dev_info {
    uint64_t rows, cols, pad_nnz;
    uint64_t values_bytes;   /* macko_values_bytes(pad_nnz), matrix.hpp:77 */
    uint64_t delta_bytes;    /* macko_delta_bytes(pad_nnz, b_delta), matrix.hpp:78-81 */
    uint64_t row_ptr_bytes;  /* 4 * (rows + 1) */
    uint64_t traffic_bytes;  /* spmv_traffic bytes_matrix + 2C + 2R */
    uint32_t b_delta;
    int32_t device;
    /* device pointers (read-only views; owned by the handle) */
    const uint16_t* d_values;
    const uint8_t* d_deltas;
    const uint32_t* d_row_ptrs;
} macko_dev_info;

const char* macko_last_error(void);
const char* macko_version(void);
/* Steps (256 elements each) per reduction unit of the SpMV's fixed summation order: per lane
 * sequential, xor-tree over the 32 lanes once per unit, units added in order. */
uint32_t macko_unit_steps(void);

/* Host MACKO arrays -> device handle (copies).  Replaces the host-resident MackoMatrix
 * produced by macko_from_csr (convert.hpp:12-16) as the SpMV operand.  n_values /
 * n_delta_bytes are the host array lengths (>= pad_nnz / ceil(pad_nnz*b_delta/8)).  The
 * arrays are validated on the device (validate_macko, convert.hpp:25-27) before return. */
macko_status macko_dev_upload(int device, uint64_t rows, uint64_t cols, uint32_t b_delta,
                              const uint16_t* values, uint64_t n_values, const uint8_t* deltas,
                              uint64_t n_delta_bytes, const uint32_t* row_ptrs, void* stream,
                              macko_dev_matrix** out);

/* GPU compressor: dense row-major fp16 (device pointer, leading dimension `ld` elements) ->
 * MACKO on the device.  Replaces csr_from_dense + macko_from_csr (convert.hpp:8-16,
 * SPEC.md:54-72); output bytes identical to the reference encoder.  Synchronises `stream`
 * once (the output size is data dependent). */
macko_status macko_dev_from_dense(int device, const uint16_t* d_dense, uint64_t rows, uint64_t cols,
                                  uint64_t ld, uint32_t b_delta, void* stream, macko_dev_matrix** out);

/* GPU compressor from a canonical CSR: replaces macko_from_csr (convert.hpp:12-16)
 * with byte-identical output.  values: nnz fp16 bits, col_idx: nnz u32 (0-based, strictly
 * increasing per row, < cols), row_ptrs: rows+1 u32.  on_device = 0: host arrays (the reference
 * CsrMatrix, matrix.hpp:39-48; uploaded), 1: device pointers.  Non-canonical input -> MACKO_EINVAL
 * (std::invalid_argument).  Synchronises `stream`. */
macko_status macko_dev_from_csr(int device, uint64_t rows, uint64_t cols, uint32_t b_delta, const uint16_t* values,
                                const uint32_t* col_idx, const uint32_t* row_ptrs, uint64_t nnz, int on_device,
                                void* stream, macko_dev_matrix** out);

/* csr_from_dense (convert.hpp:8-10) on the device: the nonzeros (+-0 dropped) of a
 * rows x cols fp16 matrix (leading dimension ld; on_device = 0 host memory, 1 device memory) in
 * row-major order, written to HOST arrays.  Call with values = col_idx = NULL to get row_ptrs
 * (rows+1) and *nnz, then again with nnz-sized values / col_idx.  Synchronous. */
macko_status macko_csr_from_dense(int device, const uint16_t* dense, uint64_t rows, uint64_t cols, uint64_t ld,
                                  int on_device, uint32_t* row_ptrs, uint16_t* values, uint32_t* col_idx,
                                  uint64_t* nnz, void* stream);

/* dense_from_macko (convert.hpp:18-20) on the device: rows x cols fp16, leading dimension ld
 * (elements); on_device = 0: `dense` is host memory (decoded on the device, then copied), 1: device
 * memory.  A decoded column >= cols -> MACKO_EFORMAT (FormatError).  Synchronous. */
macko_status macko_dev_to_dense(const macko_dev_matrix* m, uint16_t* dense, uint64_t ld, int on_device, void* stream);

/* padding_count (convert.hpp:22-23): zero-valued entries among the pad_nnz stored
 * ones (= pad_nnz - nnz of the source).  Synchronous. */
macko_status macko_dev_padding_count(const macko_dev_matrix* m, uint64_t* out, void* stream);

macko_status macko_dev_get_info(const macko_dev_matrix* m, macko_dev_info* out);

/* Device -> host copy of the three arrays in reference layout (sizes from macko_dev_info;
 * any pointer may be NULL to skip it).  Synchronous. */
macko_status macko_dev_download(const macko_dev_matrix* m, uint16_t* values, uint8_t* deltas,
                                uint32_t* row_ptrs, void* stream);

/* y = A*x on the device: fp16 in, fp32 accumulate, one RNE per row, fp16 out.
 * Replaces reference_spmv / warp_spmv.  d_x: cols fp16, d_y: rows fp16.
 * Asynchronous and stream-ordered; concurrent calls on different streams are safe (per-stream
 * workspaces, see macko_dev_matrix).  x must not overlap y. */
macko_status macko_dev_spmv(const macko_dev_matrix* m, const uint16_t* d_x, uint16_t* d_y,
                            void* stream);

/* macko_dev_spmv with launch flags.  MACKO_SPMV_PDL: programmatic dependent launch — the kernel
 * may begin (plan load, first matrix fills) while the previous kernel on the stream drains, and
 * waits for it before reading x.  For chains of SpMVs (decoder stacks); CUDA-graph capturable. */
#define MACKO_SPMV_PDL 1u
/* MACKO_SPMV_PEERS: fused all-gather — every y row is also stored into the peers' y buffers set
 * with macko_dev_set_peers (P2P over NVLink), and each CTA then adds 1 (system scope) to this
 * rank's counter in every peer's flag array; consumers wait with macko_wait_flags. */
#define MACKO_SPMV_PEERS 2u
/* With MACKO_SPMV_PEERS: store into the peer table's y bank 1 (macko_dev_set_peer_bank) instead of
 * bank 0 — double-buffered outputs, so a step may read the previous step's y as its x. */
#define MACKO_SPMV_PEER_BANK1 4u
macko_status macko_dev_spmv_ex(const macko_dev_matrix* m, const uint16_t* d_x, uint16_t* d_y, void* stream,
                               uint32_t flags);

/* Small-batch SpMM Y = A X for 1 <= batch <= 8 vectors (the paper's future work):
 * X row b at d_X + b*ldx (cols fp16), Y row b at d_Y + b*ldy (rows fp16).  The matrix streams
 * from HBM once for the whole batch; X is interleaved per column so one gather fetches every
 * vector's x value.  Column b of Y is bit-identical to macko_dev_spmv(X[b]) (same summation
 * order).  batch = 1 is macko_dev_spmv; batches 3, 5-7 run the next wider kernel with zero
 * vectors.  b_delta = 4 only (MACKO_EINVAL otherwise).  Asynchronous, stream-ordered. */
macko_status macko_dev_spmm(const macko_dev_matrix* m, const uint16_t* d_X, uint64_t ldx, uint16_t* d_Y, uint64_t ldy,
                            uint32_t batch, void* stream);

/* End-to-end call with HOST buffers (what a CPU caller of reference_spmv would bind): x
 * host->device, the SpMV, y device->host, then the stream is synchronised.  Pinned
 * (device-mapped) host buffers are read and written by the kernels directly: a one-CTA kernel
 * pulls x, the SpMV follows as its programmatic dependent and stores every y row into the host
 * buffer as well; pageable buffers take cudaMemcpyAsync both ways.  h_x: cols fp16, h_y: rows
 * fp16.  Device scratch is per stream (thread-safe like macko_dev_spmv). */
macko_status macko_spmv_host(const macko_dev_matrix* m, const uint16_t* h_x, uint16_t* h_y, void* stream);

/* Device-side validate_macko (convert.hpp:25-27): every decoded column < cols.  Synchronous. */
macko_status macko_dev_validate(const macko_dev_matrix* m, void* stream);

macko_status macko_dev_free(macko_dev_matrix* m);

/* Re-plan a matrix for PDL-chained launches (decoder stacks): in a chain, CTA c of an SpMV starts
 * when the previous SpMV releases the c-th SM, up to start_spread_ns after CTA 0, so the plan gives
 * late CTAs proportionally less work.  0 restores the equal split.  y is unchanged (the summation
 * order never depends on the plan).  Synchronises the stream. */
macko_status macko_dev_set_chain_skew(macko_dev_matrix* m, uint32_t start_spread_ns, void* stream);

/* Device blocks of >= 1 MiB released by the library (matrices freed, compressor scratch) are kept
 * per process (up to 4 GiB) and reused by later builds; a release synchronises the device first,
 * as cudaFree does.  This returns every cached block to the driver. */
macko_status macko_release_cached_memory(void);

/* ---- MCKO container (io.cpp write_macko / read_macko are absent) ----------
 * File: 32-byte little-endian header "MCKO" | u16 version=1 | u8 b_val=16 | u8 b_delta | u64 R |
 * u64 C | u64 pad_nnz, then row_pointers ((R+1) x u32), packed_deltas (macko_delta_bytes) and
 * values (u16, macko_values_bytes).  read(write(m)) is bit-identical.  Errors: bad magic /
 * version / truncated section -> MACKO_EIO (IoError); invariant violation after decode ->
 * MACKO_EFORMAT (FormatError). */
macko_status macko_mcko_write(const char* path, uint64_t rows, uint64_t cols, uint32_t b_delta, const uint16_t* values,
                              uint64_t n_values, const uint8_t* deltas, uint64_t n_delta_bytes, const uint32_t* row_ptrs);
/* Header only: rows, cols, pad_nnz, b_delta and the array sizes (values_bytes, delta_bytes) a
 * caller allocates for macko_mcko_read; device = -1. */
macko_status macko_mcko_read_info(const char* path, macko_dev_info* out);
/* read_macko into caller arrays (sizes from macko_mcko_read_info); fully validated on the host. */
macko_status macko_mcko_read(const char* path, uint16_t* values, uint8_t* deltas, uint32_t* row_ptrs);
/* Device matrix -> file (pinned staging, synchronous). */
macko_status macko_mcko_write_dev(const macko_dev_matrix* m, const char* path, void* stream);
/* File -> device matrix without a host copy of the payload: the sections stream through two
 * pinned buffers (disk read overlapped with the H2D copy), then validate_macko runs on the
 * device and the SpMV plan is built.  Synchronises `stream`. */
macko_status macko_mcko_read_dev(int device, const char* path, void* stream, macko_dev_matrix** out);

/* Matrix Market reader: "%%MatrixMarket matrix coordinate real|integer
 * general" -> dense row-major fp16 (1-based indices, entries rounded to fp16 RNE).  Call with
 * dense = NULL to get the dimensions, then with rows*cols uint16 of storage.  Unsupported
 * header / parse errors -> MACKO_EIO; out-of-range index / duplicate coordinate -> MACKO_EFORMAT. */
macko_status macko_mm_read_dense(const char* path, uint64_t* rows, uint64_t* cols, uint16_t* dense);

/* ---- synthetic inputs (counter-hash generator, bit-identical to oracle/macko_oracle.c) ---- */
uint32_t macko_density_threshold(double density);
/* Dense rows [row0, row0+rows) of a conceptual (row0+rows) x cols matrix; element (r, c) is
 * drawn from hash(seed, (row0 + r) * cols + c). */
macko_status macko_gen_dense(int device, uint16_t* d_out, uint64_t rows, uint64_t cols, uint64_t ld,
                             uint64_t row0, uint32_t thr24, uint64_t seed, int int_mode, void* stream);
macko_status macko_gen_vector(int device, uint16_t* d_out, uint64_t n, uint64_t seed, int int_mode,
                              void* stream);

/* ---- row sharding (contiguous equal-row slabs) ---- */
macko_status macko_shard_rows(uint64_t rows, uint32_t n_shards, uint32_t shard, uint64_t* r0,
                              uint64_t* r1);

/* One row-sharded SpMV step over NCCL: rank g of `nccl_comm` (an ncclComm_t)
 * holds slab g = rows [g*R/N, (g+1)*R/N) of an R x C matrix (R = rows_total, equal slabs).
 * d_x (C fp16) is broadcast in place from `root`, the slab's SpMV writes its part of d_y (R fp16)
 * and an in-place all-gather completes d_y on every rank.  Stream-ordered.  NCCL is loaded at run
 * time (libnccl.so.2); MACKO_ENCCL reports its errors. */
macko_status macko_sharded_spmv(const macko_dev_matrix* slab, void* nccl_comm, int root, uint16_t* d_x,
                                uint16_t* d_y, uint64_t rows_total, void* stream);

/* Fused all-gather destinations of a row slab (n <= 8, n = 0 disables): peer_y[p] = peer p's
 * full-y buffer already offset to this slab's first row, peer_flags[p] = this rank's u32 counter
 * in peer p's flag array (device or IPC-mapped pointers; one of them may be this rank's own).
 * After a MACKO_SPMV_PEERS launch every counter has grown by the launch's grid size.  Applies to
 * launches issued after the call: the table travels in the launch parameters (a captured CUDA
 * graph keeps the pointers it was captured with); `stream` is unused. */
macko_status macko_dev_set_peers(macko_dev_matrix* m, uint16_t* const* peer_y, uint32_t* const* peer_flags, uint32_t n,
                                 void* stream);
/* Second y destination set (bank 1, used with MACKO_SPMV_PEER_BANK1): same peer count and flags as
 * macko_dev_set_peers, which resets both banks to its peer_y.  Same timing as macko_dev_set_peers. */
macko_status macko_dev_set_peer_bank(macko_dev_matrix* m, uint32_t bank, uint16_t* const* peer_y, uint32_t n,
                                     void* stream);
/* Stream-ordered wait until d_flags[i] >= target (wrap-around compare) for i < n (n <= 32): the
 * consumer side of MACKO_SPMV_PEERS.  Traps after ~4 s instead of hanging. */
macko_status macko_wait_flags(const uint32_t* d_flags, uint32_t n, uint32_t target, void* stream);
/* CUDA IPC of device buffers between the ranks' processes: the 64-byte handle names the
 * allocation holding d_ptr, *offset is d_ptr's offset in it; macko_ipc_open returns the mapped
 * base (add the offset), macko_ipc_close unmaps that base. */
macko_status macko_ipc_get_handle(const void* d_ptr, uint8_t* handle64, uint64_t* offset);
macko_status macko_ipc_open(const uint8_t* handle64, int device, void** d_base);
macko_status macko_ipc_close(void* d_base);

/* ---- introspection ---- */
typedef struct macko_launch_info {
    uint32_t grid, block, warps, ctas_per_sm, n_split_rows;
    uint32_t x_in_smem; /* x_mode: how x is gathered — 0 texture only, 1 fp16 shared-memory table
                         * only, 6 / 7 / 8 / 10 table + texture split over the element slots
                         * */
    uint64_t n_units, smem_bytes;
    uint32_t reserved0, reserved;
} macko_launch_info;
macko_status macko_dev_launch_info(const macko_dev_matrix* m, macko_launch_info* out);
/* Re-plan the SpMV launch: x_mode (-1 automatic, else as above) and a cap on CTAs (k > 0: use
 * k/4 of the persistent CTAs; 0 automatic).  Results are identical for every setting (the
 * summation order does not depend on the plan); exposed for tuning and for the grid-independence
 * tests.  Synchronous; not concurrent with SpMVs of the handle. */
macko_status macko_dev_configure(macko_dev_matrix* m, int x_mode, int ctas_per_sm, void* stream);
/* The SpMV work plan (spmv.cuh): launch_info.warps 48-byte warp records and n_split_rows 16-byte
 * split-row records, copied to host buffers (NULL skips).  Introspection for tests.  Synchronous. */
macko_status macko_dev_plan_records(const macko_dev_matrix* m, void* recs, uint64_t recs_bytes, void* splits,
                                    uint64_t splits_bytes, void* stream);
/* Number of kernels this library has launched in the process (for bench gpu_launches). */
uint64_t macko_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* MACKO_CUDA_H */
