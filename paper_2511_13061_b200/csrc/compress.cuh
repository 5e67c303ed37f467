// compress.cuh — launchers of the dense -> MACKO compressor kernels (compress.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mk {

cudaError_t launch_count_rows(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, uint32_t bits,
                              uint32_t* counts, int32_t* lastcol, int sms, cudaStream_t s);
cudaError_t launch_scan_counts(const uint32_t* counts, uint32_t rows, uint32_t* row_ptrs, unsigned long long* total,
                               cudaStream_t s);
cudaError_t launch_emit_rows(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, uint32_t bits,
                             const uint32_t* row_ptrs, const int32_t* lastcol, uint16_t* values, uint32_t* delta_words,
                             int sms, cudaStream_t s);

// generate.cu
cudaError_t launch_gen_dense(uint16_t* out, uint64_t rows, uint64_t cols, uint64_t ld, uint64_t row0, uint32_t thr24,
                             uint64_t seed, int int_mode, int sms, cudaStream_t s);
cudaError_t launch_gen_vector(uint16_t* out, uint64_t n, uint64_t seed, int int_mode, cudaStream_t s);
// validate.cu-style check inside generate.cu: *err |= 1 on a column overflow, 2 on a -0 pad.
cudaError_t launch_validate(const uint16_t* values, const uint8_t* deltas, const uint32_t* row_ptrs, uint32_t rows,
                            uint32_t cols, uint32_t bits, uint32_t* err, int sms, cudaStream_t s);

}  // namespace mk

namespace mk {
// convert.cu: macko_from_csr / dense_from_macko / padding_count on the device
cudaError_t launch_csr_count(const uint32_t* rp, const uint32_t* ci, uint32_t rows, uint32_t cols, uint32_t bits,
                             uint32_t* counts, uint32_t* err, int sms, cudaStream_t s);
cudaError_t launch_csr_emit(const uint32_t* rp, const uint32_t* ci, const uint16_t* cv, uint32_t rows, uint32_t bits,
                            const uint32_t* mrp, uint16_t* values, uint8_t* codes, int sms, cudaStream_t s);
cudaError_t launch_pack_codes(const uint8_t* codes, uint64_t n, uint32_t bits, uint8_t* out, uint64_t out_bytes,
                              int sms, cudaStream_t s);
cudaError_t launch_to_dense(const uint16_t* values, const uint8_t* deltas, const uint32_t* rp, uint32_t rows,
                            uint32_t cols, uint32_t bits, uint16_t* dense, uint64_t ld, uint32_t* err, int sms,
                            cudaStream_t s);
cudaError_t launch_padding_count(const uint16_t* values, uint64_t n, unsigned long long* count, int sms,
                                 cudaStream_t s);
cudaError_t launch_dense_nnz(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, uint32_t* counts,
                             int sms, cudaStream_t s);
cudaError_t launch_dense_csr_emit(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, const uint32_t* rp,
                                  uint16_t* vals, uint32_t* ci, int sms, cudaStream_t s);
}  // namespace mk
