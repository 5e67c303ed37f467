// generate.cu — synthetic inputs on the device and the device-side validate_macko.
//
// The generator is bit-identical to oracle/macko_oracle.c (mo_gen_value / mo_gen_vector): the
// reference's gen_random leaves RNG and magnitude distribution unspecified,
// so benchmark matrices are produced directly in HBM by a counter hash instead of being copied
// from the host.
#include "common.cuh"
#include "compress.cuh"

#include <algorithm>

namespace mk {

namespace {

__global__ void gen_dense_kernel(uint16_t* out, uint64_t rows, uint64_t cols, uint64_t ld, uint64_t row0,
                                 uint32_t thr24, uint64_t seed, int int_mode, bool vec_ok) {
    const uint64_t groups_per_row = (cols + 7) / 8;
    const uint64_t n = rows * groups_per_row;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n; g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = g / groups_per_row, c = (g - r * groups_per_row) * 8;
        const uint64_t base = (row0 + r) * cols + c;
        uint16_t* dst = out + r * ld + c;
        if (vec_ok && c + 8 <= cols) {
            uint32_t w[4];
#pragma unroll
            for (int m = 0; m < 4; ++m)
                w[m] = (uint32_t)gen_value(seed, base + 2 * m, thr24, int_mode) |
                       ((uint32_t)gen_value(seed, base + 2 * m + 1, thr24, int_mode) << 16);
            *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
            for (uint64_t k = 0; k < 8 && c + k < cols; ++k) dst[k] = gen_value(seed, base + k, thr24, int_mode);
        }
    }
}

__global__ void gen_vector_kernel(uint16_t* out, uint64_t n, uint64_t seed, int int_mode) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = gen_vector_value(seed, i, int_mode);
}

// validate_macko (convert.hpp:25-27): warp per row; the last decoded column
// (sum of deltas - 1) must be < cols; padding (zero) values must be +0.
__global__ void validate_kernel(const uint16_t* values, const uint8_t* deltas, const uint32_t* row_ptrs, uint32_t rows,
                                uint32_t cols, uint32_t bits, uint32_t* err) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * (blockDim.x / 32);
    const uint32_t per = 8u / bits, mask = bits == 8 ? 0xFFu : ((1u << bits) - 1u);
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += nw) {
        const uint32_t s = row_ptrs[r], e = row_ptrs[r + 1];
        if (e < s) {
            if (lane == 0) atomicOr(err, 4u);
            continue;
        }
        uint64_t sum = 0;
        uint32_t bad = 0;
        for (uint32_t i = s + lane; i < e; i += 32) {
            sum += ((deltas[i / per] >> ((i % per) * bits)) & mask) + 1u;
            bad |= values[i] == 0x8000u;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            sum += __shfl_xor_sync(kFull, sum, off);
            bad |= __shfl_xor_sync(kFull, bad, off);
        }
        if (lane == 0) {
            if (sum > cols) atomicOr(err, 1u);
            if (bad) atomicOr(err, 2u);
        }
    }
}

}  // namespace

cudaError_t launch_gen_dense(uint16_t* out, uint64_t rows, uint64_t cols, uint64_t ld, uint64_t row0, uint32_t thr24,
                             uint64_t seed, int int_mode, int sms, cudaStream_t s) {
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(out) | (ld * 2)) & 15u) == 0;
    const uint64_t n = rows * ((cols + 7) / 8);
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 16);
    if (grid > 0) gen_dense_kernel<<<grid, 256, 0, s>>>(out, rows, cols, ld, row0, thr24, seed, int_mode, vec_ok);
    return cudaGetLastError();
}

cudaError_t launch_gen_vector(uint16_t* out, uint64_t n, uint64_t seed, int int_mode, cudaStream_t s) {
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, 1024);
    if (grid > 0) gen_vector_kernel<<<grid, 256, 0, s>>>(out, n, seed, int_mode);
    return cudaGetLastError();
}

cudaError_t launch_validate(const uint16_t* values, const uint8_t* deltas, const uint32_t* row_ptrs, uint32_t rows,
                            uint32_t cols, uint32_t bits, uint32_t* err, int sms, cudaStream_t s) {
    const int grid = (int)std::min<uint64_t>(((uint64_t)rows + 7) / 8, (uint64_t)sms * 8);
    if (grid > 0) validate_kernel<<<grid, 256, 0, s>>>(values, deltas, row_ptrs, rows, cols, bits, err);
    return cudaGetLastError();
}

}  // namespace mk
