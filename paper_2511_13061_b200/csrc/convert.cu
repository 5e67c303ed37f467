// convert.cu — the rest of the reference's conversion surface on the device (convert.hpp:8-27):
// macko_from_csr (the greedy encoder fed by a canonical CSR instead of a dense matrix),
// dense_from_macko (lossless decode) and padding_count.  All row-parallel: a row's encoding
// depends only on its own nonzeros (convert.hpp:12-16, virtual column -1 per row).
//
//   csr_count_kernel : warp per row; entries = nnz_r + sum over consecutive nonzeros p < c of
//                      floor((c - p - 1) / 2^b) forced pads (SURVEY.md A.4 closed form; p = -1 for
//                      the first); flags unsorted / out-of-range columns.
//   scan_counts      : (compress.cu) row pointers + pad_nnz.
//   csr_emit_kernel  : warp per row; a lane-prefix of the pad counts places each nonzero after its
//                      pads; values and one byte codeword per element (temp), then
//   pack_codes_kernel: packs 8 / b codewords per byte, LSB-first (bitpack.cpp:18-32).
//   to_dense_kernel  : warp per row, 32 elements per iteration, warp scan of the deltas -> columns.
//   padding_kernel   : zero-valued entries in [0, pad_nnz).
#include "common.cuh"
#include "compress.cuh"

#include <algorithm>

namespace mk {

namespace {

__device__ __forceinline__ uint32_t warp_incl_u32(uint32_t v, int lane) {
#pragma unroll
    for (int off = 1; off < kWarp; off <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, v, off);
        if (lane >= off) v += t;
    }
    return v;
}

// err bits: 1 column >= cols, 2 columns not strictly increasing, 4 row pointers not monotone
__global__ void csr_count_kernel(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci, uint32_t rows,
                                 uint32_t cols, uint32_t bits, uint32_t* __restrict__ counts, uint32_t* err) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * (blockDim.x / 32);
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += nw) {
        const uint32_t s = rp[r], e = rp[r + 1];
        if (e < s) {
            if (lane == 0) {
                atomicOr(err, 4u);
                counts[r] = 0;
            }
            continue;
        }
        uint32_t pads = 0, bad = 0;
        for (uint32_t k = s + lane; k < e; k += 32) {
            const uint32_t c = ci[k];
            const int64_t p = k > s ? (int64_t)ci[k - 1] : -1;
            bad |= c >= cols ? 1u : 0u;
            bad |= (int64_t)c <= p ? 2u : 0u;
            if ((int64_t)c > p) pads += (uint32_t)(((int64_t)c - p - 1) >> bits);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            pads += __shfl_xor_sync(kFull, pads, off);
            bad |= __shfl_xor_sync(kFull, bad, off);
        }
        if (lane == 0) {
            counts[r] = (e - s) + pads;
            if (bad) atomicOr(err, bad);
        }
    }
}

// Values and one codeword byte per element: each lane takes 32 consecutive nonzeros per pass,
// the lane-inclusive prefix of (pads + 1) gives every nonzero's element offset.
__global__ void csr_emit_kernel(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                                const uint16_t* __restrict__ cv, uint32_t rows, uint32_t bits,
                                const uint32_t* __restrict__ mrp, uint16_t* __restrict__ values,
                                uint8_t* __restrict__ codes) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * (blockDim.x / 32);
    const uint32_t maxd = 1u << bits;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += nw) {
        const uint32_t s = rp[r], e = rp[r + 1];
        uint32_t at = mrp[r];  // element offset of the row's next entry
        for (uint32_t k0 = s; k0 < e; k0 += 32) {
            const uint32_t k = k0 + lane;
            uint32_t n_entries = 0, g = 0, c = 0;
            int64_t p = -1;
            if (k < e) {
                c = ci[k];
                p = k > s ? (int64_t)ci[k - 1] : -1;
                g = (uint32_t)(((int64_t)c - p - 1) >> bits);  // forced pads before this nonzero
                n_entries = g + 1;
            }
            const uint32_t incl = warp_incl_u32(n_entries, lane);
            const uint32_t first = at + incl - n_entries;
            if (k < e) {
                for (uint32_t q = 0; q < g; ++q) {  // pads at p + maxd, p + 2 maxd, ...
                    values[first + q] = 0;
                    codes[first + q] = (uint8_t)(maxd - 1u);
                }
                values[first + g] = cv[k];
                codes[first + g] = (uint8_t)((uint32_t)((int64_t)c - p - 1) - g * maxd);  // delta - 1
            }
            at += __shfl_sync(kFull, incl, 31);
        }
    }
}

// 8 / bits codewords per byte, LSB-first; bytes past pad_nnz are zero (16-byte tail).
__global__ void pack_codes_kernel(const uint8_t* __restrict__ codes, uint64_t n, uint32_t bits,
                                  uint8_t* __restrict__ out, uint64_t out_bytes) {
    const uint32_t per = 8u / bits;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < out_bytes;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t byte = 0;
        for (uint32_t j = 0; j < per; ++j) {
            const uint64_t e = i * per + j;
            if (e < n) byte |= (uint32_t)codes[e] << (j * bits);
        }
        out[i] = (uint8_t)byte;
    }
}

// dense_from_macko: dense rows are zeroed by the caller; warp per row, 32 elements per pass.
// err |= 1 when a decoded column reaches cols (corruption).
__global__ void to_dense_kernel(const uint16_t* __restrict__ values, const uint8_t* __restrict__ deltas,
                                const uint32_t* __restrict__ rp, uint32_t rows, uint32_t cols, uint32_t bits,
                                uint16_t* __restrict__ dense, uint64_t ld, uint32_t* err) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * (blockDim.x / 32);
    const uint32_t per = 8u / bits, mask = bits == 8 ? 0xFFu : ((1u << bits) - 1u);
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += nw) {
        const uint32_t s = rp[r], e = rp[r + 1];
        int64_t col = -1;
        for (uint32_t i0 = s; i0 < e; i0 += 32) {
            const uint32_t i = i0 + lane;
            const uint32_t d = i < e ? ((deltas[i / per] >> ((i % per) * bits)) & mask) + 1u : 0u;
            const uint32_t incl = warp_incl_u32(d, lane);
            const int64_t c = col + incl;
            if (i < e) {
                if (c >= (int64_t)cols) {
                    atomicOr(err, 1u);
                } else {
                    dense[(uint64_t)r * ld + (uint64_t)c] = values[i];
                }
            }
            col += __shfl_sync(kFull, incl, 31);
        }
    }
}

__global__ void padding_kernel(const uint16_t* __restrict__ values, uint64_t n, unsigned long long* count) {
    uint32_t mine = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        mine += (values[i] & 0x7FFFu) == 0;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) mine += __shfl_xor_sync(kFull, mine, off);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(count, (unsigned long long)mine);
}

// csr_from_dense (convert.hpp:8-10): nonzeros (+-0 dropped) in row-major order.
// Warp per row, 32 columns per pass: ballot of the nonzero flags, popc ranks.
__global__ void dense_nnz_kernel(const uint16_t* __restrict__ dense, uint64_t ld, uint32_t rows, uint32_t cols,
                                 uint32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * (blockDim.x / 32);
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += nw) {
        const uint16_t* row = dense + (uint64_t)r * ld;
        uint32_t n = 0;
        for (uint32_t c = lane; c < cols; c += 32) n += (row[c] & 0x7FFFu) != 0;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) n += __shfl_xor_sync(kFull, n, off);
        if (lane == 0) counts[r] = n;
    }
}

__global__ void dense_csr_emit_kernel(const uint16_t* __restrict__ dense, uint64_t ld, uint32_t rows, uint32_t cols,
                                      const uint32_t* __restrict__ rp, uint16_t* __restrict__ vals,
                                      uint32_t* __restrict__ ci) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * (blockDim.x / 32);
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += nw) {
        const uint16_t* row = dense + (uint64_t)r * ld;
        uint32_t at = rp[r];
        for (uint32_t c0 = 0; c0 < cols; c0 += 32) {
            const uint32_t c = c0 + lane;
            const uint16_t v = c < cols ? row[c] : 0;
            const bool nz = (v & 0x7FFFu) != 0;
            const uint32_t b = __ballot_sync(kFull, nz);
            if (nz) {
                const uint32_t k = at + __popc(b & ((1u << lane) - 1u));
                vals[k] = v;
                ci[k] = c;
            }
            at += __popc(b);
        }
    }
}

int row_grid(uint32_t rows, int sms) { return (int)std::max<uint64_t>(1, std::min<uint64_t>((rows + 7) / 8, (uint64_t)sms * 8)); }

}  // namespace

cudaError_t launch_csr_count(const uint32_t* rp, const uint32_t* ci, uint32_t rows, uint32_t cols, uint32_t bits,
                             uint32_t* counts, uint32_t* err, int sms, cudaStream_t s) {
    if (rows) csr_count_kernel<<<row_grid(rows, sms), 256, 0, s>>>(rp, ci, rows, cols, bits, counts, err);
    return cudaGetLastError();
}

cudaError_t launch_csr_emit(const uint32_t* rp, const uint32_t* ci, const uint16_t* cv, uint32_t rows, uint32_t bits,
                            const uint32_t* mrp, uint16_t* values, uint8_t* codes, int sms, cudaStream_t s) {
    if (rows) csr_emit_kernel<<<row_grid(rows, sms), 256, 0, s>>>(rp, ci, cv, rows, bits, mrp, values, codes);
    return cudaGetLastError();
}

cudaError_t launch_pack_codes(const uint8_t* codes, uint64_t n, uint32_t bits, uint8_t* out, uint64_t out_bytes,
                              int sms, cudaStream_t s) {
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((out_bytes + 255) / 256, (uint64_t)sms * 16));
    if (out_bytes) pack_codes_kernel<<<grid, 256, 0, s>>>(codes, n, bits, out, out_bytes);
    return cudaGetLastError();
}

cudaError_t launch_to_dense(const uint16_t* values, const uint8_t* deltas, const uint32_t* rp, uint32_t rows,
                            uint32_t cols, uint32_t bits, uint16_t* dense, uint64_t ld, uint32_t* err, int sms,
                            cudaStream_t s) {
    if (rows) to_dense_kernel<<<row_grid(rows, sms), 256, 0, s>>>(values, deltas, rp, rows, cols, bits, dense, ld, err);
    return cudaGetLastError();
}

cudaError_t launch_dense_nnz(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, uint32_t* counts,
                             int sms, cudaStream_t s) {
    if (rows) dense_nnz_kernel<<<row_grid(rows, sms), 256, 0, s>>>(dense, ld, rows, cols, counts);
    return cudaGetLastError();
}

cudaError_t launch_dense_csr_emit(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, const uint32_t* rp,
                                  uint16_t* vals, uint32_t* ci, int sms, cudaStream_t s) {
    if (rows) dense_csr_emit_kernel<<<row_grid(rows, sms), 256, 0, s>>>(dense, ld, rows, cols, rp, vals, ci);
    return cudaGetLastError();
}

cudaError_t launch_padding_count(const uint16_t* values, uint64_t n, unsigned long long* count, int sms,
                                 cudaStream_t s) {
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 8));
    if (n) padding_kernel<<<grid, 256, 0, s>>>(values, n, count);
    return cudaGetLastError();
}

}  // namespace mk
