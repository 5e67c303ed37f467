// llm_ops.cuh — the per-token elementwise / normalisation steps of the Llama decode, as device
// functions shared by libmacko_llm.so's stand-alone kernels (llm.cu) and the SpMV's last-CTA
// epilogue (spmv.cu), so a fused step produces exactly the stand-alone kernel's bits.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace llmops {

__device__ __forceinline__ float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }
__device__ __forceinline__ uint16_t f2h(float f) { return __half_as_ushort(__float2half_rn(f)); }

template <int kThreads>
__device__ __forceinline__ float block_sum(float v, float* red) {
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < kThreads / 32 ? red[l] : 0.0f;
        for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (l == 0) red[0] = v;
    }
    __syncthreads();
    const float r = red[0];
    __syncthreads();
    return r;
}

// One CTA of 1024 threads: h += delta (fp16 residual stream; delta may be null); out = h / rms(h) * weight
__device__ __forceinline__ void add_rmsnorm_block(uint16_t* h, const uint16_t* delta, const uint16_t* weight, uint16_t* out,
                                                  uint32_t n, float eps, float* red) {
    float ss = 0.0f;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        float v = h2f(h[i]);
        if (delta) {
            v = h2f(f2h(v + h2f(delta[i])));
            h[i] = f2h(v);
        }
        ss += v * v;
    }
    const float inv = rsqrtf(block_sum<1024>(ss, red) / (float)n + eps);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = f2h(h2f(h[i]) * inv * h2f(weight[i]));
}

// gu = [gate; up] (2 * inter): out[i] = silu(gate[i]) * up[i] for i = first, first + stride, ...
__device__ __forceinline__ void silu_mul_range(const uint16_t* gu, uint16_t* out, uint32_t inter, uint32_t first,
                                               uint32_t stride) {
    for (uint32_t i = first; i < inter; i += stride) {
        const float g = h2f(gu[i]), u = h2f(gu[inter + i]);
        out[i] = f2h(g / (1.0f + __expf(-g)) * u);
    }
}

}  // namespace llmops
