// llm.cu — libmacko_llm.so: the small per-token kernels of a Llama-style batch-1 decode step, the
// caller of the MACKO path in the paper's end-to-end measurement (Llama2-7B,
// 100 generated tokens, MACKO linears vs dense cuBLAS).  Not part of the SpMV boundary; the
// linears themselves are libmacko_cuda.so SpMVs (or cuBLAS GEMVs for the dense baseline).
//
// Every kernel reads the decode position / token id from device memory, so one decode step is a
// fixed sequence of launches that a CUDA graph replays token after token.  All of them are
// programmatic dependent launches (PDL): each lets the next kernel launch at its start and waits for
// its predecessor (griddepcontrol.wait) before touching data, so the SpMVs' prologues (plan record,
// first matrix fills) and these kernels' launches overlap the previous kernel's tail.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "../../include/macko_llm.h"
#include "llm_ops.cuh"

namespace {

using llmops::block_sum;
using llmops::f2h;
using llmops::h2f;

__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// h += delta (fp16 residual stream, as the fp16 model keeps it); out = h / rms(h) * weight
__global__ void __launch_bounds__(1024) add_rmsnorm_kernel(uint16_t* h, const uint16_t* delta, const uint16_t* weight,
                                                           uint16_t* out, uint32_t n, float eps) {
    __shared__ float red[32];
    pdl_enter();
    llmops::add_rmsnorm_block(h, delta, weight, out, n, eps, red);
}

// Rotary embedding + KV append + attention of one query, fused: a CTA of 8 warps per head rotates
// its head's q and k at position *pos (rotate-half convention, base theta; the rotation partner
// d +- head_dim/2 is in the same head), appends k / v to cache row *pos, then attends over rows
// [0, *pos] (fp32 scores and softmax).  Scores: one thread per position, its K row in 16-byte
// loads; output: warp w takes positions t = w (mod 8), lane l owns dims [l D, l D + D), D =
// head_dim / 32, one D-element vector load per row, partial sums combined in shared memory.
// qkv = [q; k; v] (3 * heads * head_dim).
constexpr int kAttnWarps = 8;

template <int kHeadDim>
__global__ void __launch_bounds__(kAttnWarps * 32) rope_attention_kernel(const uint16_t* qkv, const int32_t* pos,
                                                                         uint16_t* k_cache, uint16_t* v_cache,
                                                                         uint16_t* out, uint32_t heads,
                                                                         uint32_t max_len, float theta) {
    pdl_enter();
    constexpr uint32_t D = kHeadDim / 32, half = kHeadDim / 2;
    extern __shared__ float sm[];  // scores[max_len]
    __shared__ float part[kAttnWarps][kHeadDim];
    __shared__ float qs[kHeadDim];
    __shared__ float red[32];
    float* sc = sm;
    const uint32_t h = blockIdx.x, H = heads * kHeadDim;
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    const int32_t p = *pos, n = p + 1;
    for (uint32_t d = threadIdx.x; d < kHeadDim; d += blockDim.x) {
        const uint32_t i = h * kHeadDim + d, j = d % half;
        const float inv_freq = powf(theta, -2.0f * (float)j / (float)kHeadDim);
        float sn, cs;
        sincosf((float)p * inv_freq, &sn, &cs);
        const uint32_t partner = d < half ? i + half : i - half;
        const float sign = d < half ? -1.0f : 1.0f;  // rotate_half: [-x2, x1]
        qs[d] = h2f(f2h(h2f(qkv[i]) * cs + sign * h2f(qkv[partner]) * sn));
        k_cache[(size_t)p * H + i] = f2h(h2f(qkv[H + i]) * cs + sign * h2f(qkv[H + partner]) * sn);
        v_cache[(size_t)p * H + i] = qkv[2 * H + i];
    }
    __syncthreads();
    const float scale = rsqrtf((float)kHeadDim);
    for (int32_t t = threadIdx.x; t < n; t += blockDim.x) {
        const uint4* kr = reinterpret_cast<const uint4*>(k_cache + (size_t)t * H + h * kHeadDim);
        uint4 kv[kHeadDim / 8];
#pragma unroll
        for (uint32_t v = 0; v < kHeadDim / 8; ++v) kv[v] = kr[v];
        float s = 0.0f;
#pragma unroll
        for (uint32_t v = 0; v < kHeadDim / 8; ++v) {
            const uint32_t wds[4] = {kv[v].x, kv[v].y, kv[v].z, kv[v].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&wds[k]));
                s += qs[8 * v + 2 * k] * f.x + qs[8 * v + 2 * k + 1] * f.y;
            }
        }
        sc[t] = s * scale;
    }
    __syncthreads();
    float mx = -INFINITY;
    for (int32_t t = threadIdx.x; t < n; t += blockDim.x) mx = fmaxf(mx, sc[t]);
    for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (l == 0) red[w] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int i = 1; i < kAttnWarps; ++i) mx = fmaxf(mx, red[i]);
    __syncthreads();
    float sum = 0.0f;
    for (int32_t t = threadIdx.x; t < n; t += blockDim.x) {
        const float e = __expf(sc[t] - mx);
        sc[t] = e;
        sum += e;
    }
    sum = block_sum<kAttnWarps * 32>(sum, red);  // (its barriers also publish sc)
    float acc[D];
#pragma unroll
    for (uint32_t i = 0; i < D; ++i) acc[i] = 0.0f;
#pragma unroll 4
    for (int32_t t = w; t < n; t += kAttnWarps) {
        const float pt = sc[t];
        const uint16_t* vr = v_cache + (size_t)t * H + h * kHeadDim + l * D;
        uint16_t vv[D];
        if constexpr (D == 4) {
            const uint2 q2 = *reinterpret_cast<const uint2*>(vr);
            vv[0] = (uint16_t)q2.x; vv[1] = (uint16_t)(q2.x >> 16); vv[2] = (uint16_t)q2.y; vv[3] = (uint16_t)(q2.y >> 16);
        } else {
#pragma unroll
            for (uint32_t i = 0; i < D; ++i) vv[i] = vr[i];
        }
#pragma unroll
        for (uint32_t i = 0; i < D; ++i) acc[i] += pt * h2f(vv[i]);
    }
#pragma unroll
    for (uint32_t i = 0; i < D; ++i) part[w][l * D + i] = acc[i];
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < kHeadDim; d += blockDim.x) {
        float o = 0.0f;
#pragma unroll
        for (int i = 0; i < kAttnWarps; ++i) o += part[i][d];
        out[h * kHeadDim + d] = f2h(o / sum);
    }
}

// gu = [gate; up] (2 * inter): out = silu(gate) * up
__global__ void silu_mul_kernel(const uint16_t* gu, uint16_t* out, uint32_t inter) {
    pdl_enter();
    llmops::silu_mul_range(gu, out, inter, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

__global__ void embed_kernel(const uint16_t* table, const int32_t* token, uint16_t* h, uint32_t hidden) {
    pdl_enter();
    const int32_t t = *token;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < hidden; i += gridDim.x * blockDim.x)
        h[i] = table[(size_t)t * hidden + i];
}

// Greedy sampling: token = argmax(logits) (lowest index on ties), then *pos += 1.
__global__ void __launch_bounds__(1024) argmax_kernel(const uint16_t* logits, uint32_t n, int32_t* token, int32_t* pos,
                                                      int32_t* history, uint32_t history_len) {
    pdl_enter();
    __shared__ float bv[32];
    __shared__ int32_t bi[32];
    float best = -INFINITY;
    int32_t idx = 0x7FFFFFFF;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const float v = h2f(logits[i]);
        if (v > best || (v == best && (int32_t)i < idx)) {
            best = v;
            idx = (int32_t)i;
        }
    }
    for (int off = 16; off >= 1; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int32_t oi = __shfl_xor_sync(0xffffffffu, idx, off);
        if (ov > best || (ov == best && oi < idx)) {
            best = ov;
            idx = oi;
        }
    }
    if (threadIdx.x % 32 == 0) {
        bv[threadIdx.x / 32] = best;
        bi[threadIdx.x / 32] = idx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t w = 1; w < blockDim.x / 32; ++w)
            if (bv[w] > best || (bv[w] == best && bi[w] < idx)) {
                best = bv[w];
                idx = bi[w];
            }
        const int32_t p = *pos;
        *token = idx;
        if (history && (uint32_t)p < history_len) history[p] = idx;
        *pos = p + 1;
    }
}

template <typename... KArgs, typename... Args>
int launch(void (*k)(KArgs...), int grid, int block, size_t smem, void* stream, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, k, args...);
}

int grid_for(uint32_t n, int threads) { return (int)((n + threads - 1) / threads < 1024 ? (n + threads - 1) / threads : 1024); }

}  // namespace

extern "C" {

int macko_llm_add_rmsnorm(uint16_t* h, const uint16_t* delta, const uint16_t* weight, uint16_t* out, uint32_t n,
                          float eps, void* stream) {
    return launch(add_rmsnorm_kernel, 1, 1024, 0, stream, h, delta, weight, out, n, eps);
}

int macko_llm_rope_attention(const uint16_t* qkv, const int32_t* pos, uint16_t* k_cache, uint16_t* v_cache,
                             uint16_t* out, uint32_t heads, uint32_t head_dim, uint32_t max_len, float theta,
                             void* stream) {
    const size_t smem = max_len * sizeof(float);
    if (head_dim == 128)
        return launch(rope_attention_kernel<128>, (int)heads, kAttnWarps * 32, smem, stream, qkv, pos, k_cache, v_cache,
                      out, heads, max_len, theta);
    if (head_dim == 64)
        return launch(rope_attention_kernel<64>, (int)heads, kAttnWarps * 32, smem, stream, qkv, pos, k_cache, v_cache,
                      out, heads, max_len, theta);
    return (int)cudaErrorInvalidValue;  // head_dim 64 or 128 (Llama)
}

int macko_llm_silu_mul(const uint16_t* gu, uint16_t* out, uint32_t inter, void* stream) {
    return launch(silu_mul_kernel, grid_for(inter, 256), 256, 0, stream, gu, out, inter);
}

int macko_llm_embed(const uint16_t* table, const int32_t* token, uint16_t* h, uint32_t hidden, void* stream) {
    return launch(embed_kernel, grid_for(hidden, 256), 256, 0, stream, table, token, h, hidden);
}

int macko_llm_argmax(const uint16_t* logits, uint32_t n, int32_t* token, int32_t* pos, int32_t* history,
                     uint32_t history_len, void* stream) {
    return launch(argmax_kernel, 1, 1024, 0, stream, logits, n, token, pos, history, history_len);
}

}  // extern "C"
