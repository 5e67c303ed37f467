// Microbenchmark: does a TMA bulk-copy (cp.async.bulk global->smem) stream compete with
// random LDS gathers for the L1/shared data pipe on sm_100a, and how does an LDG.128 stream
// compare?  Each kernel runs 1 CTA/SM x 16 warps; warps 0..14 gather, warp 15 streams.
// Prints gathers/clk/SM and streamed bytes/clk/SM.  See profiles/r01_pipes.md.
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int kGatherIters = 4096;
constexpr int kStreamBytes = 48 * 1024;  // per TMA transfer

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float gather_loop(const uint16_t* xs, uint32_t seed) {
    float acc = 0.f;
    uint32_t h = seed * 2654435761u;
#pragma unroll 8
    for (int i = 0; i < kGatherIters; ++i) {
        h = h * 1664525u + 1013904223u;
        const uint16_t v = xs[(h >> 16) & 8191];
        acc += __half2float(__ushort_as_half(v));
    }
    return acc;
}

// mode 0: gathers only; 1: gathers + TMA stream; 2: gathers + LDG.128 stream; 3: TMA only; 4: LDG only
__global__ void __launch_bounds__(512, 1) k(const uint4* __restrict__ g, size_t g_elems, float* out, int mode,
                                             unsigned long long* bytes_out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint16_t* xs = reinterpret_cast<uint16_t*>(sm);                 // 16 KB gather table
    uint8_t* buf = sm + 16384;                                        // TMA landing zone
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) xs[i] = (uint16_t)(i * 7);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float acc = 0.f;
    unsigned long long streamed = 0;
    const bool gathers = (mode <= 2) && warp < 15;
    const bool streamer = warp == 15;
    if (gathers) acc = gather_loop(xs, threadIdx.x + blockIdx.x * 977);
    if (streamer && (mode == 1 || mode == 3)) {
        // TMA: one elected lane keeps a 48 KB bulk copy in flight per round
        uint32_t phase = 0;
        const size_t per_cta = g_elems / gridDim.x;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(g + per_cta * blockIdx.x);
        const int rounds = 64;
        for (int r = 0; r < rounds; ++r) {
            if (lane == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                             "r"(kStreamBytes));
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(buf)),
                    "l"(src + (size_t)(r % 16) * kStreamBytes), "r"(kStreamBytes), "r"(smem_u32(&bar))
                    : "memory");
                uint32_t done = 0;
                while (!done) {
                    asm volatile(
                        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                        : "=r"(done)
                        : "r"(smem_u32(&bar)), "r"(phase));
                }
                phase ^= 1;
            }
            __syncwarp();
            streamed += kStreamBytes;
        }
    }
    if (streamer && (mode == 2 || mode == 4)) {
        const size_t per_cta = g_elems / gridDim.x;
        const uint4* src = g + per_cta * blockIdx.x;
        uint32_t x = 0;
        const int n = 64 * kStreamBytes / 16 / 32;
        for (int i = 0; i < n; i += 4) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldg(src + ((size_t)(i + u) * 32 + lane) % per_cta);
#pragma unroll
            for (int u = 0; u < 4; ++u) x ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
        acc += (float)x;
        streamed += (unsigned long long)n * 512;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 32 * 15) atomicAdd(bytes_out, streamed);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t g_elems = (size_t)1 << 26;  // 1 GiB of uint4
    uint4* g;
    float* out;
    unsigned long long* bytes;
    cudaMalloc(&g, g_elems * 16);
    cudaMemset(g, 1, g_elems * 16);
    cudaMalloc(&out, sms * 512 * 4);
    cudaMalloc(&bytes, 8);
    const int smem = 16384 + kStreamBytes;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const char* names[] = {"gathers", "gathers+TMA", "gathers+LDG", "TMA only", "LDG only"};
    for (int mode = 0; mode < 5; ++mode) {
        k<<<sms, 512, smem>>>(g, g_elems, out, mode, bytes);
        cudaMemset(bytes, 0, 8);
        cudaEventRecord(a);
        k<<<sms, 512, smem>>>(g, g_elems, out, mode, bytes);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long hb = 0;
        cudaMemcpy(&hb, bytes, 8, cudaMemcpyDeviceToHost);
        const double cyc = ms * 1e-3 * clk_khz * 1e3;
        const double gathers = (mode <= 2) ? 15.0 * kGatherIters : 0;  // warp-gathers per SM
        printf("%-14s %8.3f ms  warp-gathers/clk/SM %.3f  stream B/clk/SM %.1f  (err %s)\n", names[mode], ms,
               gathers / cyc, hb / (double)sms / cyc, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
