// Microbenchmark: stream a large array through the TEX pipe (tex1Dfetch<uint4>, one 16-B texel
// per lane, 512 B per warp step) with cp.async.bulk.prefetch.L2 issued ahead, optionally while
// other warps run LDS gathers.  Reports achieved HBM GB/s and gathers/clk.
// mode 0: TEX stream only (32 warps); 1: TEX stream, no L2 prefetch; 2: LDG.128 stream (LSU);
// 3: TEX stream (24 warps) + LDS gathers (8 warps)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kWarps = 32;
constexpr uint32_t kPf = 8192;  // prefetch distance (bytes) per warp

__global__ void __launch_bounds__(1024, 1) k(cudaTextureObject_t t, const uint4* __restrict__ g, size_t n16,
                                              uint32_t* out, int mode) {
    __shared__ uint16_t xs[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) xs[i] = (uint16_t)i;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool gatherer = mode == 3 && warp >= 24;
    const int streamers = mode == 3 ? 24 : kWarps;
    uint32_t acc = 0;
    if (gatherer) {
        uint32_t h = 777u * threadIdx.x + blockIdx.x;
        for (int i = 0; i < 8192; ++i) {
            h = h * 1664525u + 1013904223u;
            acc += xs[((h >> 8) + 16 * lane) & 8191];
        }
    } else {
        // contiguous range per warp
        const size_t per = n16 / (gridDim.x * streamers) / 32 * 32;
        const size_t b = (size_t)(blockIdx.x * streamers + warp) * per;
        if (lane == 0 && mode != 1 && mode != 2) {
            for (uint32_t o = 0; o < kPf; o += 4096)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;" ::"l"(g + b + o / 16) : "memory");
        }
        uint32_t pf = kPf;
        for (size_t i = 0; i < per; i += 64) {
            if (mode == 2) {
                const uint4 v0 = __ldg(g + b + i + lane), v1 = __ldg(g + b + i + 32 + lane);
                acc += v0.x ^ v0.w ^ v1.y ^ v1.z;
            } else {
                const uint4 v0 = tex1Dfetch<uint4>(t, (int)(b + i + lane));
                const uint4 v1 = tex1Dfetch<uint4>(t, (int)(b + i + 32 + lane));
                acc += v0.x ^ v0.w ^ v1.y ^ v1.z;
            }
            if (mode != 1 && mode != 2 && (i * 16 + 1024) % 4096 == 0 && pf < per * 16) {
                if (lane == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 4096;" ::"l"(g + b + pf / 16) : "memory");
                pf += 4096;
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    int sms = 0, clk = 0, maxw = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxTexture1DLinearWidth, 0);
    printf("max 1D linear texture width %d\n", maxw);
    const size_t n16 = (size_t)1 << 25;  // 512 MiB
    uint4* g;
    uint32_t* out;
    cudaMalloc(&g, n16 * 16);
    cudaMemset(g, 1, n16 * 16);
    cudaMalloc(&out, sms * 1024 * 4);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = g;
    rd.res.linear.desc = cudaCreateChannelDesc<uint4>();
    rd.res.linear.sizeInBytes = n16 * 16;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t;
    cudaError_t e = cudaCreateTextureObject(&t, &rd, &td, nullptr);
    printf("tex create: %s\n", cudaGetErrorString(e));
    float* fl;
    cudaMalloc(&fl, 512 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"TEX+L2pf", "TEX no pf", "LDG.128", "TEX24+LDS8"};
    for (int mode = 0; mode < 4; ++mode) {
        float best = 1e9;
        for (int r = 0; r < 4; ++r) {
            cudaMemset(fl, 0, 512 << 20);  // evict L2
            cudaEventRecord(a);
            k<<<sms, 1024>>>(t, g, n16, out, mode);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const int streamers = mode == 3 ? 24 : 32;
        const size_t per = n16 / (sms * streamers) / 32 * 32;
        const double bytes = (double)per * sms * streamers * 16;
        printf("%-12s %8.3f ms  %7.1f GB/s  (err %s)\n", names[mode], best, bytes / best / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
