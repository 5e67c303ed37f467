// Microbenchmark: can x gathers be split between the LSU data pipe (LDS from a shared-memory
// table) and the TEX pipe (tex1Dfetch from an L1-resident texture) so that the two run in
// parallel?  1 CTA/SM x 16 warps.  Each warp-gather mimics the SpMV's lane-consecutive pattern:
// lane l reads column base + S l + r (r random in [0,S)), S = argv[1] (16: a 1 KiB window of fp16,
// the lane-consecutive SpMV at d = 0.5; 4: the pair-interleaved mapping).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kTable = 8192;  // fp16 entries (16 KiB)

__device__ uint32_t g_lanerand = 0;  // 1: the in-lane offset r is random per lane (the SpMV's
                                     // pattern); 0: warp-uniform r (a pathological bank pattern)
__device__ __forceinline__ uint32_t col_of(uint32_t& h, int lane, uint32_t stride) {
    h = h * 1664525u + 1013904223u;
    const uint32_t base = (h >> 8) & (kTable - 1);  // varies per step (warp-uniform)
    const uint32_t hl = g_lanerand ? h ^ (uint32_t)(lane * 0x9E3779B9u) : h;
    return (base + stride * lane + ((hl >> 24) & (stride - 1u))) & (kTable - 1);
}

// mode: 0 all LDS, 1 all TEX, 2 half LDS + half TEX, 3 half LDS only, 4 half TEX only, 5 all LDG(L1)
__global__ void __launch_bounds__(512, 1) k(cudaTextureObject_t tex, const uint16_t* __restrict__ g, float* out,
                                             int mode, uint32_t stride) {
    __shared__ uint16_t xs[kTable];
    for (int i = threadIdx.x; i < kTable; i += blockDim.x) xs[i] = (uint16_t)(i * 7);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t h = 12345u + 977u * (warp + 16 * blockIdx.x);  // warp-uniform seed
    uint32_t hl = h;
    uint32_t acc = 0;
    bool lds = false, tx = false, ldg = false;
    if (mode == 0) lds = true;
    if (mode == 1) tx = true;
    if (mode == 2) (warp & 1 ? tx : lds) = true;
    if (mode == 3) lds = (warp & 1) == 0;
    if (mode == 4) tx = (warp & 1) == 1;
    if (mode == 5) ldg = true;
    if (lds) {
#pragma unroll 8
        for (int i = 0; i < kIters; ++i) acc += xs[col_of(hl, lane, stride)];
    } else if (tx) {
#pragma unroll 8
        for (int i = 0; i < kIters; ++i) acc += tex1Dfetch<unsigned short>(tex, (int)col_of(hl, lane, stride));
    } else if (ldg) {
#pragma unroll 8
        for (int i = 0; i < kIters; ++i) acc += __ldg(g + col_of(hl, lane, stride));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

int main(int argc, char** argv) {
    const uint32_t stride = argc > 1 ? (uint32_t)atoi(argv[1]) : 16u;  // lane column stride (power of 2)
    const uint32_t lanerand = argc > 2 ? (uint32_t)atoi(argv[2]) : 1u;
    cudaMemcpyToSymbol(g_lanerand, &lanerand, 4);
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    uint16_t* g;
    float* out;
    cudaMalloc(&g, kTable * 2);
    cudaMemset(g, 1, kTable * 2);
    cudaMalloc(&out, sms * 512 * 4);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = g;
    rd.res.linear.desc = cudaCreateChannelDesc<unsigned short>();
    rd.res.linear.sizeInBytes = kTable * 2;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex;
    cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"16w LDS", "16w TEX", "8 LDS + 8 TEX", "8w LDS only", "8w TEX only", "16w LDG"};
    const double gw[] = {16, 16, 16, 8, 8, 16};
    for (int mode = 0; mode < 6; ++mode) {
        k<<<sms, 512>>>(tex, g, out, mode, stride);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k<<<sms, 512>>>(tex, g, out, mode, stride);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        const double cyc = ms * 1e-3 * clk_khz * 1e3;
        printf("%-16s %8.3f ms  warp-gathers/clk/SM %.3f  (err %s)\n", names[mode], ms, gw[mode] * kIters / cyc,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
