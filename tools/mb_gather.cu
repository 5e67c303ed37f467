// Microbenchmark: gather throughput of the two x paths with the SpMV's access pattern and ILP.
// 1 CTA/SM x 32 warps; per iteration a warp computes 8 columns per lane (lane l: base_k + S*l + r,
// r random per lane in [0, S)) and issues 8 independent 16-bit gathers, each through LDS (fp16
// table in shared memory) or TEX (tex1Dfetch on an L1-resident texture) by a mask over the 8
// slots — the SpMV's x_mode.  Reports clocks per warp-gather and per 8-gather step.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kIters = 2048;
constexpr int kTable = 12288;  // fp16 entries (24 KiB): the headline's x

template <uint32_t kTexMask>
__global__ void __launch_bounds__(1024, 1) k(cudaTextureObject_t tex, float* out, uint32_t stride) {
    __shared__ uint16_t xs[kTable];
    for (int i = threadIdx.x; i < kTable; i += blockDim.x) xs[i] = (uint16_t)(i * 7);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t h = 12345u + 977u * (warp + 32 * blockIdx.x);
    const uint32_t lh = (uint32_t)lane * 0x9E3779B9u;
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < kIters; ++i) {
        h = h * 1664525u + 1013904223u;
        const uint32_t hl = h ^ lh;
        const uint32_t base = (h >> 16) + stride * (uint32_t)lane;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const uint32_t c = (base + 512u * s + ((hl >> (4 * s)) & (stride - 1u))) % kTable;
            if ((kTexMask >> s) & 1u)
                acc[s] += tex1Dfetch<unsigned short>(tex, (int)c);
            else
                acc[s] += xs[c];
        }
    }
    uint32_t t = 0;
#pragma unroll
    for (int s = 0; s < 8; ++s) t += acc[s];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)t;
}

template <uint32_t M>
float run(cudaTextureObject_t tex, float* out, int sms, uint32_t stride) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<M><<<sms, 1024>>>(tex, out, stride);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<M><<<sms, 1024>>>(tex, out, stride);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main(int argc, char** argv) {
    const uint32_t stride = argc > 1 ? (uint32_t)atoi(argv[1]) : 16u;
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    uint16_t* g;
    float* out;
    cudaMalloc(&g, kTable * 2);
    cudaMemset(g, 1, kTable * 2);
    cudaMalloc(&out, sms * 1024 * 4);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = g;
    rd.res.linear.desc = cudaCreateChannelDesc<unsigned short>();
    rd.res.linear.sizeInBytes = kTable * 2;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex;
    cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    auto report = [&](const char* name, float ms) {
        const double cyc = ms * 1e-3 * clk_khz * 1e3;
        const double steps = 32.0 * kIters;  // warp-steps per SM
        printf("stride %2u %-22s %7.3f ms  clk per 8-gather warp-step per SM %.2f\n", stride, name, ms, cyc / steps);
    };
    report("8 LDS (mode 1)", run<0x00>(tex, out, sms, stride));
    report("8 TEX (mode 0)", run<0xFF>(tex, out, sms, stride));
    report("5 LDS + 3 TEX (mode 6)", run<0x49>(tex, out, sms, stride));
    report("4 LDS + 4 TEX (mode 7)", run<0x55>(tex, out, sms, stride));
    report("6 LDS + 2 TEX (mode 8)", run<0x11>(tex, out, sms, stride));
    report("2 LDS + 6 TEX", run<0x77>(tex, out, sms, stride));
    printf("(err %s)\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
