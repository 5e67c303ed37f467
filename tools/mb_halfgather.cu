// Microbenchmark: does an LDS gather with half of the lanes predicated off cost half the
// L1 data-pipe time?  (Skipping the gather of an element whose column follows its predecessor's,
// when a 32-bit load of x[c], x[c+1] already fetched it.)  1 CTA/SM x 16 warps; lane l reads
// column base + 16 l + r (r random in [0,16)), the SpMV's pattern at density 0.5.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kTable = 8192;

__global__ void __launch_bounds__(512, 1) k(float* out, int mode) {
    __shared__ uint32_t xs[kTable / 2 + 8];
    for (int i = threadIdx.x; i < kTable / 2 + 8; i += blockDim.x) xs[i] = (uint32_t)(i * 7);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t h = 12345u + 977u * (warp + 16 * blockIdx.x);
    uint32_t acc = 0;
    const uint16_t* xs16 = reinterpret_cast<const uint16_t*>(xs);
#pragma unroll 8
    for (int i = 0; i < kIters; ++i) {
        h = h * 1664525u + 1013904223u;
        const uint32_t hl = h ^ (uint32_t)(lane * 0x9E3779B9u);
        const uint32_t base = (h >> 8) & (kTable - 1);
        const uint32_t c = (base + 16u * lane + ((hl >> 24) & 15u)) & (kTable - 1);
        if (mode == 0) {
            acc += xs16[c];                                  // LDS.U16, all lanes
        } else if (mode == 1) {
            if ((hl >> 20) & 1u) acc += xs16[c];             // LDS.U16, ~half the lanes
        } else if (mode == 2) {
            acc += xs[c >> 1];                               // LDS.32, all lanes
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

int main() {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, sms * 512 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"LDS.U16 all lanes", "LDS.U16 half lanes", "LDS.32 all lanes"};
    for (int mode = 0; mode < 3; ++mode) {
        k<<<sms, 512>>>(out, mode);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k<<<sms, 512>>>(out, mode);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        const double cyc = ms * 1e-3 * clk_khz * 1e3;
        printf("%-20s %8.3f ms  warp-gathers/clk/SM %.3f  clk/gather %.2f (err %s)\n", names[mode], ms, 16.0 * kIters / cyc,
               cyc / (16.0 * kIters), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
