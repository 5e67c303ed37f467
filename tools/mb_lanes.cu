// Microbenchmark: x-gather cost versus how a warp's 256-element step is spread over its lanes.
//
// Every warp holds one real d-density step pattern (host-generated Bernoulli(d) row, 256
// consecutive stored elements, columns relative to the step start) and replays it at a moving
// base: per iteration 8 independent 16-bit gathers per lane through LDS (fp16 table in shared
// memory) or TEX (tex1Dfetch, L1-resident) by a slot mask.  Lane granularity g: lane l's slot j
// is element (j / g) * 32g + l*g + (j % g) of the step — g = 8 is the current kernel's
// lane-consecutive layout, g = 1 the fully interleaved one.  Reports SM clocks per 8-gather
// warp-step (clock64 inside the kernel, 32 warps per SM).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_lanes tools/mb_lanes.cu
//   ./tools/mb_lanes [density]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kTable = 16384;  // fp16 entries (32 KiB), power of two
constexpr int kSlack = 2048;

template <uint32_t kTexMask>
__global__ void __launch_bounds__(1024, 1) k(cudaTextureObject_t tex, const uint16_t* pat, uint32_t* out,
                                             unsigned long long* cyc) {
    __shared__ uint16_t xs[kTable + kSlack];
    for (int i = threadIdx.x; i < kTable + kSlack; i += blockDim.x) xs[i] = (uint16_t)(i * 7);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * 32 + warp;
    uint32_t off[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) off[j] = pat[(gw * 8 + j) * 32 + lane];
    const uint32_t xs_addr = (uint32_t)__cvta_generic_to_shared(xs);
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t base = (uint32_t)gw * 97u;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
        base = (base + 523u) & (kTable - 1u);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const uint32_t c = base + off[s];
            if ((kTexMask >> s) & 1u) {
                acc[s] += tex1Dfetch<unsigned short>(tex, (int)c);
            } else {
                uint16_t v;
                asm volatile("ld.shared.b16 %0, [%1];" : "=h"(v) : "r"(xs_addr + 2u * c));
                acc[s] += v;
            }
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    uint32_t t = 0;
#pragma unroll
    for (int s = 0; s < 8; ++s) t += acc[s];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <uint32_t M>
double run(cudaTextureObject_t tex, const uint16_t* pat, uint32_t* out, unsigned long long* cyc, int sms) {
    k<M><<<sms, 1024>>>(tex, pat, out, cyc);
    k<M><<<sms, 1024>>>(tex, pat, out, cyc);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(sms);
    cudaMemcpy(h.data(), cyc, sms * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    for (auto v : h) s += (double)v;
    return s / sms / (32.0 * kIters);  // clocks per warp-step (8 gathers) per SM
}

int main(int argc, char** argv) {
    const double d = argc > 1 ? atof(argv[1]) : 0.5;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nw = sms * 32;
    uint16_t* g;
    uint32_t* out;
    unsigned long long* cyc;
    uint16_t* pat;
    cudaMalloc(&g, (kTable + kSlack) * 2);
    cudaMemset(g, 1, (kTable + kSlack) * 2);
    cudaMalloc(&out, sms * 1024 * 4);
    cudaMalloc(&cyc, sms * 8);
    cudaMalloc(&pat, (size_t)nw * 256 * 2);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = g;
    rd.res.linear.desc = cudaCreateChannelDesc<unsigned short>();
    rd.res.linear.sizeInBytes = (kTable + kSlack) * 2;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex;
    cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    std::mt19937_64 rng(42);
    std::bernoulli_distribution bern(d);
    // per warp: 256 consecutive stored elements of a Bernoulli(d) row, columns relative to the step
    std::vector<std::vector<uint16_t>> steps(nw);
    for (int w = 0; w < nw; ++w) {
        uint32_t c = 0;
        steps[w].resize(256);
        for (int e = 0; e < 256; ++e) {
            do { ++c; } while (!bern(rng));
            steps[w][e] = (uint16_t)c;
        }
    }
    printf("density %.2f, %d SMs, clocks per 8-gather warp-step per SM (32 warps/SM)\n", d, sms);
    printf("%-4s %8s %8s %8s %8s %8s %8s %8s\n", "g", "8LDS", "1TEX", "2TEX", "3TEX", "4TEX", "6TEX", "8TEX");
    for (int gran : {1, 2, 4, 8}) {
        std::vector<uint16_t> h((size_t)nw * 256);
        for (int w = 0; w < nw; ++w)
            for (int j = 0; j < 8; ++j)
                for (int l = 0; l < 32; ++l) {
                    const int e = (j / gran) * 32 * gran + l * gran + (j % gran);
                    h[((size_t)w * 8 + j) * 32 + l] = steps[w][e];
                }
        cudaMemcpy(pat, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
        printf("%-4d %8.2f %8.2f %8.2f %8.2f %8.2f %8.2f %8.2f\n", gran, run<0x00>(tex, pat, out, cyc, sms),
               run<0x01>(tex, pat, out, cyc, sms), run<0x11>(tex, pat, out, cyc, sms),
               run<0x49>(tex, pat, out, cyc, sms), run<0x55>(tex, pat, out, cyc, sms),
               run<0x77>(tex, pat, out, cyc, sms), run<0xFF>(tex, pat, out, cyc, sms));
    }
    printf("(err %s)\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
