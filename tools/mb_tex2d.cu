// Microbenchmark: does a block-linear 2-D texture (cudaArray) make the SpMV's x gathers cheaper
// for the TEX pipe than the 1-D linear texture?  Same replayed d-density step patterns as
// mb_lanes.cu (g = 8: lane l holds elements 8l..8l+7 of a 256-element step); column c is fetched
// at (c mod W, c / W) with integer coordinates (tex.2d ... .s32), all 8 slots through TEX.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_tex2d tools/mb_tex2d.cu
//   ./tools/mb_tex2d [density]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kTable = 16384;

__device__ __forceinline__ uint32_t tex2d_u16(cudaTextureObject_t t, int x, int y) {
    uint32_t r0, r1, r2, r3;
    asm volatile("tex.2d.v4.u32.s32 {%0, %1, %2, %3}, [%4, {%5, %6}];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "l"(t), "r"(x), "r"(y));
    return r0;
}

template <int kLogW>  // kLogW < 0: 1-D linear texture
__global__ void __launch_bounds__(1024, 1) k(cudaTextureObject_t tex, const uint16_t* pat, uint32_t* out,
                                             unsigned long long* cyc) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * 32 + warp;
    uint32_t off[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) off[j] = pat[(gw * 8 + j) * 32 + lane];
    uint32_t acc = 0;
    uint32_t base = (uint32_t)gw * 97u;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
        base = (base + 523u) & (kTable / 2 - 1u);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const uint32_t c = base + off[s];
            if constexpr (kLogW < 0) {
                acc += tex1Dfetch<unsigned short>(tex, (int)c);
            } else {
                acc += tex2d_u16(tex, (int)(c & ((1u << kLogW) - 1u)), (int)(c >> kLogW));
            }
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int L>
double run(cudaTextureObject_t tex, const uint16_t* pat, uint32_t* out, unsigned long long* cyc, int sms) {
    k<L><<<sms, 1024>>>(tex, pat, out, cyc);
    k<L><<<sms, 1024>>>(tex, pat, out, cyc);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(sms);
    cudaMemcpy(h.data(), cyc, sms * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    for (auto v : h) s += (double)v;
    return s / sms / (32.0 * kIters);
}

cudaTextureObject_t make2d(int logw, cudaArray_t* arr) {
    const int W = 1 << logw, H = kTable / W;
    cudaChannelFormatDesc cd = cudaCreateChannelDesc<unsigned short>();
    cudaMallocArray(arr, &cd, W, H);
    std::vector<uint16_t> h(kTable, 1);
    cudaMemcpy2DToArray(*arr, 0, 0, h.data(), W * 2, W * 2, H, cudaMemcpyHostToDevice);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = *arr;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    td.filterMode = cudaFilterModePoint;
    td.normalizedCoords = 0;
    td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
    cudaTextureObject_t t;
    cudaCreateTextureObject(&t, &rd, &td, nullptr);
    return t;
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
    cudaMalloc(&g, kTable * 2);
    cudaMemset(g, 1, kTable * 2);
    cudaMalloc(&out, sms * 1024 * 4);
    cudaMalloc(&cyc, sms * 8);
    cudaMalloc(&pat, (size_t)nw * 256 * 2);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = g;
    rd.res.linear.desc = cudaCreateChannelDesc<unsigned short>();
    rd.res.linear.sizeInBytes = kTable * 2;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex1;
    cudaCreateTextureObject(&tex1, &rd, &td, nullptr);
    std::mt19937_64 rng(42);
    std::bernoulli_distribution bern(d);
    std::vector<uint16_t> h((size_t)nw * 256);
    for (int w = 0; w < nw; ++w) {
        uint32_t c = 0;
        std::vector<uint16_t> st(256);
        for (int e = 0; e < 256; ++e) {
            do { ++c; } while (!bern(rng));
            st[e] = (uint16_t)c;
        }
        for (int j = 0; j < 8; ++j)
            for (int l = 0; l < 32; ++l) h[((size_t)w * 8 + j) * 32 + l] = st[l * 8 + j];
    }
    cudaMemcpy(pat, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    printf("density %.2f: clocks per 8-TEX-gather warp-step per SM (32 warps/SM)\n", d);
    printf("1-D linear: %.2f\n", run<-1>(tex1, pat, out, cyc, sms));
    cudaArray_t arr[8];
    printf("2-D block-linear W=8: %.2f\n", run<3>(make2d(3, &arr[0]), pat, out, cyc, sms));
    printf("2-D block-linear W=16: %.2f\n", run<4>(make2d(4, &arr[1]), pat, out, cyc, sms));
    printf("2-D block-linear W=32: %.2f\n", run<5>(make2d(5, &arr[2]), pat, out, cyc, sms));
    printf("2-D block-linear W=64: %.2f\n", run<6>(make2d(6, &arr[3]), pat, out, cyc, sms));
    printf("2-D block-linear W=128: %.2f\n", run<7>(make2d(7, &arr[4]), pat, out, cyc, sms));
    printf("2-D block-linear W=256: %.2f\n", run<8>(make2d(8, &arr[5]), pat, out, cyc, sms));
    printf("(err %s)\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
