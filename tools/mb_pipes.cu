// Microbenchmark: which warp-collective instructions consume L1/LSU data-pipe wavefronts on
// sm_100a (SHFL vs VOTE.ballot + POPC vs REDUX).  Run under ncu; see profiles/r01_pipes.md.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_shfl(unsigned* out, int n) {
    unsigned v = threadIdx.x;
    for (int i = 0; i < n; ++i) v += __shfl_up_sync(0xffffffffu, v, 1 + (i & 7));
    out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
__global__ void k_vote(unsigned* out, int n) {
    unsigned v = threadIdx.x;
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    for (int i = 0; i < n; ++i) v += __popc(__ballot_sync(0xffffffffu, (v >> (i & 7)) & 1u) & lt);
    out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
__global__ void k_redux(unsigned* out, int n) {
    unsigned v = threadIdx.x;
    for (int i = 0; i < n; ++i) v += __reduce_add_sync(0xffffffffu, v & (255u >> (i & 3)));
    out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
__global__ void k_match(unsigned* out, int n) {
    unsigned v = threadIdx.x;
    for (int i = 0; i < n; ++i) v += __popc(__match_any_sync(0xffffffffu, v & 7u));
    out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
int main() {
    unsigned* d;
    cudaMalloc(&d, 148 * 1024 * 4 * 8);
    const int n = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, void (*k)(unsigned*, int)) {
        k<<<148 * 4, 256>>>(d, n);
        cudaEventRecord(a);
        k<<<148 * 4, 256>>>(d, n);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = 148.0 * 4 * 8 * n;  // warp-instructions of the collective
        printf("%-6s %8.3f ms  %.2f warp-ops/clk/SM @1.9GHz\n", name, ms, ops / (ms * 1e-3) / 148 / 1.9e9);
    };
    run("shfl", k_shfl);
    run("vote", k_vote);
    run("redux", k_redux);
    run("match", k_match);
    return 0;
}
