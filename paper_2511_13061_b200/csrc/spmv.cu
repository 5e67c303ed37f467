// spmv.cu — MACKO SpMV for sm_100a (b_delta = 4, fp16 values, fp32 accumulation).
//
// Realises the paper's warp kernel (SPEC.md:255-264 warp_spmv) natively:
//   * one warp walks a row in steps of 256 elements, lane l owning elements 8l..8l+7 of the
//     step: one 16-B streaming load of values and one 4-B load of packed deltas per lane
//     (PAPER.md:318-323), both L1::no_allocate;
//   * ROMA: the row start is aligned down to 8 elements and the elements
//     before it are masked in the first step; lanes past the row end are masked in the last;
//   * column reconstruction: the 8 nibbles are widened to bytes, paired and prefix-summed with
//     one integer multiply (byte-SIMD), then Algorithm 1's 5-level shfl_up scan gives the lane
//     offset and lane 31's total advances the running column;
//   * x is staged once per CTA in shared memory and gathered per element; the multiply-add is
//     FHFMA (fp16 x fp16 -> fp32 accumulate, exact product);
//   * B200 work distribution: a persistent grid (SM count x occupancy) where every warp owns
//     an equal-weight contiguous range of 1024-element units (a static plan built once per
//     matrix), so short matrices and long rows are balanced; rows cut between warps are
//     finished by the last-arriving warp, which adds the per-unit partials in unit order.
// Summation order (all lanes, every run, any grid): per lane sequential over its elements,
// xor-tree over lanes once per unit, sequential over units — mirrored bit-exactly by
// oracle mo_b200_order_spmv(unit_steps = kUnitSteps).
#include "common.cuh"
#include "spmv.cuh"

namespace mk {

namespace {

// Byte-wise masks for the 4 even (elements 0,2,4,6) and 4 odd (1,3,5,7) deltas of a lane.
__device__ __forceinline__ void edge_masks(uint32_t vm, uint32_t& me, uint32_t& mo) {
    me = 0;
    mo = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        me |= ((vm >> (2 * m)) & 1u) ? (0xFFu << (8 * m)) : 0u;
        mo |= ((vm >> (2 * m + 1)) & 1u) ? (0xFFu << (8 * m)) : 0u;
    }
}

template <bool kSmemX>
__device__ __forceinline__ uint16_t xload(const uint16_t* xs, const uint16_t* xg, int c) {
    if constexpr (kSmemX) {
        return xs[c];
    } else {
        return __ldg(xg + c);
    }
}

// One warp step over 8 elements per lane.  vm = valid-element mask (0xFF when kEdge false).
template <bool kEdge, bool kSmemX>
__device__ __forceinline__ void step(const uint16_t* xs, const uint16_t* xg, const uint4& v, uint32_t d,
                                     uint32_t vm, int lane, int& col_base, float& acc) {
    uint32_t dl = (d & 0x0F0F0F0Fu) + 0x01010101u;         // deltas of elements 0,2,4,6
    uint32_t dh = ((d >> 4) & 0x0F0F0F0Fu) + 0x01010101u;  // deltas of elements 1,3,5,7
    if constexpr (kEdge) {
        uint32_t me, mo;
        edge_masks(vm, me, mo);
        dl &= me;
        dh &= mo;
    }
    const uint32_t pp = (dl + dh) * 0x01010101u;  // byte m: inclusive delta sum to element 2m+1
    const uint32_t odd = pp;
    const uint32_t even = pp - dh;                 // byte m: inclusive delta sum to element 2m
    const uint32_t local = pp >> 24;
    const uint32_t incl = warp_incl_scan(local, lane);
    const uint32_t total = __shfl_sync(kFull, incl, kWarp - 1);
    const int lb = col_base + (int)(incl - local);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int c0 = lb + (int)((even >> (8 * m)) & 0xFFu);
        const int c1 = lb + (int)((odd >> (8 * m)) & 0xFFu);
        if (!kEdge || ((vm >> (2 * m)) & 1u))
            acc = fma_f16f16f32((uint16_t)(w[m] & 0xFFFFu), xload<kSmemX>(xs, xg, c0), acc);
        if (!kEdge || ((vm >> (2 * m + 1)) & 1u))
            acc = fma_f16f16f32((uint16_t)(w[m] >> 16), xload<kSmemX>(xs, xg, c1), acc);
    }
    col_base += (int)total;
}

template <bool kSmemX>
__global__ void __launch_bounds__(kSpmvWarpsPerCta * kWarp)
    macko_spmv_b4(const SpmvArgs a) {
    extern __shared__ __align__(16) uint16_t xs[];
    const int lane = threadIdx.x & (kWarp - 1);
    if constexpr (kSmemX) {
        const uint32_t C = a.cols;
        if ((reinterpret_cast<uintptr_t>(a.x) & 15u) == 0) {
            const uint32_t nv = C / 8;
            for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x)
                reinterpret_cast<uint4*>(xs)[i] = __ldg(reinterpret_cast<const uint4*>(a.x) + i);
            for (uint32_t i = nv * 8 + threadIdx.x; i < C; i += blockDim.x) xs[i] = a.x[i];
        } else {
            for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) xs[i] = a.x[i];
        }
        __syncthreads();
    }
    const uint32_t w = blockIdx.x * kSpmvWarpsPerCta + (threadIdx.x >> 5);
    const SpmvPlanDev& P = a.plan;
    uint32_t u = P.chunk_unit[w];
    const uint32_t u_end = P.chunk_unit[w + 1];
    if (u >= u_end) return;
    uint32_t r = P.chunk_row[w];
    uint32_t j = P.chunk_j[w];
    bool first_row = true;

    while (u < u_end) {
        const uint32_t s = __ldg(a.row_ptrs + r), e = __ldg(a.row_ptrs + r + 1);
        const uint32_t al = s & ~7u;
        const uint32_t T = e > s ? (e - al + kStepElts - 1) / kStepElts : 0u;
        const uint32_t n_r = T ? (T + kUnitSteps - 1) / kUnitSteps : 1u;
        const uint32_t nu = min(n_r - j, u_end - u);
        const bool split = !(j == 0 && j + nu == n_r);
        int col_base = j ? P.chunk_colbase[w] : -1;
        int32_t sid = -1;
        uint32_t slot = 0;
        if (split) {
            sid = first_row ? P.chunk_sid[2 * w] : P.chunk_sid[2 * w + 1];
            slot = P.split_slot[sid];
        }
        float row_acc = 0.0f;
        for (uint32_t uu = j; uu < j + nu; ++uu) {
            float acc = 0.0f;
            const uint32_t t0 = uu * kUnitSteps, t1 = min(T, t0 + kUnitSteps);
            for (uint32_t t = t0; t < t1; ++t) {
                const uint32_t eb = al + t * kStepElts + 8u * lane;  // lane's first element
                if (t == 0 || t + 1 == T) {
                    // edge step: ROMA mask before the row start, tail mask past the row end
                    const int klo = (int)max(0LL, min(8LL, (long long)s - (long long)eb));
                    const int khi = (int)max(0LL, min(8LL, (long long)e - (long long)eb));
                    const uint32_t vm = (0xFFu << klo) & (0xFFu >> (8 - khi)) & 0xFFu;
                    uint4 v = make_uint4(0, 0, 0, 0);
                    uint32_t d = 0;
                    if (vm) {
                        v = ldg_stream_v4(a.values + eb);
                        d = ldg_stream_u32(a.deltas + eb / 2);
                    }
                    step<true, kSmemX>(xs, a.x, v, d, vm, lane, col_base, acc);
                } else {
                    const uint4 v = ldg_stream_v4(a.values + eb);
                    const uint32_t d = ldg_stream_u32(a.deltas + eb / 2);
                    step<false, kSmemX>(xs, a.x, v, d, 0xFFu, lane, col_base, acc);
                }
            }
            const float red = warp_tree_sum(acc);
            if (split && j > 0 && lane == 0) P.partials[slot + uu] = red;
            row_acc += red;
        }
        if (!split) {
            if (lane == 0) a.y[r] = f32_to_f16_rn(row_acc);
        } else {
            // Rows cut between warps: the first piece stores its running sum, later pieces
            // stored per-unit partials above; the last arrival adds them in unit order.
            uint32_t last = 0;
            if (lane == 0) {
                if (j == 0) P.partials[slot + nu - 1] = row_acc;
                __threadfence();
                const uint32_t prev = atomicAdd(P.counters + sid, 1u);
                last = prev + 1 == P.split_pieces[sid];
            }
            last = __shfl_sync(kFull, last, 0);
            if (last) {
                __threadfence();
                const uint32_t f = P.split_first[sid];
                float tot = 0.0f;
                if (lane == 0) {
                    tot = __ldcg(P.partials + slot + f - 1);
                    for (uint32_t q = f; q < n_r; ++q) tot += __ldcg(P.partials + slot + q);
                    a.y[r] = f32_to_f16_rn(tot);
                    P.counters[sid] = 0;
                }
            }
        }
        u += nu;
        ++r;
        j = 0;
        first_row = false;
    }
}

// Column just before the first unit of every chunk that starts inside a row:
// sum of the row's deltas over [row start, unit start) minus one.  Setup only.
__global__ void plan_colbase_kernel(const uint8_t* deltas, const uint32_t* row_ptrs, const uint32_t* chunk_row,
                                    const uint32_t* chunk_j, int32_t* chunk_colbase, uint32_t n_chunks) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & (kWarp - 1);
    if (w >= n_chunks) return;
    const uint32_t j = chunk_j[w];
    if (j == 0) {
        if (lane == 0) chunk_colbase[w] = -1;
        return;
    }
    const uint32_t r = chunk_row[w];
    const uint32_t s = row_ptrs[r];
    const uint32_t lim = (s & ~7u) + j * kUnitElts;
    uint32_t sum = 0;
    for (uint32_t i = s + lane; i < lim; i += kWarp) sum += ((deltas[i >> 1] >> ((i & 1u) * 4)) & 15u) + 1u;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) sum += __shfl_xor_sync(kFull, sum, off);
    if (lane == 0) chunk_colbase[w] = (int32_t)sum - 1;
}

}  // namespace

cudaError_t spmv_occupancy(bool x_in_smem, size_t smem, int* ctas_per_sm) {
    if (x_in_smem) {
        cudaError_t e = cudaFuncSetAttribute(macko_spmv_b4<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, macko_spmv_b4<true>, kSpmvWarpsPerCta * kWarp, smem);
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, macko_spmv_b4<false>, kSpmvWarpsPerCta * kWarp, 0);
}

cudaError_t launch_spmv(const SpmvArgs& a, int grid, bool x_in_smem, size_t smem, cudaStream_t s) {
    if (x_in_smem)
        macko_spmv_b4<true><<<grid, kSpmvWarpsPerCta * kWarp, smem, s>>>(a);
    else
        macko_spmv_b4<false><<<grid, kSpmvWarpsPerCta * kWarp, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_plan_colbase(const uint8_t* deltas, const uint32_t* row_ptrs, const uint32_t* chunk_row,
                                const uint32_t* chunk_j, int32_t* chunk_colbase, uint32_t n_chunks, cudaStream_t s) {
    const int threads = 256;
    const int blocks = (int)((n_chunks * (uint64_t)kWarp + threads - 1) / threads);
    if (blocks) plan_colbase_kernel<<<blocks, threads, 0, s>>>(deltas, row_ptrs, chunk_row, chunk_j, chunk_colbase, n_chunks);
    return cudaGetLastError();
}

}  // namespace mk
