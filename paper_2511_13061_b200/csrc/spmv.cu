// spmv.cu — MACKO SpMV for sm_100a (b_delta = 4, fp16 values, fp32 accumulation).
//
// Realises the paper's warp kernel (SPEC.md:255-264 warp_spmv) natively:
//   * one warp walks a row in steps of 256 elements, lane l owning elements 8l..8l+7 of the
//     step: one 16-B streaming load of values and one 4-B load of packed deltas per lane
//     (PAPER.md:318-323), both L1::no_allocate;
//   * ROMA: the row start is aligned down to 8 elements and the elements
//     before it are masked in the first step; lanes past the row end are masked in the last;
//   * column reconstruction: the 8 nibbles are widened to bytes, paired and prefix-summed with
//     one integer multiply (byte-SIMD), then Algorithm 1's shfl_up scan gives the lane offset
//     and lane 31's total advances the running column.  Two steps share one
//     scan (their lane sums packed into 16-bit halves);
//   * x is staged once per CTA in shared memory and gathered per element (PRMT + LEA + LDS);
//     the multiply-add is FHFMA (fp16 x fp16 -> fp32 accumulate, exact product);
//   * B200 work distribution and latency hiding: a persistent grid (SM count x occupancy)
//     where every warp owns an equal-weight contiguous range of 2048-element units (a static
//     plan built once per matrix).  A warp's loads run two step-pairs ahead of its math across
//     row boundaries (a 4-slot register ring fed by a loader cursor that replays the same walk),
//     so 4 x 640 B per warp are in flight.  Rows cut between warps are finished by the
//     last-arriving warp, which adds the per-unit partials in unit order.
// Summation order (every run, any grid): per lane sequential over its elements, xor-tree over
// lanes once per unit (8 steps), sequential over units — mirrored bit-exactly by
// oracle mo_b200_order_spmv(unit_steps = kUnitSteps).  The order depends on a row's elements
// and on its start offset mod 8 (ROMA), never on the plan.
#include "common.cuh"
#include "spmv.cuh"

namespace mk {

namespace {

// ------------------------------------------------------------------------------------------
// small helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void split_halves(uint32_t w, uint16_t& lo, uint16_t& hi) {
    asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(w));
}

__device__ __forceinline__ uint16_t lds_u16(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.b16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

// valid-element mask of a lane whose first element is eb, for the row [s, e)
__device__ __forceinline__ uint32_t lane_mask(uint32_t eb, uint32_t s, uint32_t e) {
    const int klo = (int)max(0LL, min(8LL, (long long)s - (long long)eb));
    const int khi = (int)max(0LL, min(8LL, (long long)e - (long long)eb));
    return (0xFFu << klo) & (0xFFu >> (8 - khi)) & 0xFFu;
}

struct Dec {
    uint32_t even, odd, local;  // inclusive in-lane column offsets (bytes m), lane total
};

// Nibbles -> byte deltas -> in-lane inclusive prefixes.  Masked elements get delta 0.
__device__ __forceinline__ Dec decode(uint32_t d, uint32_t vm) {
    uint32_t dl = (d & 0x0F0F0F0Fu) + 0x01010101u;         // elements 0,2,4,6
    uint32_t dh = ((d >> 4) & 0x0F0F0F0Fu) + 0x01010101u;  // elements 1,3,5,7
    if (vm != 0xFFu) {
        uint32_t me = 0, mo = 0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            me |= ((vm >> (2 * m)) & 1u) ? (0xFFu << (8 * m)) : 0u;
            mo |= ((vm >> (2 * m + 1)) & 1u) ? (0xFFu << (8 * m)) : 0u;
        }
        dl &= me;
        dh &= mo;
    }
    const uint32_t pp = (dl + dh) * 0x01010101u;
    return Dec{pp - dh, pp, pp >> 24};
}

// The 8 gathers + FHFMAs of one lane step.  `cb` = column of the element before the lane's
// first element; col(k) = cb + in-lane prefix byte.
template <bool kEdge, bool kSmemX>
__device__ __forceinline__ float fma_step(float acc, const uint4& v, const Dec& dc, int cb, uint32_t vm,
                                          uint32_t xs_addr, const uint16_t* xg) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    const uint32_t base = xs_addr + 2u * (uint32_t)cb;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        uint16_t v0, v1;
        split_halves(w[m], v0, v1);
        const uint32_t b0 = __byte_perm(dc.even, 0u, 0x4440u + m);
        const uint32_t b1 = __byte_perm(dc.odd, 0u, 0x4440u + m);
        if (!kEdge || ((vm >> (2 * m)) & 1u)) {
            const uint16_t x0 = kSmemX ? lds_u16(base + 2u * b0) : __ldg(xg + cb + (int)b0);
            acc = fma_f16f16f32(v0, x0, acc);
        }
        if (!kEdge || ((vm >> (2 * m + 1)) & 1u)) {
            const uint16_t x1 = kSmemX ? lds_u16(base + 2u * b1) : __ldg(xg + cb + (int)b1);
            acc = fma_f16f16f32(v1, x1, acc);
        }
    }
    return acc;
}

// ------------------------------------------------------------------------------------------
// Loader cursor: replays the warp's walk over (row, step) to issue loads ahead of the math.
// ------------------------------------------------------------------------------------------
struct Loader {
    uint32_t r, t, tend, al, e, units_left;
};

struct Slot {
    uint4 v;
    uint32_t d;
};

__device__ __forceinline__ bool loader_next(Loader& c, const uint32_t* __restrict__ rp, const uint16_t* __restrict__ values,
                                            const uint8_t* __restrict__ deltas, int lane, Slot& sl) {
    while (c.t >= c.tend) {
        if (c.units_left == 0) return false;
        ++c.r;
        const uint32_t s = __ldg(rp + c.r), e = __ldg(rp + c.r + 1);
        if (s == e) {
            c.units_left -= 1;
            continue;
        }
        c.al = s & ~7u;
        c.e = e;
        const uint32_t T = (e - c.al + kStepElts - 1) / kStepElts;
        const uint32_t nu = min((T + kUnitSteps - 1) / kUnitSteps, c.units_left);
        c.units_left -= nu;
        c.t = 0;
        c.tend = min(T, nu * kUnitSteps);
    }
    const uint32_t eb = c.al + c.t * kStepElts + 8u * lane;
    if (eb < c.e) {
        sl.v = ldg_stream_v4(values + eb);
        sl.d = ldg_stream_u32(deltas + eb / 2);
    } else {
        sl.v = make_uint4(0, 0, 0, 0);
        sl.d = 0;
    }
    ++c.t;
    return true;
}

// ------------------------------------------------------------------------------------------
// Compute-side row state
// ------------------------------------------------------------------------------------------
struct RowState {
    uint32_t r, s, e, al, T, t, tend, j0, n_r, units_left, slot;
    int32_t sid;
    bool split, first_row;
    int col_base;
    float acc, row_acc;
};

struct Ctx {
    const SpmvArgs* a;
    uint32_t w;
    int lane;
};

// Set up the piece of row rs.r starting at unit j0 (units_left = chunk units not yet placed).
__device__ __forceinline__ void begin_piece(RowState& rs, const Ctx& cx, uint32_t j0, int colbase) {
    const SpmvArgs& a = *cx.a;
    rs.s = __ldg(a.row_ptrs + rs.r);
    rs.e = __ldg(a.row_ptrs + rs.r + 1);
    rs.al = rs.s & ~7u;
    rs.T = rs.e > rs.s ? (rs.e - rs.al + kStepElts - 1) / kStepElts : 0u;
    rs.n_r = rs.T ? (rs.T + kUnitSteps - 1) / kUnitSteps : 1u;
    const uint32_t nu = min(rs.n_r - j0, rs.units_left);
    rs.units_left -= nu;
    rs.j0 = j0;
    rs.t = j0 * kUnitSteps;
    rs.tend = min(rs.T, (j0 + nu) * kUnitSteps);
    rs.split = !(j0 == 0 && j0 + nu == rs.n_r);
    rs.sid = -1;
    rs.slot = 0;
    if (rs.split) {
        rs.sid = rs.first_row ? a.plan.chunk_sid[2 * cx.w] : a.plan.chunk_sid[2 * cx.w + 1];
        rs.slot = a.plan.split_slot[rs.sid];
    }
    rs.col_base = colbase;
    rs.acc = 0.0f;
    rs.row_acc = 0.0f;
}

// Finish the current piece (write y or hand the split row to its last arrival).
__device__ __forceinline__ void finish_piece(RowState& rs, const Ctx& cx) {
    const SpmvArgs& a = *cx.a;
    const SpmvPlanDev& P = a.plan;
    if (!rs.split) {
        if (cx.lane == 0) a.y[rs.r] = f32_to_f16_rn(rs.row_acc);
        return;
    }
    uint32_t last = 0;
    if (cx.lane == 0) {
        if (rs.j0 == 0) P.partials[rs.slot + (rs.tend - 1) / kUnitSteps] = rs.row_acc;
        __threadfence();
        const uint32_t prev = atomicAdd(P.counters + rs.sid, 1u);
        last = prev + 1 == P.split_pieces[rs.sid];
    }
    last = __shfl_sync(kFull, last, 0);
    if (last && cx.lane == 0) {
        __threadfence();
        const uint32_t f = P.split_first[rs.sid];
        float tot = __ldcg(P.partials + rs.slot + f - 1);
        for (uint32_t q = f; q < rs.n_r; ++q) tot += __ldcg(P.partials + rs.slot + q);
        a.y[rs.r] = f32_to_f16_rn(tot);
        P.counters[rs.sid] = 0;  // ready for the next launch (stream order)
    }
}

// Move to the next non-empty row piece of the chunk; empty rows get y = +0.  Returns false
// when the chunk is exhausted.
__device__ __forceinline__ bool next_piece(RowState& rs, const Ctx& cx) {
    for (;;) {
        if (rs.units_left == 0) return false;
        ++rs.r;
        rs.first_row = false;
        begin_piece(rs, cx, 0, -1);
        if (rs.T) return true;
        if (cx.lane == 0) cx.a->y[rs.r] = 0;  // empty row: fp16(+0.0)
    }
}

// Account one finished step at (old) index t: unit end -> tree reduce; piece end -> finish.
// Returns false when the chunk is exhausted.
__device__ __forceinline__ bool end_step(RowState& rs, const Ctx& cx) {
    ++rs.t;
    if ((rs.t % kUnitSteps) == 0 || rs.t == rs.tend) {
        const float red = warp_tree_sum(rs.acc);
        rs.acc = 0.0f;
        if (rs.split && rs.j0 > 0 && cx.lane == 0) cx.a->plan.partials[rs.slot + (rs.t - 1) / kUnitSteps] = red;
        rs.row_acc += red;
    }
    if (rs.t == rs.tend) {
        finish_piece(rs, cx);
        return next_piece(rs, cx);
    }
    return true;
}

__device__ __forceinline__ bool is_edge(const RowState& rs, uint32_t t) { return t == 0 || t + 1 == rs.T; }

// One step alone (used when a pair would cross a piece boundary).
template <bool kSmemX>
__device__ __forceinline__ bool single_step(RowState& rs, const Ctx& cx, const Slot& sl, uint32_t xs_addr) {
    const uint32_t eb = rs.al + rs.t * kStepElts + 8u * cx.lane;
    const bool edge = is_edge(rs, rs.t);
    const uint32_t vm = edge ? lane_mask(eb, rs.s, rs.e) : 0xFFu;
    const Dec dc = decode(sl.d, vm);
    const uint32_t incl = warp_incl_scan(dc.local, cx.lane);
    const uint32_t tot = __shfl_sync(kFull, incl, kWarp - 1);
    const int cb = rs.col_base + (int)(incl - dc.local);
    if (edge)
        rs.acc = fma_step<true, kSmemX>(rs.acc, sl.v, dc, cb, vm, xs_addr, cx.a->x);
    else
        rs.acc = fma_step<false, kSmemX>(rs.acc, sl.v, dc, cb, vm, xs_addr, cx.a->x);
    rs.col_base += (int)tot;
    return end_step(rs, cx);
}

// Two consecutive steps of the same piece with one packed scan.
template <bool kSmemX>
__device__ __forceinline__ bool pair_step(RowState& rs, const Ctx& cx, const Slot& A, const Slot& B, uint32_t xs_addr) {
    const uint32_t ebA = rs.al + rs.t * kStepElts + 8u * cx.lane;
    const uint32_t ebB = ebA + kStepElts;
    const bool eA = is_edge(rs, rs.t), eB = is_edge(rs, rs.t + 1);
    const uint32_t vmA = eA ? lane_mask(ebA, rs.s, rs.e) : 0xFFu;
    const uint32_t vmB = eB ? lane_mask(ebB, rs.s, rs.e) : 0xFFu;
    const Dec dA = decode(A.d, vmA), dB = decode(B.d, vmB);
    const uint32_t packed = dA.local | (dB.local << 16);
    const uint32_t incl = warp_incl_scan(packed, cx.lane);
    const uint32_t tot = __shfl_sync(kFull, incl, kWarp - 1);
    const int cbA = rs.col_base + (int)((incl & 0xFFFFu) - dA.local);
    const int cbB = rs.col_base + (int)(tot & 0xFFFFu) + (int)((incl >> 16) - dB.local);
    if (eA)
        rs.acc = fma_step<true, kSmemX>(rs.acc, A.v, dA, cbA, vmA, xs_addr, cx.a->x);
    else
        rs.acc = fma_step<false, kSmemX>(rs.acc, A.v, dA, cbA, vmA, xs_addr, cx.a->x);
    rs.col_base += (int)(tot & 0xFFFFu);
    if (!end_step(rs, cx)) return false;  // cannot happen: B is in the same piece
    if (eB)
        rs.acc = fma_step<true, kSmemX>(rs.acc, B.v, dB, cbB, vmB, xs_addr, cx.a->x);
    else
        rs.acc = fma_step<false, kSmemX>(rs.acc, B.v, dB, cbB, vmB, xs_addr, cx.a->x);
    rs.col_base += (int)(tot >> 16);
    return end_step(rs, cx);
}

// Consume a loaded pair (A always valid; B valid iff hasB).
template <bool kSmemX>
__device__ __forceinline__ bool consume(RowState& rs, const Ctx& cx, const Slot& A, const Slot& B, bool hasB,
                                        uint32_t xs_addr) {
    if (hasB && rs.t + 1 < rs.tend) return pair_step<kSmemX>(rs, cx, A, B, xs_addr);
    if (!single_step<kSmemX>(rs, cx, A, xs_addr)) return false;
    if (hasB) return single_step<kSmemX>(rs, cx, B, xs_addr);
    return true;
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
    const uint32_t xs_addr = static_cast<uint32_t>(__cvta_generic_to_shared(xs));
    const uint32_t w = blockIdx.x * kSpmvWarpsPerCta + (threadIdx.x >> 5);
    const SpmvPlanDev& P = a.plan;
    const uint32_t u0 = P.chunk_unit[w], u_end = P.chunk_unit[w + 1];
    if (u0 >= u_end) return;
    const Ctx cx{&a, w, lane};

    RowState rs;
    rs.r = P.chunk_row[w];
    rs.units_left = u_end - u0;
    rs.first_row = true;
    const uint32_t j0 = P.chunk_j[w];
    begin_piece(rs, cx, j0, j0 ? P.chunk_colbase[w] : -1);

    Loader ld{rs.r, rs.t, rs.tend, rs.al, rs.e, rs.units_left};
    if (rs.T == 0) {
        if (lane == 0) a.y[rs.r] = 0;
        if (!next_piece(rs, cx)) return;
    }

    Slot s0, s1, s2, s3;
    bool k0 = loader_next(ld, a.row_ptrs, a.values, a.deltas, lane, s0);
    bool k1 = k0 && loader_next(ld, a.row_ptrs, a.values, a.deltas, lane, s1);
    bool k2 = k1 && loader_next(ld, a.row_ptrs, a.values, a.deltas, lane, s2);
    bool k3 = k2 && loader_next(ld, a.row_ptrs, a.values, a.deltas, lane, s3);
    for (;;) {
        if (!k0) break;
        if (!consume<kSmemX>(rs, cx, s0, s1, k1, xs_addr)) break;
        k0 = k3 && loader_next(ld, a.row_ptrs, a.values, a.deltas, lane, s0);
        k1 = k0 && loader_next(ld, a.row_ptrs, a.values, a.deltas, lane, s1);
        if (!k2) break;
        if (!consume<kSmemX>(rs, cx, s2, s3, k3, xs_addr)) break;
        k2 = k1 && loader_next(ld, a.row_ptrs, a.values, a.deltas, lane, s2);
        k3 = k2 && loader_next(ld, a.row_ptrs, a.values, a.deltas, lane, s3);
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
