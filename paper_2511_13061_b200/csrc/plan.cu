// plan.cu — the SpMV's static work plan built on the device (no host walk over rows and units).
//
// The same plan as the host builder (capi.cu build_plan_host): every row is cut into units of
// kUnitSteps warp steps from its 8-aligned start (the last unit absorbs a shorter remainder), unit
// weights are steps * 256 elements (+ plan_row_weight() for a row's first unit), and unit u goes to
// warp k(u) = min(W - 1, floor((2 cw(u) + w(u)) W / (2 total))) — its weight midpoint on an
// equal-weight grid of W warps, cw(u) the weight before u (plan_warp_of; a chain-skewed grid gives
// early CTAs larger shares, plan.cuh PlanGrid).  k(u) never decreases, so warp k owns
// the contiguous units [first unit with k(u) >= k, first unit with k(u) > k).  Rows cut between
// warps get a split id, per-unit partial slots and an arrival count.
//
//   plan_rows      : per row: units, weight                        (thread per row)
//   scan_u32/u64   : exclusive scans (one CTA)                      -> unit / weight offsets
//   plan_units     : per unit: k(u), its row and index in the row  (thread per row)
//   plan_chunk_init: chunk tables reset
//   plan_starts    : chunk_unit / row / j of every chunk a unit starts
//   plan_splits    : per row: split?, first-piece units, pieces      -> scan -> sid, slot
//   plan_split_recs: split records and the chunks' split ids
//   plan_records   : the 48-byte WarpPlan of every warp (TMA element range included)
#include "common.cuh"
#include "plan.cuh"
#include "spmv.cuh"

#include <algorithm>
#include <cstdlib>

namespace mk {

namespace {


__device__ __forceinline__ void row_geom(const uint32_t* rp, uint32_t r, uint32_t& s, uint32_t& e, uint32_t& al,
                                         uint32_t& T, uint32_t& n_r) {
    s = rp[r];
    e = rp[r + 1];
    al = s & ~7u;
    T = e > s ? (e - al + kStepElts - 1) / kStepElts : 0u;
    n_r = T >= (uint32_t)kUnitSteps ? T / kUnitSteps : 1u;
}

__device__ __forceinline__ uint32_t unit_end_step(uint32_t T, uint32_t n_r, uint32_t j) {
    return j + 1 == n_r ? T : (j + 1) * kUnitSteps;
}

__global__ void plan_rows_kernel(const uint32_t* rp, uint32_t rows, uint32_t row_w, uint32_t* nu, unsigned long long* rw) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        uint32_t s, e, al, T, n_r;
        row_geom(rp, r, s, e, al, T, n_r);
        nu[r] = n_r;
        rw[r] = (unsigned long long)T * kStepElts + row_w;
    }
}

// Exclusive scan of n values into out[0..n] (out[n] = total), one CTA of 1024 threads.
template <typename T>
__global__ void __launch_bounds__(1024) scan_kernel(const T* in, uint32_t n, T* out) {
    __shared__ T sums[32];
    const uint32_t t = threadIdx.x, nt = blockDim.x;
    const uint64_t lo = (uint64_t)n * t / nt, hi = (uint64_t)n * (t + 1) / nt;
    T mine = 0;
    for (uint64_t i = lo; i < hi; ++i) mine += in[i];
    const int lane = t & 31, wid = t >> 5;
    T incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const T v = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += v;
    }
    if (lane == 31) sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        T ws = lane < (int)(nt / 32) ? sums[lane] : (T)0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const T v = __shfl_up_sync(kFull, ws, off);
            if (lane >= off) ws += v;
        }
        sums[lane] = ws;
    }
    __syncthreads();
    T run = incl - mine + (wid ? sums[wid - 1] : (T)0);
    for (uint64_t i = lo; i < hi; ++i) {
        const T v = in[i];
        out[i] = run;
        run += v;
    }
    if (t == nt - 1) out[n] = run;
}

__global__ void plan_units_kernel(const uint32_t* rp, uint32_t rows, uint32_t row_w, const uint32_t* uo,
                                  const unsigned long long* cw, PlanGrid grid, uint32_t* ku, uint32_t* urow,
                                  uint32_t* uj) {
    const unsigned long long total = cw[rows];
    const unsigned __int128 den = 2 * (unsigned __int128)(total ? total : 1ull);
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        uint32_t s, e, al, T, n_r;
        row_geom(rp, r, s, e, al, T, n_r);
        unsigned long long c = cw[r];
        for (uint32_t j = 0; j < n_r; ++j) {
            const uint32_t steps = unit_end_step(T, n_r, j) - min(T, j * kUnitSteps);
            const unsigned long long w = (unsigned long long)steps * kStepElts + (j == 0 ? row_w : 0u);
            const unsigned __int128 mid2 = 2 * (unsigned __int128)c + w;
            const unsigned long long k = plan_warp_of(mid2, den, grid);
            const uint32_t u = uo[r] + j;
            ku[u] = (uint32_t)k;
            urow[u] = r;
            uj[u] = j;
            c += w;
        }
    }
}

__global__ void plan_chunk_init_kernel(uint32_t W, const uint32_t* d_U, uint32_t* chunk_unit, uint32_t* chunk_row,
                                       uint32_t* chunk_j, int32_t* chunk_sid) {
    const uint32_t U = *d_U;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q <= W; q += gridDim.x * blockDim.x) {
        chunk_unit[q] = U;
        if (q < W) {
            chunk_row[q] = 0;
            chunk_j[q] = 0;
            chunk_sid[2 * q] = chunk_sid[2 * q + 1] = -1;
        }
    }
}

// Unit u starts every chunk in (k(u-1), k(u)] (chunks it jumps over stay empty: they start at u too).
__global__ void plan_starts_kernel(const uint32_t* ku, const uint32_t* urow, const uint32_t* uj, const uint32_t* d_U,
                                   uint32_t* chunk_unit, uint32_t* chunk_row, uint32_t* chunk_j) {
    const uint32_t U = *d_U;
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x) {
        const int64_t kp = u ? (int64_t)ku[u - 1] : -1;
        for (int64_t q = kp + 1; q <= (int64_t)ku[u]; ++q) {
            chunk_unit[q] = u;
            chunk_row[q] = urow[u];
            chunk_j[q] = uj[u];
        }
    }
}

__global__ void plan_splits_kernel(const uint32_t* rp, uint32_t rows, const uint32_t* uo, const uint32_t* ku,
                                   uint32_t* is_split, uint32_t* split_units, uint32_t* first_units,
                                   uint32_t* pieces) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        const uint32_t u0 = uo[r], u1 = uo[r + 1];
        const uint32_t kf = ku[u0], kl = ku[u1 - 1];
        const bool split = kf != kl;
        uint32_t f = 0, pc = 0;
        if (split)
            for (uint32_t u = u0; u < u1; ++u) {
                f += ku[u] == kf;
                pc += (u == u0 || ku[u] != ku[u - 1]);
            }
        is_split[r] = split;
        split_units[r] = split ? u1 - u0 : 0u;
        first_units[r] = f;
        pieces[r] = pc;
    }
}

__global__ void plan_split_recs_kernel(uint32_t rows, const uint32_t* uo, const uint32_t* ku, const uint32_t* is_split,
                                       const uint32_t* sid_of, const uint32_t* slot_of, const uint32_t* first_units,
                                       const uint32_t* pieces, const uint32_t* chunk_row, const uint32_t* chunk_j,
                                       uint4* splits, int32_t* chunk_sid) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        if (!is_split[r]) continue;
        const int32_t sid = (int32_t)sid_of[r];
        const uint32_t kf = ku[uo[r]], kl = ku[uo[r + 1] - 1];
        splits[sid] = make_uint4(slot_of[r], first_units[r], pieces[r], 0u);
        chunk_sid[2 * kf + 1] = sid;
        if (chunk_row[kf] == r && chunk_j[kf] == 0) chunk_sid[2 * kf] = sid;
        for (uint32_t k = kf + 1; k <= kl; ++k) {
            chunk_sid[2 * k] = sid;
            if (k < kl) chunk_sid[2 * k + 1] = sid;
        }
    }
}

// The warp's record; its TMA element range [e0, e1) spans the non-empty units it owns.
__global__ void plan_records_kernel(const uint32_t* rp, uint32_t W, uint32_t pad_nnz, const uint32_t* chunk_unit,
                                    const uint32_t* chunk_row, const uint32_t* chunk_j, const int32_t* chunk_sid,
                                    const uint32_t* urow, const uint32_t* uj, const uint4* splits, WarpPlan* recs) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < W; k += gridDim.x * blockDim.x) {
        WarpPlan c;
        c.units_left = chunk_unit[k + 1] - chunk_unit[k];
        c.row = chunk_row[k];
        c.j = chunk_j[k];
        c.e0 = c.e1 = 0;
        for (uint32_t u = chunk_unit[k]; u < chunk_unit[k + 1]; ++u) {
            uint32_t s, e, al, T, n_r;
            row_geom(rp, urow[u], s, e, al, T, n_r);
            if (!T) continue;
            const uint32_t j = uj[u];
            const uint32_t lo = al + j * kUnitElts;
            const uint32_t hi = min(al + kStepElts * unit_end_step(T, n_r, j), pad_nnz);
            if (c.e1 == 0) c.e0 = lo;
            c.e1 = max(c.e1, hi);
        }
        c.s = c.units_left ? rp[c.row] : 0u;
        c.e = c.units_left ? rp[c.row + 1] : 0u;
        c.colbase = -1;  // plan_colbase_kernel
        c.sid0 = chunk_sid[2 * k];
        c.sid1 = chunk_sid[2 * k + 1];
        c.slot0 = c.sid0 >= 0 ? splits[c.sid0].x : 0u;
        c.slot1 = c.sid1 >= 0 ? splits[c.sid1].x : 0u;
        recs[k] = c;
    }
}

__global__ void plan_totals_kernel(uint32_t rows, const uint32_t* uo, const uint32_t* sid_of, const uint32_t* slot_of,
                                   PlanTotals* out) {
    out->units = uo[rows];
    out->splits = sid_of[rows];
    out->slots = slot_of[rows];
    out->pad = 0;
}

int grid_of(uint64_t n, int sms) { return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 8)); }

}  // namespace

uint32_t plan_row_weight() {
    if (const char* e = std::getenv("MACKO_ROW_WEIGHT")) return (uint32_t)std::strtoul(e, nullptr, 10);
    return kPlanRowWeight;
}

cudaError_t plan_build_device(const uint32_t* rp, uint32_t rows, uint32_t pad_nnz, const PlanGrid& grid, uint64_t ubound,
                              int sms, uint32_t row_weight, const PlanTemp& t, WarpPlan* recs, uint4* splits,
                              PlanTotals* d_totals, cudaStream_t s) {
    const uint32_t W = grid.G * grid.A;
    plan_rows_kernel<<<grid_of(rows, sms), 256, 0, s>>>(rp, rows, row_weight, t.nu, t.rw);
    scan_kernel<uint32_t><<<1, 1024, 0, s>>>(t.nu, rows, t.uo);
    scan_kernel<unsigned long long><<<1, 1024, 0, s>>>(t.rw, rows, t.cw);
    plan_units_kernel<<<grid_of(rows, sms), 256, 0, s>>>(rp, rows, row_weight, t.uo, t.cw, grid, t.ku, t.urow, t.uj);
    plan_chunk_init_kernel<<<grid_of(W + 1, sms), 256, 0, s>>>(W, t.uo + rows, t.chunk_unit, t.chunk_row, t.chunk_j,
                                                              t.chunk_sid);
    plan_starts_kernel<<<grid_of(ubound, sms), 256, 0, s>>>(t.ku, t.urow, t.uj, t.uo + rows, t.chunk_unit, t.chunk_row,
                                                           t.chunk_j);
    plan_splits_kernel<<<grid_of(rows, sms), 256, 0, s>>>(rp, rows, t.uo, t.ku, t.is_split, t.split_units,
                                                         t.first_units, t.pieces);
    scan_kernel<uint32_t><<<1, 1024, 0, s>>>(t.is_split, rows, t.sid_of);
    scan_kernel<uint32_t><<<1, 1024, 0, s>>>(t.split_units, rows, t.slot_of);
    plan_split_recs_kernel<<<grid_of(rows, sms), 256, 0, s>>>(rows, t.uo, t.ku, t.is_split, t.sid_of, t.slot_of,
                                                             t.first_units, t.pieces, t.chunk_row, t.chunk_j, splits,
                                                             t.chunk_sid);
    plan_records_kernel<<<grid_of(W, sms), 256, 0, s>>>(rp, W, pad_nnz, t.chunk_unit, t.chunk_row, t.chunk_j,
                                                       t.chunk_sid, t.urow, t.uj, splits, recs);
    plan_totals_kernel<<<1, 1, 0, s>>>(rows, t.uo, t.sid_of, t.slot_of, d_totals);
    return cudaGetLastError();
}

}  // namespace mk
