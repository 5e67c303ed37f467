// plan.cuh — the SpMV work plan built on the device (plan.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "spmv.cuh"

namespace mk {

// Device scratch of one plan build (rows R, warps W, units <= ubound = 2 R + pad_nnz / kUnitElts + 16).
struct PlanTemp {
    uint32_t* nu;                // R: units per row
    unsigned long long* rw;      // R: row weight
    uint32_t* uo;                // R + 1: unit offsets (uo[R] = U)
    unsigned long long* cw;      // R + 1: weight offsets (cw[R] = total weight)
    uint32_t *ku, *urow, *uj;    // ubound: warp, row, index in the row of every unit
    uint32_t *chunk_unit, *chunk_row, *chunk_j;  // W + 1, W, W
    int32_t* chunk_sid;          // 2 W
    uint32_t *is_split, *split_units, *first_units, *pieces;  // R
    uint32_t *sid_of, *slot_of;  // R + 1: split id / first partial slot of every row (scans)
};

struct PlanTotals {
    uint32_t units, splits, slots, pad;
};

// Plan weight of starting a row, in element equivalents (both builders).  Measured (traces of
// 36864x12288, tools/trace_corr.py): a warp's lateness against its CTA's median regresses on its
// elements and its rows with 1.64 us per row vs 0.70 us per 1000 elements (R^2 0.84 with split
// pieces and warp index): a row start (edge pairs, row set-up, y store) costs ~2000 elements of
// walk, not the 128 the first plans used.  MACKO_ROW_WEIGHT overrides (experiments).
#ifndef MACKO_PLAN_ROW_WEIGHT
#define MACKO_PLAN_ROW_WEIGHT 128
#endif
constexpr uint32_t kPlanRowWeight = MACKO_PLAN_ROW_WEIGHT;
uint32_t plan_row_weight();

// The grid a plan cuts the unit stream for: G CTAs of A active warps; CTA c's share of the weight
// is proportional to K (G-1) + R (G-1-2c) (R = 0: every warp the same share).  A positive R gives
// early CTAs more and late CTAs less: in a PDL chain CTA c starts when the c-th SM is released by
// the previous SpMV, up to ~2 us after the first (tools/trace_chain.py), so equal shares end
// late by that spread.
struct PlanGrid {
    uint32_t G, A;  // CTAs, active warps per CTA
    uint32_t K, R;  // skew r = R / K, 0 <= R < K
};

// Plan record (warp) of a unit whose weight midpoint is mid2 / 2 on a stream of total2 / 2:
// the CTA whose cumulative share C(c) = K (G-1) c + R c (G-c) (of T = K G (G-1)) contains it, then
// the warp of equal sub-shares.  Exact integer arithmetic, shared by the host and device builders;
// with R = 0 it is floor(mid2 W / total2), W = G A.
__host__ __device__ inline uint64_t plan_warp_of(unsigned __int128 mid2, unsigned __int128 total2, const PlanGrid& g) {
    const uint64_t W = (uint64_t)g.G * g.A;
    if (g.R == 0 || g.G < 2) {
        const uint64_t k = (uint64_t)(mid2 * W / total2);
        return k < W ? k : W - 1;
    }
    const uint64_t Gm = g.G - 1;
    const unsigned __int128 T = (unsigned __int128)g.K * g.G * Gm;
    const unsigned __int128 pos = mid2 * T;  // compared with C(c) total2
    uint32_t lo = 0, hi = g.G - 1;
    while (lo < hi) {  // largest c with C(c) total2 <= pos
        const uint32_t mid = (lo + hi + 1) / 2;
        const unsigned __int128 C = (unsigned __int128)g.K * Gm * mid + (unsigned __int128)g.R * mid * (g.G - mid);
        if (C * total2 <= pos)
            lo = mid;
        else
            hi = mid - 1;
    }
    const uint32_t c = lo;
    const unsigned __int128 Cc = (unsigned __int128)g.K * Gm * c + (unsigned __int128)g.R * c * (g.G - c);
    // K (G-1) + R (G-1-2c), kept non-negative term by term (R < K)
    const unsigned __int128 wc = (unsigned __int128)(g.K + g.R) * Gm - 2ull * (unsigned __int128)g.R * c;
    const unsigned __int128 rem = pos - Cc * total2;
    uint64_t warp = (uint64_t)(rem * g.A / (wc * total2));
    if (warp >= g.A) warp = g.A - 1;
    return (uint64_t)c * g.A + warp;
}

inline uint64_t plan_unit_bound(uint64_t rows, uint64_t pad_nnz) { return 2 * rows + pad_nnz / kUnitElts + 16; }

// Fills recs[W], splits[<= W] and *d_totals; stream-ordered, no host synchronisation.
cudaError_t plan_build_device(const uint32_t* rp, uint32_t rows, uint32_t pad_nnz, const PlanGrid& grid, uint64_t ubound,
                              int sms, uint32_t row_weight, const PlanTemp& t, WarpPlan* recs, uint4* splits,
                              PlanTotals* d_totals, cudaStream_t s);

}  // namespace mk
