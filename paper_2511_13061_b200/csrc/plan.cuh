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

inline uint64_t plan_unit_bound(uint64_t rows, uint64_t pad_nnz) { return 2 * rows + pad_nnz / kUnitElts + 16; }

// Fills recs[W], splits[<= W] and *d_totals; stream-ordered, no host synchronisation.
cudaError_t plan_build_device(const uint32_t* rp, uint32_t rows, uint32_t pad_nnz, uint32_t W, uint64_t ubound, int sms,
                              uint32_t row_weight, const PlanTemp& t, WarpPlan* recs, uint4* splits, PlanTotals* d_totals,
                              cudaStream_t s);

}  // namespace mk
