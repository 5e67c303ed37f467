// spmv.cuh — declarations shared by the SpMV kernel (spmv.cu) and the host runtime (capi.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mk {

// Static work plan of one matrix (built once on the host by build_plan in capi.cu, kept on the
// device).  The element stream of the matrix is cut into units of kUnitSteps warp steps per
// row; each warp ("chunk") owns a contiguous range of units of roughly equal weight.
struct SpmvPlanDev {
    const uint32_t* chunk_unit;     // W+1: first global unit of chunk w
    const uint32_t* chunk_row;      // W:   row of that unit
    const uint32_t* chunk_j;        // W:   unit index of that unit inside its row
    const uint32_t* chunk_e;        // 2W:  [first, end) element of the chunk's stream (TMA range)
    const int32_t* chunk_colbase;   // W:   decoded column just before that unit (-1 if j == 0)
    const int32_t* chunk_sid;       // 2W:  split-row id of the chunk's first / last row, or -1
    const uint32_t* split_slot;     // S:   first partial slot of split row s
    const uint32_t* split_first;    // S:   units handled by the row's first piece
    const uint32_t* split_pieces;   // S:   number of chunks touching the row
    float* partials;                // per split row, one slot per unit
    uint32_t* counters;             // S:   arrival counters (zero between launches)
};

struct SpmvArgs {
    const uint16_t* values;
    const uint8_t* deltas;
    const uint32_t* row_ptrs;
    const uint16_t* x;
    uint16_t* y;
    uint64_t value_elems, delta_bytes;  // allocated payload sizes (TMA clamp)
    uint32_t rows, cols;
    uint32_t ring;         // TMA ring slots per warp (power of two, 2..kMaxRing)
    uint32_t ring_offset;  // byte offset of the rings in dynamic shared memory (after x)
    SpmvPlanDev plan;
};

constexpr int kSpmvWarpsPerCta = 32;          // one persistent 1024-thread CTA per SM
constexpr uint32_t kChunk = 1024;             // elements per TMA chunk (two step pairs)
constexpr uint32_t kChunkVBytes = 2 * kChunk; // 2 KiB of values
constexpr uint32_t kChunkDBytes = kChunk / 2; // 512 B of 4-bit deltas
constexpr uint32_t kMaxRing = 8;

// Launchers (return cudaGetLastError()).
// x_mode: 0 = x gathered from global (L1), 1 = fp16 table in smem, 2 = (x[c], x[c+1]) pair table
cudaError_t launch_spmv(const SpmvArgs& a, int grid, int x_mode, size_t smem, cudaStream_t s);
cudaError_t spmv_occupancy(int x_mode, size_t smem, int* ctas_per_sm);
cudaError_t launch_plan_colbase(const uint8_t* deltas, const uint32_t* row_ptrs, const uint32_t* chunk_row,
                                const uint32_t* chunk_j, int32_t* chunk_colbase, uint32_t n_chunks,
                                cudaStream_t s);

}  // namespace mk
