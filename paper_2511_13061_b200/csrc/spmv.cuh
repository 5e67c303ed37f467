// spmv.cuh — declarations shared by the SpMV kernel (spmv.cu) and the host runtime (capi.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mk {

// Static work plan of one matrix (built once on the host by build_plan in capi.cu, kept on the
// device).  The element stream of the matrix is cut into units of kUnitSteps warp steps per row
// (the last unit of a row absorbs a remainder shorter than a unit); each warp ("chunk") owns a
// contiguous range of units of roughly equal weight.  Everything a warp needs to start is in one
// 48-byte record, so its prologue is a single memory round trip.
struct WarpPlan {
    uint32_t units_left;   // units in the chunk (0 = idle warp)
    uint32_t row, j;       // first unit: its row and its unit index inside the row
    uint32_t e0, e1;       // [first, end) element of the chunk's TMA stream
    uint32_t s, e;         // row_ptrs[row], row_ptrs[row + 1]
    int32_t colbase;       // decoded column just before unit j (-1 if j == 0; set on the device)
    int32_t sid0, sid1;    // split-row id of the chunk's first / last row piece, or -1
    uint32_t slot0, slot1; // first partial slot of those split rows
};
static_assert(sizeof(WarpPlan) == 48, "WarpPlan is loaded as three 16-byte vectors");

struct SpmvPlanDev {
    const WarpPlan* warps;   // W records
    const uint4* splits;     // S: {first partial slot, units of the first piece, pieces, 0}
    // Per-launch workspace (one per stream, capi.cu Workspace): launches of one matrix on different
    // streams never share these.
    float* partials;         // per split row, one slot per unit
    uint32_t* counters;      // S: arrival counters (zero between launches)
};

// Fused all-gather of y (row-sharded SpMV over NVLink peers): up to kMaxPeers destinations.
constexpr uint32_t kMaxPeers = 8;
struct PeerTable {  // host side, one per matrix (macko_dev_set_peers / macko_dev_set_peer_bank)
    uint16_t* y[2][kMaxPeers]; // bank b: peer p's full y, already offset to this slab's first row
    uint32_t* flag[kMaxPeers]; // this rank's completion counter in peer p's flag array
};

struct SpmvArgs {
    const uint16_t* values;
    const uint8_t* deltas;
    const uint32_t* row_ptrs;
    const uint16_t* x;
    uint16_t* y;
    cudaTextureObject_t xtex;           // x as a 1-D fp16 texture (x_mode 0, 6, 7, 8, 10)
    uint64_t value_elems, delta_bytes;  // allocated sizes (payload + one zeroed chunk of slack)
    uint32_t value_count;               // pad_nnz
    uint32_t rows, cols;
    uint32_t ring;         // TMA ring slots per warp (always kMaxRing; the kernel uses the constant)
    uint32_t ring_offset;  // byte offset of the rings in dynamic shared memory (after x)
    uint32_t pdl;          // launched as a PDL dependent: x may still be written by the producer
    uint32_t n_peer;       // fused all-gather: y rows also go to peer_y[0..n_peer) and each CTA adds 1
                           // to *peer_flag[p] (system scope) once its rows are written
    // The launch's bank of the peer table, in the parameter bank: every warp reads the pointers at
    // its end, and 4736 warps loading one global word at once serialise on its L2 line (+10 us).
    uint16_t* peer_y[kMaxPeers];
    uint32_t* peer_flag[kMaxPeers];
    uint32_t no_split;     // the plan has no split rows (PDL launches use the kNoSplit instance)
    uint16_t* y_mirror;    // host-buffer SpMV: y rows also stored straight into the mapped host y
    uint32_t batch;        // SpMM: vectors in the batch (<= the kernel's kB); x = XT interleaved
    uint64_t ldy;          // SpMM: element stride between the batch's y vectors
    uint32_t warps_active; // warps per CTA that own a plan record (the rest only stage x); record of
                           // warp k of CTA c: c * warps_active + k
    uint32_t trace_slot;   // trace builds only (MACKO_TRACE): which of the kept launches this is
    SpmvPlanDev plan;
};

#ifndef MACKO_WARPS_PER_CTA
#define MACKO_WARPS_PER_CTA 32
#endif
// kSpmvCtasPerSm persistent CTAs of kSpmvWarpsPerCta warps per SM (32 warps per SM either way).
// Measured: two 16-warp CTAs per SM (so the next SpMV of a PDL chain can start on half an SM) are
// 8 % slower on 36864x12288 and no faster on the decode chain; one 32-warp CTA is the default.
#ifndef MACKO_WARPS_PER_SM
#define MACKO_WARPS_PER_SM 32
#endif
constexpr int kSpmvWarpsPerCta = MACKO_WARPS_PER_CTA;
constexpr int kSpmvCtasPerSm = MACKO_WARPS_PER_SM / kSpmvWarpsPerCta;
#ifndef MACKO_CHUNK
#define MACKO_CHUNK 1024
#endif
constexpr uint32_t kChunk = MACKO_CHUNK;      // elements per TMA chunk (two step pairs)
constexpr uint32_t kChunkVBytes = 2 * kChunk; // 2 KiB of values
constexpr uint32_t kChunkDBytes = kChunk / 2; // 512 B of 4-bit deltas (b_delta = 4; kChunk * b / 8 in general)
// TMA ring slots per warp, a compile-time power of two: two 1024-element chunks (5 KiB at b_delta
// = 4) per warp, 160 KiB per SM; four would not fit beside the x table for any b_delta.
#ifndef MACKO_MAX_RING
#define MACKO_MAX_RING 2
#endif
constexpr uint32_t kMaxRing = MACKO_MAX_RING;
static_assert(kMaxRing >= 2 && (kMaxRing & (kMaxRing - 1)) == 0, "ring slots: a power of two >= 2");
// fp16 x table in shared memory with zero guards: kXGuardLo entries before x[0] (the ROMA-masked
// elements of a row's first step decode to columns -7..-1) and kXGuardHi after x[C-1] (a phantom
// step past the row end is pointed at column C, its elements land on C+1..C+8).
constexpr int kXGuardLo = 8;
constexpr int kXGuardHi = 16;

// Launchers (return cudaGetLastError()).
// x_mode: 0 = texture gathers only, 1 = fp16 shared-memory table only, 6 / 7 / 8 / 10 = table +
// texture gathers for a fixed subset of element slots (TEX pipe in parallel with the LSU pipe)
bool spmv_valid_x_mode(int x_mode);
#ifdef MACKO_TRACE
cudaError_t trace_read(unsigned long long* host, size_t n);  // trace build only
#endif
// pdl: launch with programmatic stream serialization (overlaps the previous kernel's tail)
cudaError_t launch_spmv(const SpmvArgs& a, int bits, int grid, int x_mode, size_t smem, cudaStream_t s, bool pdl);
// Small-batch SpMM over a b_delta = 4 matrix: kb in {2, 4, 8}, x_mode 0 (texture) or 7 (split);
// a.x is the interleaved XT (launch_interleave), a.xtex a texture of 2 kb-byte texels over it.
cudaError_t launch_spmm(const SpmvArgs& a, int kb, int grid, int x_mode, size_t smem, cudaStream_t s);
bool spmm_valid_x_mode(int x_mode);  // 0 (texture), 1 (table), 6 / 7 / 8 (split)
cudaError_t launch_interleave(const uint16_t* X, uint64_t ldx, uint32_t batch, uint32_t kb, uint32_t cols,
                              uint16_t* XT, uint32_t n_total, cudaStream_t s);
constexpr uint32_t kMaxBatch = 8;
cudaError_t spmv_occupancy(int x_mode, int bits, size_t smem, int* ctas_per_sm);
// Static shared memory of the SpMV kernels (mbarriers, fused all-gather stash); 0 on error.
size_t spmv_static_smem();
bool spmv_valid_config(int x_mode, int bits);
// Wait until flags[i] >= target for i < n (system-scope acquire; peers' fused all-gathers).
cudaError_t launch_wait_flags(const uint32_t* flags, uint32_t n, uint32_t target, cudaStream_t s);
// n fp16 words src -> dst (device or device-mapped host pointers); dependent: launched as the
// programmatic dependent of the previous kernel on the stream (waits for it before copying).
cudaError_t launch_copy_u16(const uint16_t* src, uint16_t* dst, uint32_t n, int blocks, bool dependent, cudaStream_t s);
cudaError_t launch_plan_colbase(const uint8_t* deltas, uint32_t bits, WarpPlan* warps, uint32_t n_chunks, cudaStream_t s);

}  // namespace mk
