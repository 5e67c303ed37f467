// common.cuh — device helpers shared by the MACKO sm_100a kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mk {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xFFFFFFFFu;

// One SpMV step = 32 lanes x 8 elements (512 B of values + 128 B of 4-bit
// deltas per warp).  A "unit" is kUnitSteps steps; lane accumulators are tree-reduced once per
// unit and unit sums are added sequentially into the row sum.
constexpr int kEltsPerLane = 8;
constexpr int kStepElts = kWarp * kEltsPerLane;  // 256
// 16 steps (4096 elements): fewer split rows (a row of up to 31 steps is one unit, so a warp
// boundary never cuts it) and half the xor-tree reductions of 8-step units.  Measured (amortised
// timing, one B200): 36864x12288 @50 % 107.1 vs 111.1 us, 4096x11008 18.8 vs 22.7 us,
// 131072x32768 @50 % 1022-1026 vs 1056 us, decode chain 2196 vs 2286 us / token; 4 steps was
// slower everywhere (chain 2586), 24-64 lose on 131072x32768 (1092-1100 us).
#ifndef MACKO_UNIT_STEPS
#define MACKO_UNIT_STEPS 16
#endif
constexpr int kUnitSteps = MACKO_UNIT_STEPS;  // build knob for experiments (the oracle takes it as a parameter)
constexpr int kUnitElts = kStepElts * kUnitSteps;  // 4096

// ---- streaming loads (read-once data: no L1 allocation) ----
__device__ __forceinline__ uint4 ldg_stream_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ldg_stream_u32(const void* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// acc += a*b with a, b fp16 and acc fp32 (single rounding; the f16xf16 product is exact in
// fp32, so this equals the reference's fp32 multiply-then-add).  SASS: FHFMA.
__device__ __forceinline__ float fma_f16f16f32(uint16_t a, uint16_t b, float acc) {
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(a), "h"(b));
    return acc;
}

__device__ __forceinline__ uint16_t f32_to_f16_rn(float v) {
    return __half_as_ushort(__float2half_rn(v));
}

// Inclusive warp scan (Algorithm 1 structure).
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int off = 1; off < kWarp; off <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, v, off);
        if (lane >= off) v += t;
    }
    return v;
}

// Same scan with the shuffle's in-range predicate driving a predicated add (2 SASS per level).
__device__ __forceinline__ uint32_t warp_incl_scan_p(uint32_t v) {
    asm("{\n\t.reg .u32 t;\n\t.reg .pred p;\n\t"
        "shfl.sync.up.b32 t|p, %0, 1, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
        "shfl.sync.up.b32 t|p, %0, 2, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
        "shfl.sync.up.b32 t|p, %0, 4, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
        "shfl.sync.up.b32 t|p, %0, 8, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t"
        "shfl.sync.up.b32 t|p, %0, 16, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t}"
        : "+r"(v));
    return v;
}

// xor-butterfly sum; every lane ends with identical bits (oracle lane_tree()).
__device__ __forceinline__ float warp_tree_sum(float v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
}

// ---- counter-hash generator (oracle/macko_oracle.c mix64 / mo_gen_value) ----
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint16_t gen_value(uint64_t seed, uint64_t idx, uint32_t thr24, int int_mode) {
    const uint64_t h = mix64(seed ^ (idx * 0xD1B54A32D192ED03ull));
    if ((uint32_t)(h >> 40) >= thr24) return 0;
    if (int_mode) {
        int v = (int)(h & 15u) - 8;
        if (v >= 0) v += 1;
        return f32_to_f16_rn((float)v);
    }
    uint32_t u = (uint32_t)(h & 0xFFFFu);
    if (u == 32768u) u = 32769u;
    return f32_to_f16_rn((float)((int32_t)u - 32768) * (1.0f / 32768.0f));
}

__device__ __forceinline__ uint16_t gen_vector_value(uint64_t seed, uint64_t i, int int_mode) {
    const uint64_t h = mix64(seed ^ (i * 0xD1B54A32D192ED03ull));
    if (int_mode) return f32_to_f16_rn((float)((int)((h & 0xFFFFu) % 17u) - 8));
    return f32_to_f16_rn((float)((int32_t)(h & 0xFFFFu) - 32768) * (1.0f / 32768.0f));
}

}  // namespace mk
