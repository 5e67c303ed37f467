// spmv.cu — MACKO SpMV for sm_100a (b_delta 1/2/4/8, fp16 values, fp32 accumulation).
//
// Realises the paper's warp kernel (SPEC.md:255-264 warp_spmv) natively:
//   * one warp walks a row in steps of 256 elements, lane l owning elements 8l..8l+7 of the
//     step;
//   * ROMA: the row start is aligned down to 8 elements; elements outside
//     the row (before its start in the first step, past its end in the last) are masked;
//   * column reconstruction: the codewords are widened to bytes, paired and prefix-summed with
//     one integer multiply (byte-SIMD), then Algorithm 1's shfl_up scan gives the lane offset
//     and the warp total advances the running column.  Two steps share one
//     scan (their lane sums packed into 16-bit halves); the total comes from REDUX;
//   * every element's x value is gathered and multiply-added with FHFMA (fp16 x fp16 -> fp32
//     accumulate, exact product).
// B200 specifics (profiles/r01_pipes.md, r01_experiments.md): the kernel is bound by the L1TEX
// data pipes and the latency of each warp's pair chain, not by HBM.
//   * The matrix stream arrives by TMA: every warp owns a contiguous element range (static
//     equal-weight plan of 4096-element units, built once per matrix) and keeps a ring of
//     1024-element chunks in flight with cp.async.bulk + mbarrier (no LSU wavefronts; issued by
//     one elect.sync lane, L2 evict_first); values and codewords are read back with one LDS.128
//     + one LDS per lane step.
//   * x gathers are split between two pipes that run in parallel: an fp16 copy of x in shared
//     memory (LDS, LSU pipe) and x as a 1-D texture (TEX pipe, L1-resident); which of a lane's
//     8 element slots use the texture is a compile-time mask (x_mode).
//   * Row edges (a row's first and last step pair) run the interior code with predication: the
//     ROMA head gets codeword 0 (delta 1, so the scan stays exact), and every element outside
//     the row skips its gather and FHFMA, so nothing outside the row reaches the sum, not even
//     0 * inf.
//   * One persistent CTA of 32 warps per SM.  Rows cut between warps are finished by the
//     last-arriving warp, which adds the per-unit partials in unit order.
// Summation order (every run, any grid): per lane sequential over its elements, xor-tree over
// lanes once per unit (kUnitSteps = 16 steps; the row's last unit absorbs a shorter remainder), sequential
// over units — mirrored bit-exactly by oracle mo_b200_order_spmv(unit_steps = kUnitSteps).  It
// depends on a row's elements and on its start offset mod 8 (ROMA), never on the plan.
#include "common.cuh"
#include "spmv.cuh"

#include <type_traits>

#ifdef MACKO_TRACE
// Opt-in trace build (`make trace` -> libmacko_cuda_trace.so): per warp, %globaltimer at each
// prologue phase and at the end, for latency studies of small SpMVs (tools/trace_spmv.py).
// kTraceSlots launches are kept (SpmvArgs::trace_slot, set by the host round robin), so a chain
// of SpMVs can be traced op by op (tools/trace_chain.py).
constexpr int kTraceSlots = 8;
__device__ unsigned long long g_macko_trace[kTraceSlots * 148 * 32 * 8];
#define MK_TRACE(i)                                                                                    \
    do {                                                                                                \
        if ((threadIdx.x & 31) == 0 && blockIdx.x < 148) {                                              \
            unsigned long long t_;                                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
            g_macko_trace[((a.trace_slot % kTraceSlots) * 148 * 32 + blockIdx.x * 32 + (threadIdx.x >> 5)) * 8 + (i)] = t_; \
        }                                                                                               \
    } while (0)
#else
#define MK_TRACE(i) \
    do {            \
    } while (0)
#endif

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

__device__ __forceinline__ uint16_t xtex(cudaTextureObject_t t, int col) {
    return tex1Dfetch<unsigned short>(t, col);
}

// Lane element slots k (0..7) gathered through the texture (bit k set) rather than the shared
// table.  x_mode 0: texture only (x too large for shared memory); 1: shared table only;
// 6, 7, 8, 10: split between the LSU and TEX data pipes (profiles/r01_pipes.md).
template <int kXMode>
constexpr uint32_t tex_slots() {
    return kXMode == 0 ? 0xFFu : kXMode == 6 ? 0x2Au : kXMode == 7 ? 0xAAu : kXMode == 8 ? 0x22u : kXMode == 10 ? 0xAAu : 0u;
}

// Second step of a pair: x_mode 10 alternates 4 and 3 texture slots between the two steps
// (3.5 of 8 on average).
template <int kXMode>
constexpr uint32_t tex_slots_b() {
    return kXMode == 10 ? 0x2Au : tex_slots<kXMode>();
}

template <int kXMode>
constexpr bool x_table() {
    return kXMode != 0;
}

template <int kBits>
constexpr uint32_t dbytes() {  // delta bytes of one kChunk-element chunk
    return kChunk * kBits / 8;
}

struct Dec {
    uint32_t even, odd, local;  // in-lane inclusive column offsets of elements 0,2,4,6 / 1,3,5,7; lane total
};

// b_delta <= 4: codewords -> byte deltas (codeword + 1) -> in-lane inclusive prefixes (byte m of
// even/odd; at most 8 x 16 = 128, so bytes never carry).  Nibbles (b = 4) are split directly;
// crumbs (b = 2) are first spread to one nibble per byte, bits (b = 1) to one per byte.
template <int kBits>
__device__ __forceinline__ Dec decode(uint32_t d) {
    uint32_t dl, dh;
    if constexpr (kBits == 4) {
        dl = (d & 0x0F0F0F0Fu) + 0x01010101u;         // elements 0,2,4,6
        dh = ((d >> 4) & 0x0F0F0F0Fu) + 0x01010101u;  // elements 1,3,5,7
    } else if constexpr (kBits == 2) {
        uint32_t nib;  // byte m = crumbs of elements 2m (bits 0-1) and 2m+1 (bits 2-3)
        asm("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(nib) : "r"(d & 0x0F0Fu), "r"((d >> 4) & 0x0F0Fu));
        dl = (nib & 0x03030303u) + 0x01010101u;
        dh = ((nib >> 2) & 0x03030303u) + 0x01010101u;
    } else {  // kBits == 1: bit k = element k
        dl = (((d & 0x55u) * 0x41041u) & 0x01010101u) + 0x01010101u;
        dh = ((((d >> 1) & 0x55u) * 0x41041u) & 0x01010101u) + 0x01010101u;
    }
    const uint32_t pp = (dl + dh) * 0x01010101u;
    return Dec{pp - dh, pp, pp >> 24};
}

// b_delta = 8: byte codewords, deltas up to 256, so prefixes (up to 2048) live in 16-bit halves:
// p[j] = (offset of element 2j, offset of element 2j+1).
struct Dec8 {
    uint32_t p[4];
    uint32_t local;
};

__device__ __forceinline__ Dec8 decode8(uint32_t w0, uint32_t w1) {
    Dec8 r;
    uint32_t h[4];
    asm("prmt.b32 %0, %1, 0, 0x4140;" : "=r"(h[0]) : "r"(w0));
    asm("prmt.b32 %0, %1, 0, 0x4342;" : "=r"(h[1]) : "r"(w0));
    asm("prmt.b32 %0, %1, 0, 0x4140;" : "=r"(h[2]) : "r"(w1));
    asm("prmt.b32 %0, %1, 0, 0x4342;" : "=r"(h[3]) : "r"(w1));
    uint32_t carry = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t q = h[j] + 0x00010001u;         // (delta 2j, delta 2j+1)
        r.p[j] = q + (q << 16) + carry * 0x00010001u;  // inclusive prefixes
        carry = r.p[j] >> 16;
    }
    r.local = carry;
    return r;
}

#ifdef MACKO_OPAQUE_SEL
__device__ __forceinline__ uint32_t opaque(uint32_t v) {
    asm("mov.b32 %0, %0;" : "+r"(v));
    return v;
}
#else
__device__ __forceinline__ uint32_t opaque(uint32_t v) { return v; }
#endif

#ifdef MACKO_CONST_SEL
// dp4a byte selectors k << 8m (k = 1, 2) in the constant bank, so IDP.4A reads them as c[3][...]
// operands instead of re-materialising uniform registers every step pair.
__constant__ uint32_t c_sel[2][4] = {{1u, 1u << 8, 1u << 16, 1u << 24}, {2u, 2u << 8, 2u << 16, 2u << 24}};
#define MK_SEL(k, m) c_sel[(k) - 1][m]
#else
#define MK_SEL(k, m) opaque((uint32_t)(k) << (8 * (m)))
#endif

// c + (byte-wise dot product of a and sel): with one non-zero selector byte, c + k * byte m of a.
__device__ __forceinline__ uint32_t dp4a_sel(uint32_t a, uint32_t sel, uint32_t c) {
    uint32_t d;
    asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(sel), "r"(c));
    return d;
}

// 8 gathers + FHFMAs of one lane step.  cb = column before the lane's first element.  Masked
// steps (row edges): element m gathers and accumulates only if bit m of vm is set (predicated
// gather and FHFMA), so nothing outside the row reaches the sum, not even 0 * inf.  Skipping
// equals adding +0 here: a lane sum that starts at +0 never becomes -0.
template <int kXMode, bool kMasked, uint32_t kTex = tex_slots<kXMode>(), class D>
__device__ __forceinline__ float lane_step(float acc, const uint4& v, const D& dc, int cb, uint32_t xs_addr,
                                           cudaTextureObject_t xt, uint32_t vm) {
#ifdef MACKO_EXP_NO_GATHER  // experiment builds only (tools/build_variant.sh): the walk without x gathers
    return acc + __int_as_float((int)((v.x ^ v.w ^ (uint32_t)cb) & 0x3FFu));
#endif
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    // shared address of column cb: per element one PRMT (offset extract) + one IADD3
    uint32_t base = xs_addr + 2u * (uint32_t)cb;
    asm("mov.b32 %0, %0;" : "+r"(base));  // opaque: keeps base + 2b a single IADD3 per element
    uint32_t even2 = 0;
    if constexpr (!std::is_same<D, Dec8>::value && (kTex & 0x55u) != 0x55u) even2 = dc.even * 2u;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        uint16_t v0, v1;
        split_halves(w[m], v0, v1);
        uint32_t b0, b1;
#ifndef MACKO_NO_DP4A
        if constexpr (!std::is_same<D, Dec8>::value) {
            // one IDP.4A per element: the byte-m prefix times 1 (TEX coordinate) or 2 (shared
            // address) plus the base, instead of a PRMT extract and an add
            // Even elements gather from shared memory in every x_mode but 0: their offsets are
            // pre-doubled (2 x 112 < 256), so they share the TEX elements' selectors.
            const bool t0 = (kTex >> (2 * m)) & 1u, t1 = (kTex >> (2 * m + 1)) & 1u;
            const uint32_t a0 = t0 ? dp4a_sel(dc.even, MK_SEL(1, m), (uint32_t)cb) : dp4a_sel(even2, MK_SEL(1, m), base);
            const uint32_t a1 = dp4a_sel(dc.odd, MK_SEL(t1 ? 1 : 2, m), t1 ? (uint32_t)cb : base);
            if (!kMasked || ((vm >> (2 * m)) & 1u)) acc = fma_f16f16f32(v0, t0 ? xtex(xt, (int)a0) : lds_u16(a0), acc);
            if (!kMasked || ((vm >> (2 * m + 1)) & 1u)) acc = fma_f16f16f32(v1, t1 ? xtex(xt, (int)a1) : lds_u16(a1), acc);
            continue;
        }
#endif
        if constexpr (std::is_same<D, Dec8>::value) {
            b0 = __byte_perm(dc.p[m], 0u, 0x4410u);
            b1 = __byte_perm(dc.p[m], 0u, 0x4432u);
        } else {
            b0 = __byte_perm(dc.even, 0u, 0x4440u + m);
            b1 = __byte_perm(dc.odd, 0u, 0x4440u + m);
        }
        if (!kMasked || ((vm >> (2 * m)) & 1u))
            acc = fma_f16f16f32(v0, ((kTex >> (2 * m)) & 1u) ? xtex(xt, cb + (int)b0) : lds_u16(base + 2u * b0), acc);
        if (!kMasked || ((vm >> (2 * m + 1)) & 1u))
            acc = fma_f16f16f32(v1, ((kTex >> (2 * m + 1)) & 1u) ? xtex(xt, cb + (int)b1) : lds_u16(base + 2u * b1), acc);
    }
    return acc;
}

// Batched lane step (SpMM, kB vectors): x is interleaved per column (kB fp16 = 2 kB bytes per
// column, XT[c][b]), so one gather fetches all kB values of a column — one TLD of a 32 / 64 / 128-bit
// texel or one LDS.32 / .64 / .128 — and kB FHFMAs take its halves.  Column b's summation order is
// exactly the SpMV's (the same element -> lane -> unit structure), so Y[b] == SpMV(X[b]) bit for bit.
template <int kB>
struct XVec {
    uint32_t w[kB / 2];
};

template <int kB>
__device__ __forceinline__ XVec<kB> xtex_b(cudaTextureObject_t t, int col) {
    XVec<kB> r;
    if constexpr (kB == 2) {
        r.w[0] = tex1Dfetch<unsigned int>(t, col);
    } else if constexpr (kB == 4) {
        const uint2 q = tex1Dfetch<uint2>(t, col);
        r.w[0] = q.x;
        r.w[1] = q.y;
    } else {
        const uint4 q = tex1Dfetch<uint4>(t, col);
        r.w[0] = q.x;
        r.w[1] = q.y;
        r.w[2] = q.z;
        r.w[3] = q.w;
    }
    return r;
}

template <int kB>
__device__ __forceinline__ XVec<kB> lds_b(uint32_t addr) {
    XVec<kB> r;
    if constexpr (kB == 2) {
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(r.w[0]) : "r"(addr));
    } else if constexpr (kB == 4) {
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(r.w[0]), "=r"(r.w[1]) : "r"(addr));
    } else {
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
                     : "r"(addr));
    }
    return r;
}

template <int kB>
__device__ __forceinline__ void fma_b(float (&acc)[kB], uint16_t v, const XVec<kB>& x) {
#pragma unroll
    for (int q = 0; q < kB / 2; ++q) {
        uint16_t lo, hi;
        split_halves(x.w[q], lo, hi);
        acc[2 * q] = fma_f16f16f32(v, lo, acc[2 * q]);
        acc[2 * q + 1] = fma_f16f16f32(v, hi, acc[2 * q + 1]);
    }
}

template <int kXMode, bool kMasked, int kB, uint32_t kTex = tex_slots<kXMode>(), class D>
__device__ __forceinline__ void lane_step_b(float (&acc)[kB], const uint4& v, const D& dc, int cb, uint32_t xs_addr,
                                            cudaTextureObject_t xt, uint32_t vm) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t base = xs_addr + 2u * kB * (uint32_t)cb;
    asm("mov.b32 %0, %0;" : "+r"(base));
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        uint16_t v0, v1;
        split_halves(w[m], v0, v1);
        const uint32_t b0 = __byte_perm(dc.even, 0u, 0x4440u + m);
        const uint32_t b1 = __byte_perm(dc.odd, 0u, 0x4440u + m);
        if (!kMasked || ((vm >> (2 * m)) & 1u))
            fma_b<kB>(acc, v0, ((kTex >> (2 * m)) & 1u) ? xtex_b<kB>(xt, cb + (int)b0) : lds_b<kB>(base + 2u * kB * b0));
        if (!kMasked || ((vm >> (2 * m + 1)) & 1u))
            fma_b<kB>(acc, v1, ((kTex >> (2 * m + 1)) & 1u) ? xtex_b<kB>(xt, cb + (int)b1) : lds_b<kB>(base + 2u * kB * b1));
    }
}

// y[r] = v (lane 0).  Fused all-gather: a split row's last arrival may sit in another CTA than the
// warps around it, so it stores its 2 bytes straight into every peer's y (kDirect); every other
// row belongs to the warp that walked it and reaches the peers through the warp's stash
// (own_row_put).
// kMirror: the plain instance also serves the host-buffer path (y_mirror); the chain and peers
// instances carry no mirror code (chain 2172 -> 2151 us per token without it).
template <bool kDirect, bool kMirror>
__device__ __forceinline__ void put_y(const SpmvArgs& a, uint32_t r, uint16_t v) {
    a.y[r] = v;
    if constexpr (kMirror)
        if (a.y_mirror) a.y_mirror[r] = v;
    if constexpr (kDirect)
        for (uint32_t p = 0; p < a.n_peer; ++p) a.peer_y[p][r] = v;
}

// Fused all-gather of the rows a warp finishes alone (its whole rows and empty rows): lane 0 parks
// y[r] in the warp's 16-row stash (slot r mod 16) and the warp stores a full group of 16 rows to
// every other rank's y with one 32-byte store per peer (round 1: one 2-byte NVLink write per row
// per peer).  s_own_first: the warp's first own row (its first row unless that one is split).
// The stash, not a re-read of y: loading just-written y lines (written by many SMs at once) cost
// 10 us per launch at 4096x4096.  Only the peers instance of the kernel carries it (1 KiB).
constexpr uint32_t kOwnGroup = 16;
__shared__ uint16_t s_own_y[kSpmvWarpsPerCta][kOwnGroup];
__shared__ uint32_t s_own_first[kSpmvWarpsPerCta];

// Store the stashed own rows of [lo, hi) (one group) to the peers (whole warp).
__device__ __forceinline__ void flush_own(const SpmvArgs& a, uint32_t lo, uint32_t hi, int lane) {
    const uint32_t warp = threadIdx.x >> 5;
    __syncwarp();  // lane 0's stash writes
    const uint32_t r = lo + (uint32_t)lane;
    if (lane < (int)kOwnGroup && r >= s_own_first[warp] && r < hi) {
        const uint16_t v = s_own_y[warp][r & (kOwnGroup - 1)];
        for (uint32_t p = 0; p < a.n_peer; ++p)
            if (a.peer_y[p] != a.y) a.peer_y[p][r] = v;
    }
    __syncwarp();  // before the slots are reused
}

// Row r (own, y[r] = v in lane 0) is done: stash it; a full group goes out (whole warp).
__device__ __forceinline__ void own_row_put(const SpmvArgs& a, uint32_t r, uint16_t v, int lane) {
    if (lane == 0) s_own_y[threadIdx.x >> 5][r & (kOwnGroup - 1)] = v;
    if ((r & (kOwnGroup - 1)) == kOwnGroup - 1) flush_own(a, r + 1 - kOwnGroup, r + 1, lane);
}

// Batched outputs (SpMM): Y[b][r] for b < a.batch (Y rows ldy apart).
template <int kB, bool kDirect, bool kMirror>
__device__ __forceinline__ void put_y_b(const SpmvArgs& a, uint32_t r, const uint16_t (&v)[kB]) {
    if constexpr (kB == 1) {
        put_y<kDirect, kMirror>(a, r, v[0]);
    } else {
#pragma unroll
        for (int b = 0; b < kB; ++b)
            if ((uint32_t)b < a.batch) a.y[(size_t)b * a.ldy + r] = v[b];
    }
}

// Fused all-gather: once all warps of the CTA wrote their rows, make them visible system-wide and
// count the CTA in every peer's flag slot for this rank (consumers: wait_flags_kernel).
__device__ __forceinline__ void signal_peers(const SpmvArgs& a) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (uint32_t p = 0; p < a.n_peer; ++p) atomicAdd_system(a.peer_flag[p], 1u);
    }
}

// ------------------------------------------------------------------------------------------
// Compute-side row state
// ------------------------------------------------------------------------------------------
template <int kB>
struct RowState {
    uint32_t r, s, e, e_next, al, T, t, tend, j0, n_r, last_b, units_left, slot;
    int32_t sid;
    bool split;
    int col_base;
    float acc[kB], row_acc[kB];  // per lane / per row, one per vector of the batch
};

// Set up the piece of row rs.r = [rs.s, rs.e) starting at unit j0.  sid / slot: the chunk's
// split-row id for this piece (used only if the piece turns out to be split).
template <int kB>
__device__ __forceinline__ void begin_piece(RowState<kB>& rs, uint32_t j0, int colbase, int32_t sid, uint32_t slot) {
    // A row's first step starts at the 8-aligned al (ROMA); its k = s - al leading elements
    // belong to the previous row and are decoded as codeword 0 (delta 1) after masking, so the
    // column before the row is -1 - k (the masked elements sit at columns -k..-1).
    rs.al = rs.s & ~7u;
    rs.T = rs.e > rs.s ? (rs.e - rs.al + kStepElts - 1) / kStepElts : 0u;
    // units of kUnitSteps steps; the last unit absorbs a remainder shorter than a unit
    rs.n_r = rs.T >= (uint32_t)kUnitSteps ? rs.T / kUnitSteps : 1u;
    rs.last_b = (rs.n_r - 1u) * kUnitSteps;
    const uint32_t nu = min(rs.n_r - j0, rs.units_left);
    rs.units_left -= nu;
    rs.j0 = j0;
    rs.t = j0 * kUnitSteps;
    rs.tend = j0 + nu == rs.n_r ? rs.T : (j0 + nu) * kUnitSteps;
    rs.split = !(j0 == 0 && j0 + nu == rs.n_r);
    rs.sid = sid;
    rs.slot = slot;
    rs.col_base = j0 ? colbase : -1 - (int)(rs.s - rs.al);
#pragma unroll
    for (int b = 0; b < kB; ++b) {
        rs.acc[b] = 0.0f;
        rs.row_acc[b] = 0.0f;
    }
}

// Finish the current piece (write y or hand the split row to its last arrival).  Lane 0 wrote
// the piece's unit partials; the acq_rel arrival releases them and, for the last arrival,
// acquires every other piece's partials, which it then reads from L2 (ld.cg).
// Returns y[r]'s fp16 bits in lane 0 of the last arrival, -1 elsewhere (the caller stores it).
__device__ __noinline__ int finish_split(uint32_t j0, uint32_t tend, uint32_t n_r, uint32_t slot, int32_t sid,
                                         float row_acc, const SpmvPlanDev P, int lane) {
    uint32_t last = 0, first = 0;
    if (lane == 0) {
        if (j0 == 0) P.partials[slot + tend / kUnitSteps - 1u] = row_acc;  // a first piece ends on a unit boundary
        const uint4 sp = P.splits[sid];
        first = sp.y;
        uint32_t prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(P.counters + sid) : "memory");
        last = prev + 1 == sp.z;
    }
    last = __shfl_sync(kFull, last, 0);
    if (last && lane == 0) {
        float tot = __ldcg(P.partials + slot + first - 1);
        for (uint32_t q = first; q < n_r; ++q) tot += __ldcg(P.partials + slot + q);
        P.counters[sid] = 0;  // ready for the next launch (stream order)
        return (int)f32_to_f16_rn(tot);
    }
    return -1;
}

// finish_split for a batch: partial slot q of vector b at partials[(slot + q) kB + b].  Returns
// true in lane 0 of the last arrival with the rows' fp16 bits in out.
template <int kB>
__device__ __forceinline__ bool finish_split_b(uint32_t j0, uint32_t tend, uint32_t n_r, uint32_t slot, int32_t sid,
                                               const float (&row_acc)[kB], const SpmvPlanDev P, int lane,
                                               uint16_t (&out)[kB]) {
    uint32_t last = 0, first = 0;
    if (lane == 0) {
        if (j0 == 0) {  // a first piece ends on a unit boundary
#pragma unroll
            for (int b = 0; b < kB; ++b) P.partials[(size_t)(slot + tend / kUnitSteps - 1u) * kB + b] = row_acc[b];
        }
        const uint4 sp = P.splits[sid];
        first = sp.y;
        uint32_t prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(P.counters + sid) : "memory");
        last = prev + 1 == sp.z;
    }
    last = __shfl_sync(kFull, last, 0);
    if (last && lane == 0) {
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            float tot = __ldcg(P.partials + (size_t)(slot + first - 1) * kB + b);
            for (uint32_t q = first; q < n_r; ++q) tot += __ldcg(P.partials + (size_t)(slot + q) * kB + b);
            out[b] = f32_to_f16_rn(tot);
        }
        P.counters[sid] = 0;  // ready for the next launch (stream order)
        return true;
    }
    return false;
}

// Move to the next non-empty row piece of the chunk; empty rows get y = +0.  Returns false
// when the chunk is exhausted.  The row pointer after the next row is prefetched one row ahead.
template <int kB, bool kPeers, bool kMirror>
__device__ __forceinline__ bool next_piece(RowState<kB>& rs, const SpmvArgs& a, uint32_t w, int lane) {
    for (;;) {
        if (rs.units_left == 0) return false;
        ++rs.r;
        rs.s = rs.e;
        rs.e = rs.e_next;
        if (rs.r + 2u <= a.rows) rs.e_next = __ldg(a.row_ptrs + rs.r + 2u);
        begin_piece(rs, 0, -1, -1, 0);
        if (rs.split) {  // only the chunk's last row can be cut here: its split id is in the record
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(a.plan.warps + w) + 2);
            rs.sid = (int32_t)q.y;
            rs.slot = q.w;
        }
        if (rs.T) return true;
        if (lane == 0) {  // empty row: fp16(+0.0)
            const uint16_t z[kB] = {};
            put_y_b<kB, false, kMirror>(a, rs.r, z);
        }
        if constexpr (kPeers) own_row_put(a, rs.r, 0, lane);
    }
}

// ------------------------------------------------------------------------------------------
// Per-warp TMA ring of kChunk-element chunks (values 2 KiB + deltas 512 B per chunk).  The warp
// streams its contiguous element range through the ring with cp.async.bulk + mbarrier
// complete_tx; a slot is refilled (chunk k -> chunk k + ring) as soon as the walk has moved past
// chunk k.  The payload buffers carry one zeroed chunk of slack, so copies are never clamped.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}

__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t done;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(bar), "r"(parity)
                 : "memory");
    return done != 0;
}

// Wait for a TMA chunk.  A chunk that never lands (a bug, or a fault in the copy) traps after
// ~2 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try(bar, parity))
        if (clock64() - t0 > 4000000000LL) __trap();
}

// Chunk c of the warp's stream (elements [e0 + c kChunk, e0 + (c+1) kChunk)) lives in slot
// c & (ring - 1) and completes phase (c / ring) & 1 of that slot's mbarrier.  The walk position S
// only grows, by at most one step pair per pair, so at most one chunk is released per pair.
constexpr uint32_t kNever = 0xFFFFFFFFu;

#ifndef MACKO_EDGE_SPLIT
#define MACKO_EDGE_SPLIT 1
#endif
constexpr bool kEdgeSplit = MACKO_EDGE_SPLIT;  // 0: every edge pair masks both steps
// Edge step pairs (run_rows): which steps are masked, and whether the pair is a single step.
constexpr uint32_t kEdgeMaskA = 1u, kEdgeMaskB = 2u, kEdgeSingle = 4u;

struct Ring {
    uint32_t vbase, dbase, bar0;  // this warp's value ring, delta ring, first mbarrier (smem)
    uint32_t e0;                  // first element of the warp's chunk stream (chunk aligned)
    uint32_t emask;               // ring elements - 1 (power of two)
    uint32_t lane_rel;            // 8 lane - e0: the lane's element of a step at S sits at (S + lane_rel) & emask
    uint32_t n_chunks;            // chunks in the stream
    uint32_t released;            // chunks consumed and refilled (or nothing left to refill)
    uint32_t landed;              // chunks waited for
    uint32_t rel_at, wait_at;     // S thresholds of the next release / the next wait (kNever: none)
};

__device__ __forceinline__ uint32_t ring_ev(const Ring& g) { return min(g.rel_at, g.wait_at); }

// Refill slot (released & (ring-1)) with chunk released + ring (one elected lane; full-size copies,
// never clamped: the payload buffers carry a zeroed chunk of slack).  Called by the whole warp with
// warp-uniform operands: elect.sync inside the asm keeps the copies to one lane without a
// divergent branch around them.
template <int kBits>
__device__ __forceinline__ void ring_issue(const Ring& g, const SpmvArgs& a) {
    constexpr uint32_t ring = kMaxRing;
    const uint32_t slot = g.released & (ring - 1u);
    const uint32_t e = g.e0 + (g.released + ring) * kChunk;
    const uint32_t bar = g.bar0 + 8u * slot;
    // relaxed: the arrive only arms the transaction count, so no MEMBAR precedes it
    // No L2 eviction hint: the policy operand costs two uniform-register moves per copy and two
    // live registers in the walk, and the streamed matrix does not displace anything the SpMV
    // re-reads (x is staged once per CTA, the plan record once per warp).
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%4], %5;\n\t"
        "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %6, [%4];\n\t"
        "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %7, [%4];\n\t}" ::"r"(
            g.vbase + slot * kChunkVBytes),
        "l"(a.values + e), "r"(g.dbase + slot * dbytes<kBits>()), "l"(a.deltas + (size_t)(e / 8u) * kBits), "r"(bar),
        "n"(kChunkVBytes + dbytes<kBits>()), "n"(kChunkVBytes), "n"(dbytes<kBits>())
        : "memory");
}

// The walk reached S (slow path, S >= ring_ev): release the chunk the walk has left (every lane's
// LDS of it fed earlier FHFMAs; __syncwarp orders them before the refill) and wait until the
// chunks holding [S, S + span) have landed.
template <int kBits>
__device__ __forceinline__ void ring_advance(Ring& g, const SpmvArgs& a, uint32_t S, uint32_t span) {
    constexpr uint32_t ring = kMaxRing;
    if (S >= g.rel_at) {
        __syncwarp();
        ring_issue<kBits>(g, a);
        ++g.released;
        g.rel_at = g.released + ring < g.n_chunks ? g.e0 + (g.released + 1u) * kChunk : kNever;
    }
    const uint32_t need = min(g.n_chunks, (S + span - 1u - g.e0) / kChunk + 1u);
    for (; g.landed < need; ++g.landed)
        mbar_wait(g.bar0 + 8u * (g.landed & (ring - 1u)), (g.landed / ring) & 1u);
    g.wait_at = g.landed < g.n_chunks ? g.e0 + g.landed * kChunk - (2u * kStepElts - 1u) : kNever;
}

struct Slot {
    uint4 v;
    uint32_t d, d2;  // the lane's 8 codewords (d2: elements 4..7 when b_delta = 8)
};

// The lane's 8 elements at ring position 8 q (q: ring position in 8-element groups; 16 value
// bytes and kBits delta bytes per group).
template <int kBits>
__device__ __forceinline__ Slot lds_slot(uint32_t vbase, uint32_t dbase, uint32_t q) {
    Slot sl;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(sl.v.x), "=r"(sl.v.y), "=r"(sl.v.z), "=r"(sl.v.w)
                 : "r"(vbase + 16u * q));
    const uint32_t da = dbase + q * kBits;
    sl.d2 = 0;
    if constexpr (kBits == 8) {
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(sl.d), "=r"(sl.d2) : "r"(da));
    } else if constexpr (kBits == 4) {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(sl.d) : "r"(da));
    } else if constexpr (kBits == 2) {
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(sl.d) : "r"(da));
    } else {
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(sl.d) : "r"(da));
    }
    return sl;
}

// Valid-element mask of a lane's elements [eb, eb + 8) for the row [s, e).  The ROMA head (the
// previous row's elements before s: lane 0 of the row's first step, klo <= 7) also gets codeword
// 0 (delta 1) so the scan stays exact — the row's column base is shifted by the ROMA offset.
// Elements past e need no codeword change (prefixes run forward); values are never touched:
// masked elements skip their gather and FHFMA (lane_step).
template <int kBits>
__device__ __forceinline__ uint32_t mask_slot(Slot& sl, uint32_t eb, uint32_t s, uint32_t e) {
    const int klo = min(max((int)(s - eb), 0), 7);
    const int khi = min(max((int)(e - eb), klo), 8);
    const uint32_t vm = (0xFFu >> (8 - khi)) & (0xFFu << klo) & 0xFFu;  // valid-element mask
    if constexpr (kBits == 8) {
        sl.d &= klo >= 4 ? 0u : ~0u << (8 * klo);
        sl.d2 &= ~0u << (8 * max(klo - 4, 0));
    } else {
        sl.d &= ~0u << (kBits * klo);
    }
    return vm;
}

// ------------------------------------------------------------------------------------------
// Per-SpMV building blocks
// ------------------------------------------------------------------------------------------
struct PlanRecord {
    uint4 q0, q1, q2;  // the warp's WarpPlan (48 bytes)
};

__device__ __forceinline__ PlanRecord load_record(const SpmvArgs& a, uint32_t w) {
    const uint4* rec = reinterpret_cast<const uint4*>(a.plan.warps + w);
    return PlanRecord{__ldg(rec), __ldg(rec + 1), __ldg(rec + 2)};
}

// One bulk global -> shared copy completing on mbarrier bar (one lane).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src),
                 "r"(bytes), "r"(bar)
                 : "memory");
}

// PDL launches (decode chains) stagger the first fill: each warp requests chunk 0 of its ring before
// griddepcontrol.wait and the rest only after the CTA barrier, so every warp's first chunk is in the
// memory system first and the walks start as soon as it lands (decoder chain 2409 -> 2347 us per
// token).  A stand-alone SpMV keeps one two-chunk copy per array (0.1 % faster there).
// First-phase fill of ring slot i with chunk i of the warp's stream (one lane).
template <int kBits>
__device__ __forceinline__ void fill_chunk(const Ring& g, const SpmvArgs& a, uint32_t i) {
    const uint32_t bar = g.bar0 + 8u * i, e = g.e0 + i * kChunk;
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(kChunkVBytes + dbytes<kBits>())
                 : "memory");
    bulk_g2s(g.vbase + i * kChunkVBytes, a.values + e, kChunkVBytes, bar);
    bulk_g2s(g.dbase + i * dbytes<kBits>(), a.deltas + (size_t)(e / 8u) * kBits, dbytes<kBits>(), bar);
}

// Ring set-up for the warp's element stream [E0, E1): the barriers are initialised and the first
// fill is one copy per array.
template <int kBits, bool kStagger>
__device__ __forceinline__ void ring_begin(const SpmvArgs& a, uint32_t E0, uint32_t E1, uint32_t warp, int lane,
                                           uint32_t smem_base, uint32_t bar0, Ring& g) {
    constexpr uint32_t ring = kMaxRing;  // the host sizes a.ring_offset for exactly this ring
    g.vbase = smem_base + a.ring_offset + warp * ring * kChunkVBytes;
    g.dbase = smem_base + a.ring_offset + kSpmvWarpsPerCta * ring * kChunkVBytes + warp * ring * dbytes<kBits>();
    g.bar0 = bar0;
    g.e0 = E0 & ~(kChunk - 1u);
    g.emask = ring * kChunk - 1u;
    g.lane_rel = 8u * (uint32_t)lane - g.e0;
    g.n_chunks = E1 > E0 ? ((E1 - 1u) - g.e0) / kChunk + 1u : 0u;
    g.released = 0;
    g.landed = 0;
    g.rel_at = ring < g.n_chunks ? g.e0 + kChunk : kNever;
    g.wait_at = g.n_chunks ? 0u : kNever;  // the first pair waits for the first fill
    const uint32_t n = min(ring, g.n_chunks);
    if (lane == 0) {
        // The barriers are used by this warp and its own bulk copies only (no cluster): the
        // async-proxy fence orders their initialisation before the copies' complete_tx.
        for (uint32_t i = 0; i < ring; ++i) mbar_init(g.bar0 + 8u * i);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        MK_TRACE(5);
        // Initial fill: the first `ring` chunks are contiguous in global and shared memory, so one
        // copy per array fills them all and completes on barrier 0; the other barriers complete
        // their first phase with a plain arrive (the consumer passes barrier 0 first).
        // PDL launches (decode chains): chunk 0 alone now, the rest after the CTA barrier.
        if (n && !kStagger) {
            asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(g.bar0),
                         "r"(n * (kChunkVBytes + dbytes<kBits>()))
                         : "memory");
            bulk_g2s(g.vbase, a.values + g.e0, n * kChunkVBytes, g.bar0);
            bulk_g2s(g.dbase, a.deltas + (size_t)(g.e0 / 8u) * kBits, n * dbytes<kBits>(), g.bar0);
            for (uint32_t i = 1; i < n; ++i)
                asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(g.bar0 + 8u * i) : "memory");
        } else if (n) {
            fill_chunk<kBits>(g, a, 0);
        }
        MK_TRACE(7);
    }
    __syncwarp();
}

// Set up the warp's ring and ROMA walk for one SpMV (plan record pr) and issue the first fills.
template <int kBits, int kB, bool kStagger>
__device__ __forceinline__ bool op_begin(const SpmvArgs& a, const PlanRecord& pr, uint32_t warp, int lane,
                                         uint32_t smem_base, uint32_t bar0, Ring& g, RowState<kB>& rs) {
    const uint4 q0 = pr.q0, q1 = pr.q1, q2 = pr.q2;
    MK_TRACE(1);
    if (q0.x == 0) return false;
    ring_begin<kBits, kStagger>(a, q0.w, q1.x, warp, lane, smem_base, bar0, g);
    rs.r = q0.y;
    rs.units_left = q0.x;
    rs.s = q1.y;
    rs.e = q1.z;
    rs.e_next = rs.r + 2u <= a.rows ? __ldg(a.row_ptrs + rs.r + 2u) : 0u;
    begin_piece(rs, q0.z, (int)q1.w, (int32_t)q2.x, q2.z);
    return true;
}

// Stage x in shared memory (fp16, with zero guards of kXGuardLo / kXGuardHi entries); all
// threads of the CTA, the caller synchronises.  Batches: the interleaved XT (kB halves per column,
// guards kB halves per guard column) is staged the same way.
template <int kXMode, int kB = 1>
__device__ __forceinline__ void stage_x(const SpmvArgs& a, uint16_t* xs) {
    if constexpr (x_table<kXMode>() && kB > 1) {
        const uint32_t nv = a.cols * kB / 8;  // 16-byte vectors of XT (cols * kB is a multiple of 8 for kB >= 8;
        const uint4* x4 = reinterpret_cast<const uint4*>(a.x);  // capi pads XT to 16 bytes otherwise)
        const uint32_t nvp = (a.cols * kB + 7) / 8;
        for (uint32_t i = threadIdx.x; i < nvp; i += blockDim.x) reinterpret_cast<uint4*>(xs)[i] = __ldg(x4 + i);
        (void)nv;
        for (uint32_t i = nvp * 8 + threadIdx.x; i < (a.cols + kXGuardHi) * kB; i += blockDim.x) xs[i] = 0;
        if (threadIdx.x < kXGuardLo * kB) xs[(int)threadIdx.x - kXGuardLo * kB] = 0;
    } else if constexpr (x_table<kXMode>()) {
        const uint32_t C = a.cols;
        const uint4* x4 = reinterpret_cast<const uint4*>(a.x);  // 16-byte aligned (capi guarantees)
        const uint32_t nv = C / 8;
        // every CTA reads all of x: start each CTA at a different place so the 148 concurrent
        // streams spread over the L2 slices instead of queueing on the same lines
        const uint32_t rot = nv ? (blockIdx.x * 97u) % nv : 0u;
        for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
            const uint32_t k = i + rot < nv ? i + rot : i + rot - nv;
            reinterpret_cast<uint4*>(xs)[k] = __ldg(x4 + k);
        }
        for (uint32_t i = nv * 8 + threadIdx.x; i < C + kXGuardHi; i += blockDim.x)
            xs[i] = i < C ? a.x[i] : (uint16_t)0;
        if (threadIdx.x < kXGuardLo) xs[(int)threadIdx.x - kXGuardLo] = 0;
    }
}

#ifndef MACKO_TMA_X
#define MACKO_TMA_X 1
#endif
// x staged by one bulk copy per CTA (chain instance, SpMV with an x table): thread 0 issues it on
// barrier xbar, the other threads write the zero guards and the < 8-element tail; everyone waits
// on xbar after the CTA barrier.  Decoder chain 2284 vs 2337 us per token; stand-alone launches
// after an L2 flush were mixed (11008x4096 21.6 vs 20.8 us, 4096x11008 21.5 vs 22.4 us: all 148
// CTAs then fetch the same x lines from HBM in the same order), so they keep the threaded
// staging with per-CTA rotated order.
template <int kXMode, int kB>
constexpr bool x_by_tma() {
    return MACKO_TMA_X && kB == 1 && x_table<kXMode>();
}

// xbar completes when the bulk copy has landed (thread 0's expect_tx arrival) and thread 32 has
// written the guards and the tail (it arrives after them: release), so every warp waits on it
// alone — no CTA barrier between griddepcontrol.wait and the walk.
__device__ __forceinline__ void stage_x_tma_init(uint32_t xbar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(xbar) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void stage_x_tma_issue(const SpmvArgs& a, uint16_t* xs, uint32_t xbar) {
    const uint32_t nbytes = (a.cols / 8u) * 16u;  // x is 16-byte aligned (capi)
    if (nbytes) {
        asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(xbar), "r"(nbytes) : "memory");
        bulk_g2s(static_cast<uint32_t>(__cvta_generic_to_shared(xs)), a.x, nbytes, xbar);
    } else {
        asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(xbar) : "memory");
    }
}

// one thread: zero guards and the < 8-element tail (<= 31 entries), then it arrives on xbar itself,
// so its release covers exactly the writes it made
__device__ __forceinline__ void stage_x_tma_rest(const SpmvArgs& a, uint16_t* xs, uint32_t xbar) {
    const uint32_t C = a.cols;
    for (uint32_t i = (C / 8u) * 8u; i < C + kXGuardHi; ++i) xs[i] = i < C ? a.x[i] : (uint16_t)0;
    for (int i = 1; i <= kXGuardLo; ++i) xs[-i] = 0;
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(xbar) : "memory");
}

// The warp's walk over its rows of one SpMV (x staged, ring and walk set up by op_begin).
template <int kXMode, int kBits, int kB, bool kSplitEdges, bool kPeers, bool kNoSplit>
__device__ __forceinline__ void run_rows(const SpmvArgs& a, uint32_t w, int lane, uint32_t xs_addr_in, Ring& g,
                                         RowState<kB>& rs) {
    constexpr bool kMirror = !kSplitEdges && !kPeers;  // only the plain instance serves y_mirror
    if (rs.T == 0) {
        if (lane == 0) {
            const uint16_t z[kB] = {};
            put_y_b<kB, false, kMirror>(a, rs.r, z);
        }
        if constexpr (kPeers) own_row_put(a, rs.r, 0, lane);
        if (!next_piece<kB, kPeers, kMirror>(rs, a, w, lane)) return;
    }
    // loop invariants pinned in registers (not re-derived from the CTA's shared window per pair)
    // (ring positions in 8-element groups: the lane's group of a step at S is (S / 8 + lane_q) & qmask)
    uint32_t xs_addr, vbase, dbase, lane_q, qmask;
    asm volatile("mov.b32 %0, %1;" : "=r"(xs_addr) : "r"(xs_addr_in));
    asm volatile("mov.b32 %0, %1;" : "=r"(vbase) : "r"(g.vbase));
    asm volatile("mov.b32 %0, %1;" : "=r"(dbase) : "r"(g.dbase));
    asm volatile("mov.b32 %0, %1;" : "=r"(lane_q) : "r"(g.lane_rel / 8u));
    asm volatile("mov.b32 %0, %1;" : "=r"(qmask) : "r"(g.emask / 8u));
    uint32_t ev = ring_ev(g);

    // One step pair (steps t, t+1 of the current row); `edge` (kEdge*) says which of its steps
    // need the valid-element mask and whether step B exists.  Only a row's first pair (the ROMA
    // head in step A) and its last (the row end) are edges: the first pair's B is whole when the
    // row has >= 3 steps, the last pair's A is whole unless it is also the first step, and a row
    // with an odd number of steps ends in a single step (no phantom B).
    auto pair = [&](auto edge, uint32_t t) {
        constexpr uint32_t kE = decltype(edge)::value;
        constexpr bool kMaskA = kE & kEdgeMaskA, kMaskB = kE & kEdgeMaskB, kHasB = !(kE & kEdgeSingle);
        const uint32_t S = rs.al + t * kStepElts;
        if (S >= ev) {
            ring_advance<kBits>(g, a, S, (kHasB ? 2u : 1u) * kStepElts);
            ev = ring_ev(g);
        }
        const uint32_t qA = ((rs.al >> 3) + t * (kStepElts / 8u) + lane_q) & qmask;  // S is 8-aligned
        Slot A = lds_slot<kBits>(vbase, dbase, qA);
        Slot B{};
        if constexpr (kHasB) B = lds_slot<kBits>(vbase, dbase, (qA + kStepElts / 8u) & qmask);
        uint32_t vmA = 0xFFu, vmB = 0xFFu;
        if constexpr (kMaskA) vmA = mask_slot<kBits>(A, S + 8u * lane, rs.s, rs.e);
        if constexpr (kMaskB) vmB = mask_slot<kBits>(B, S + kStepElts + 8u * lane, rs.s, rs.e);
        using D = typename std::conditional<kBits == 8, Dec8, Dec>::type;
        D dA, dB{};
        uint32_t bias = 0;  // b = 8: lane totals reach 2048, so the packed scan runs on (total - 8)
        if constexpr (kBits == 8) {
            dA = decode8(A.d, A.d2);
            if constexpr (kHasB) dB = decode8(B.d, B.d2);
            bias = 8;
        } else {
            dA = decode<kBits>(A.d);
            if constexpr (kHasB) dB = decode<kBits>(B.d);
        }
        const uint32_t pk = (dA.local - bias) | (kHasB ? (dB.local - bias) << 16 : 0u);
        const uint32_t incl = warp_incl_scan_p(pk);
        const uint32_t tot = __reduce_add_sync(kFull, pk);
        const uint32_t lane_bias = bias * (uint32_t)lane, tot_bias = bias * kWarp;
        const int cbA = rs.col_base + (int)((incl & 0xFFFFu) - (dA.local - bias) + lane_bias);
        if constexpr (kB == 1) {
            rs.acc[0] = lane_step<kXMode, kMaskA>(rs.acc[0], A.v, dA, cbA, xs_addr, a.xtex, vmA);
        } else {
            lane_step_b<kXMode, kMaskA, kB>(rs.acc, A.v, dA, cbA, xs_addr, a.xtex, vmA);
        }
        if constexpr (kHasB) {
            const int cbB = rs.col_base + (int)((tot & 0xFFFFu) + tot_bias) + (int)((incl >> 16) - (dB.local - bias) + lane_bias);
            if constexpr (kB == 1) {
                rs.acc[0] = lane_step<kXMode, kMaskB, tex_slots_b<kXMode>()>(rs.acc[0], B.v, dB, cbB, xs_addr, a.xtex, vmB);
            } else {
                lane_step_b<kXMode, kMaskB, kB, tex_slots_b<kXMode>()>(rs.acc, B.v, dB, cbB, xs_addr, a.xtex, vmB);
            }
            rs.col_base += (int)(tot & 0xFFFFu) + (int)(tot >> 16) + 2 * (int)tot_bias;
        }
    };
    using EdgeFirst = std::integral_constant<uint32_t, kEdgeMaskA>;                  // ROMA head, B whole
    using EdgeFirstLast = std::integral_constant<uint32_t, kEdgeMaskA | kEdgeMaskB>; // a two-step row
    using EdgeLast = std::integral_constant<uint32_t, kEdgeMaskB>;                   // A whole, B ends the row
    using EdgeSingle = std::integral_constant<uint32_t, kEdgeMaskA | kEdgeSingle>;   // the row's last step alone
    using Interior = std::integral_constant<uint32_t, 0u>;

    // Per-step edge masking (kSplitEdges) is the kernel instance of PDL launches (decode chains,
    // where consecutive SpMVs keep the kernel's code warm: 2343 vs 2378 us per token).  A
    // stand-alone launch after an L2 flush fetches its code from HBM, and the four extra edge
    // variants cost more in cold instruction misses than they save (11008x4096: 21.8 vs 20.8 us),
    // so that instance masks both steps of an edge pair.  (A run-time switch between the two costs
    // registers: 121 vs 111 us at 36864x12288.)
    constexpr bool split_edges = kSplitEdges && kEdgeSplit;
    for (;;) {
        // the piece's units: [8j, 8j+8) steps, the row's last unit [last_b, T).  Pair t is an edge
        // iff it is the row's first (t = 0) or last (t + 2 >= T); interior pairs run unmasked.
        for (uint32_t t = rs.t; t < rs.tend;) {
            const uint32_t ue = t < rs.last_b ? t + kUnitSteps : rs.tend;
            if (t == 0u) {
                if (!split_edges) {
                    pair(EdgeFirstLast{}, 0u);
                } else if (rs.T >= 3u) {
                    pair(EdgeFirst{}, 0u);
                } else if (rs.T == 2u) {
                    pair(EdgeFirstLast{}, 0u);
                } else {
                    pair(EdgeSingle{}, 0u);
                }
                t = 2u;
            }
            const uint32_t lim = min(ue, rs.T - min(rs.T, 2u));
            for (; t < lim; t += 2u) pair(Interior{}, t);
            if (t < ue) {  // the row's last pair (t >= 2)
                if (!split_edges) {
                    pair(EdgeFirstLast{}, t);
                } else if (rs.T - t == 2u) {
                    pair(EdgeLast{}, t);
                } else {
                    pair(EdgeSingle{}, t);
                }
                t += 2u;
            }
            const uint32_t pslot = rs.slot + min((ue - 1u) / kUnitSteps, rs.n_r - 1u);
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                const float red = warp_tree_sum(rs.acc[b]);
                rs.acc[b] = 0.0f;
                if (!kNoSplit && rs.split && rs.j0 > 0 && lane == 0) a.plan.partials[(size_t)pslot * kB + b] = red;
                rs.row_acc[b] += red;
            }
            t = ue;
        }
        // -- piece end
        if constexpr (kB == 1) {
            if (kNoSplit || !rs.split) {
                const uint16_t v = f32_to_f16_rn(rs.row_acc[0]);
                if (lane == 0) put_y<false, kMirror>(a, rs.r, v);
                if constexpr (kPeers) own_row_put(a, rs.r, v, lane);
            } else {
                const int v = finish_split(rs.j0, rs.tend, rs.n_r, rs.slot, rs.sid, rs.row_acc[0], a.plan, lane);
                if (v >= 0) put_y<kPeers, kMirror>(a, rs.r, (uint16_t)v);
            }
        } else {
            uint16_t out[kB];
            if (!rs.split) {
#pragma unroll
                for (int b = 0; b < kB; ++b) out[b] = f32_to_f16_rn(rs.row_acc[b]);
                if (lane == 0) put_y_b<kB, false, kMirror>(a, rs.r, out);
            } else if (finish_split_b<kB>(rs.j0, rs.tend, rs.n_r, rs.slot, rs.sid, rs.row_acc, a.plan, lane, out)) {
                put_y_b<kB, kPeers, kMirror>(a, rs.r, out);
            }
        }
        if (!next_piece<kB, kPeers, kMirror>(rs, a, w, lane)) break;
    }
}

// kChain: the instance of PDL launches (decode chains): per-step edge masking (run_rows) and x
// staged by one bulk copy per CTA (stage_x_tma_*).  Both pay only with the kernel's code and x
// warm in L2, as in a chain; a stand-alone launch after an L2 flush is faster without them.
// kNoSplit: the chain instance for plans without split rows (every row one unit, as in the Llama
// linears): no partial stores or split finish in the walk (chain 2154 -> 2129 us per token; the
// plain instance gains nothing from it).
template <int kXMode, int kBits, int kB = 1, bool kChain = false, bool kPeers = false, bool kNoSplit = false>
__global__ void __launch_bounds__(kSpmvWarpsPerCta * kWarp, kSpmvCtasPerSm) macko_spmv(const SpmvArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[kSpmvWarpsPerCta][kMaxRing];
    const int lane = threadIdx.x & (kWarp - 1);
    const uint32_t warp = threadIdx.x >> 5;
    const bool active = warp < a.warps_active;
    const uint32_t w = blockIdx.x * a.warps_active + warp;  // this warp's plan record (active warps)
    const uint32_t smem_base = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    MK_TRACE(0);
    // Programmatic dependent launch (chains of SpMVs): the next kernel in the stream may start
    // its prologue (plan record, first matrix ring fills) on SMs this grid has left; everything
    // it reads before griddepcontrol.wait is static matrix data.  No-ops without the attribute.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const PlanRecord pr = active ? load_record(a, w) : PlanRecord{};
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem) + kXGuardLo * kB;
    __shared__ __align__(8) uint64_t xbar_s;
    const uint32_t xbar = static_cast<uint32_t>(__cvta_generic_to_shared(&xbar_s));
    constexpr bool kTmaX = x_by_tma<kXMode, kB>() && kChain;
    // Without a PDL producer x is final at entry: its loads overlap the plan record's latency.
    if constexpr (kTmaX) {
        if (threadIdx.x == 0) stage_x_tma_init(xbar);
        __syncthreads();  // xbar initialised before any warp polls it (every warp is here at entry)
        if (!a.pdl && threadIdx.x == 0) stage_x_tma_issue(a, xs, xbar);
    } else {
#ifndef MACKO_RING_FIRST
        if (!a.pdl) stage_x<kXMode, kB>(a, xs);
#endif
    }
    // The first ring fills go out before a PDL wait; x staging overlaps their HBM latency.
    RowState<kB> rs;
    Ring g;
    const bool has_work = op_begin<kBits, kB, kChain>(a, pr, warp, lane, smem_base,
                                         static_cast<uint32_t>(__cvta_generic_to_shared(&bars[warp][0])), g, rs);
    if (kPeers && has_work && lane == 0) s_own_first[warp] = rs.r + (rs.split ? 1u : 0u);
#ifdef MACKO_RING_FIRST
    if (!a.pdl) stage_x<kXMode, kB>(a, xs);
#endif
    MK_TRACE(2);
    // x (and y) may be produced / consumed by the previous kernel of a PDL chain.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    MK_TRACE(3);
    if constexpr (kTmaX) {
        if (a.pdl && threadIdx.x == 0) stage_x_tma_issue(a, xs, xbar);
        if (threadIdx.x == 32) stage_x_tma_rest(a, xs, xbar);  // warp 1: warp 0's thread 0 issues the copy
        mbar_wait(xbar, 0);  // this warp alone: x landed, guards and tail written
    } else {
        if (a.pdl) stage_x<kXMode, kB>(a, xs);
        __syncthreads();
    }
    MK_TRACE(4);
    const uint32_t xs_addr = static_cast<uint32_t>(__cvta_generic_to_shared(xs));
    if (kChain && has_work && lane == 0)  // the staggered first fill's remaining chunks (ring_begin), once x is in
        for (uint32_t i = 1; i < min(kMaxRing, g.n_chunks); ++i) fill_chunk<kBits>(g, a, i);
    if (has_work) run_rows<kXMode, kBits, kB, kChain, kPeers, kNoSplit>(a, w, lane, xs_addr, g, rs);
    MK_TRACE(6);
    if constexpr (kPeers) {
        if (has_work) {  // the stash's last, partial group
            const uint32_t r1 = rs.r + (rs.split ? 0u : 1u);
            flush_own(a, r1 & ~(kOwnGroup - 1), r1, lane);
        }
        signal_peers(a);
    }
}

// Column just before the first unit of every chunk that starts inside a row: sum of the row's
// deltas over [row start, the row's 8-aligned start + j units) minus one.  Setup only.
__global__ void plan_colbase_kernel(const uint8_t* deltas, uint32_t bits, WarpPlan* warps, uint32_t n_chunks) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & (kWarp - 1);
    if (w >= n_chunks) return;
    const uint32_t s = warps[w].s;
    const uint32_t lim = (s & ~7u) + warps[w].j * kUnitElts;
    if (warps[w].units_left == 0 || warps[w].j == 0) {
        if (lane == 0) warps[w].colbase = -1;
        return;
    }
    const uint32_t per = 8u / bits, mask = bits == 8 ? 0xFFu : (1u << bits) - 1u;
    uint32_t sum = 0;
    for (uint32_t i = s + lane; i < lim; i += kWarp) sum += ((deltas[i / per] >> ((i % per) * bits)) & mask) + 1u;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) sum += __shfl_xor_sync(kFull, sum, off);
    if (lane == 0) warps[w].colbase = (int32_t)sum - 1;
}

}  // namespace

template <int kXMode, int kBits>
static cudaError_t occ_one(size_t smem, int* ctas_per_sm) {
    const int threads = kSpmvWarpsPerCta * kWarp;
    cudaError_t e = cudaFuncSetAttribute(macko_spmv<kXMode, kBits>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(macko_spmv<kXMode, kBits, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(macko_spmv<kXMode, kBits, 1, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(macko_spmv<kXMode, kBits, 1, true, false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, macko_spmv<kXMode, kBits>, threads, smem);
    if (e == cudaSuccess) {
        int c2 = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c2, macko_spmv<kXMode, kBits, 1, true>, threads, smem);
        *ctas_per_sm = std::min(*ctas_per_sm, c2);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c2, macko_spmv<kXMode, kBits, 1, true, true>, threads, smem);
        *ctas_per_sm = std::min(*ctas_per_sm, c2);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c2, macko_spmv<kXMode, kBits, 1, true, false, true>, threads,
                                                              smem);
        *ctas_per_sm = std::min(*ctas_per_sm, c2);
    }
    return e;
}

#ifndef MACKO_CHAIN_FOR_ALL
#define MACKO_CHAIN_FOR_ALL 0
#endif
constexpr bool kChainForAll = MACKO_CHAIN_FOR_ALL;  // experiments: the chain instance for every launch

template <int kXMode, int kBits>
static cudaError_t launch_one(const SpmvArgs& a, int grid, size_t smem, cudaStream_t s, bool pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kSpmvWarpsPerCta * kWarp);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    // fused all-gather: the chain instance with the peer stores (the others carry none of that code);
    // the host-buffer path's y_mirror: the plain instance alone
    if (a.n_peer && a.y_mirror) return cudaErrorInvalidValue;
    if (a.y_mirror) return cudaLaunchKernelEx(&cfg, macko_spmv<kXMode, kBits>, a);
    if (a.n_peer) return cudaLaunchKernelEx(&cfg, macko_spmv<kXMode, kBits, 1, true, true>, a);
    if (pdl || kChainForAll)
        return a.no_split ? cudaLaunchKernelEx(&cfg, macko_spmv<kXMode, kBits, 1, true, false, true>, a)
                          : cudaLaunchKernelEx(&cfg, macko_spmv<kXMode, kBits, 1, true>, a);
    return cudaLaunchKernelEx(&cfg, macko_spmv<kXMode, kBits>, a);
}

// Small-batch SpMM (b_delta 4): x_mode 0 (TEX gathers of 2 kB-byte texels) or 7 (the SpMV's
// LSU / TEX split over an interleaved shared-memory table).
template <int kXMode, int kB>
static cudaError_t launch_spmm_one(const SpmvArgs& a, int grid, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(macko_spmv<kXMode, 4, kB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    macko_spmv<kXMode, 4, kB><<<grid, kSpmvWarpsPerCta * kWarp, smem, s>>>(a);
    return cudaGetLastError();
}

template <int kXMode>
static cudaError_t launch_spmm_mode(const SpmvArgs& a, int kb, int grid, size_t smem, cudaStream_t s) {
    switch (kb) {
        case 2: return launch_spmm_one<kXMode, 2>(a, grid, smem, s);
        case 4: return launch_spmm_one<kXMode, 4>(a, grid, smem, s);
        case 8: return launch_spmm_one<kXMode, 8>(a, grid, smem, s);
        default: return cudaErrorInvalidValue;
    }
}

bool spmm_valid_x_mode(int x_mode) { return x_mode == 0 || x_mode == 1 || x_mode == 6 || x_mode == 7 || x_mode == 8; }

cudaError_t launch_spmm(const SpmvArgs& a, int kb, int grid, int x_mode, size_t smem, cudaStream_t s) {
    switch (x_mode) {
        case 0: return launch_spmm_mode<0>(a, kb, grid, smem, s);
        case 1: return launch_spmm_mode<1>(a, kb, grid, smem, s);
        case 6: return launch_spmm_mode<6>(a, kb, grid, smem, s);
        case 7: return launch_spmm_mode<7>(a, kb, grid, smem, s);
        case 8: return launch_spmm_mode<8>(a, kb, grid, smem, s);
        default: return cudaErrorInvalidValue;
    }
}

// XT[c * kb + b] = X[b][c] (b < batch; 0 for the padding vectors), the SpMM's interleaved x.
__global__ void interleave_kernel(const uint16_t* __restrict__ X, uint64_t ldx, uint32_t batch, uint32_t kb,
                                  uint32_t cols, uint16_t* __restrict__ XT, uint32_t n_total) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_total; i += gridDim.x * blockDim.x) {
        const uint32_t c = i / kb, b = i - c * kb;
        XT[i] = (c < cols && b < batch) ? X[(size_t)b * ldx + c] : (uint16_t)0;
    }
}

cudaError_t launch_interleave(const uint16_t* X, uint64_t ldx, uint32_t batch, uint32_t kb, uint32_t cols,
                              uint16_t* XT, uint32_t n_total, cudaStream_t s) {
    const int grid = (int)std::min<uint32_t>((n_total + 255) / 256, 1024u);
    if (grid) interleave_kernel<<<grid, 256, 0, s>>>(X, ldx, batch, kb, cols, XT, n_total);
    return cudaGetLastError();
}

// Host-buffer SpMV (macko_spmv_host) with pinned, device-mapped host x / y: a one-CTA kernel pulls
// x over the host link into the device buffer, the SpMV follows as its programmatic dependent (its
// plan load and first matrix fills overlap the pull), and a second small kernel pushes y to the
// host buffer as the SpMV's dependent.  n16: 16-byte vectors; the remainder moves as 2-byte words.
__global__ void __launch_bounds__(1024) copy_u16_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst,
                                                         uint32_t n, uint32_t wait_producer) {
    if (wait_producer) asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t n16 = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) ? 0u : n / 8u;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    for (uint32_t i = tid; i < n16; i += nt)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (uint32_t i = n16 * 8u + tid; i < n; i += nt) dst[i] = src[i];
}

// Consumer side of the fused all-gather: one thread per rank slot spins (system-scope acquire)
// until every peer's CTAs have signalled; traps after ~4 s instead of hanging the GPU.
__global__ void wait_flags_kernel(const uint32_t* flags, uint32_t n, uint32_t target) {
    if (threadIdx.x < n) {
        const long long t0 = clock64();
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + threadIdx.x) : "memory");
            if ((int32_t)(v - target) >= 0) break;
            __nanosleep(64);
            if (clock64() - t0 > 8000000000LL) __trap();
        }
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

cudaError_t launch_wait_flags(const uint32_t* flags, uint32_t n, uint32_t target, cudaStream_t s) {
    wait_flags_kernel<<<1, 32, 0, s>>>(flags, n, target);
    return cudaGetLastError();
}

cudaError_t launch_copy_u16(const uint16_t* src, uint16_t* dst, uint32_t n, int blocks, bool dependent, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(1024);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = dependent ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, copy_u16_kernel, src, dst, n, dependent ? 1u : 0u);
}

// Every width gets the x_modes of the automatic rule (build_plan).
bool spmv_valid_x_mode(int x_mode) { return x_mode == 0 || x_mode == 1 || (x_mode >= 6 && x_mode <= 8) || x_mode == 10; }
bool spmv_valid_config(int x_mode, int bits) {
    return (bits == 1 || bits == 2 || bits == 4 || bits == 8) && spmv_valid_x_mode(x_mode);
}

template <int kBits>
static cudaError_t occ_bits(int x_mode, size_t smem, int* c) {
    switch (x_mode) {
        case 10: return occ_one<10, kBits>(smem, c);
        case 8: return occ_one<8, kBits>(smem, c);
        case 7: return occ_one<7, kBits>(smem, c);
        case 6: return occ_one<6, kBits>(smem, c);
        case 1: return occ_one<1, kBits>(smem, c);
        case 0: return occ_one<0, kBits>(smem, c);
        default: break;
    }
    return cudaErrorInvalidValue;
}

template <int kBits>
static cudaError_t launch_bits(const SpmvArgs& a, int grid, int x_mode, size_t smem, cudaStream_t s, bool pdl) {
    switch (x_mode) {
        case 10: return launch_one<10, kBits>(a, grid, smem, s, pdl);
        case 8: return launch_one<8, kBits>(a, grid, smem, s, pdl);
        case 7: return launch_one<7, kBits>(a, grid, smem, s, pdl);
        case 6: return launch_one<6, kBits>(a, grid, smem, s, pdl);
        case 1: return launch_one<1, kBits>(a, grid, smem, s, pdl);
        case 0: return launch_one<0, kBits>(a, grid, smem, s, pdl);
        default: break;
    }
    return cudaErrorInvalidValue;
}

size_t spmv_static_smem() {
    cudaFuncAttributes f0{}, f1{}, f2{};
    if (cudaFuncGetAttributes(&f0, macko_spmv<10, 2, 1, false>) != cudaSuccess ||
        cudaFuncGetAttributes(&f1, macko_spmv<10, 2, 1, true>) != cudaSuccess ||
        cudaFuncGetAttributes(&f2, macko_spmv<10, 2, 1, true, true>) != cudaSuccess)
        return 0;
    return std::max(std::max(f0.sharedSizeBytes, f1.sharedSizeBytes), f2.sharedSizeBytes);
}

cudaError_t spmv_occupancy(int x_mode, int bits, size_t smem, int* ctas_per_sm) {
    switch (bits) {
        case 4: return occ_bits<4>(x_mode, smem, ctas_per_sm);
        case 2: return occ_bits<2>(x_mode, smem, ctas_per_sm);
        case 8: return occ_bits<8>(x_mode, smem, ctas_per_sm);
        case 1: return occ_bits<1>(x_mode, smem, ctas_per_sm);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_spmv(const SpmvArgs& a, int bits, int grid, int x_mode, size_t smem, cudaStream_t s, bool pdl) {
    switch (bits) {
        case 4: return launch_bits<4>(a, grid, x_mode, smem, s, pdl);
        case 2: return launch_bits<2>(a, grid, x_mode, smem, s, pdl);
        case 8: return launch_bits<8>(a, grid, x_mode, smem, s, pdl);
        case 1: return launch_bits<1>(a, grid, x_mode, smem, s, pdl);
        default: return cudaErrorInvalidValue;
    }
}

#ifdef MACKO_TRACE
cudaError_t trace_read(unsigned long long* host, size_t n) {
    n = n < sizeof(g_macko_trace) / 8 ? n : sizeof(g_macko_trace) / 8;
    return cudaMemcpyFromSymbol(host, g_macko_trace, n * 8);
}
#endif

cudaError_t launch_plan_colbase(const uint8_t* deltas, uint32_t bits, WarpPlan* warps, uint32_t n_chunks, cudaStream_t s) {
    const int threads = 256;
    const int blocks = (int)((n_chunks * (uint64_t)kWarp + threads - 1) / threads);
    if (blocks) plan_colbase_kernel<<<blocks, threads, 0, s>>>(deltas, bits, warps, n_chunks);
    return cudaGetLastError();
}

}  // namespace mk
