// compress.cu — dense fp16 -> MACKO on the GPU (bit-exact with the reference encoder).
//
// Reference semantics: csr_from_dense + macko_from_csr (convert.hpp:8-16):
// drop ±0, per row prev = -1, pad with (+0, 2^b) while c - prev > 2^b, no trailing pads,
// codeword delta-1 LSB-first (bitpack.cpp:18-32), 16-byte zero tails (matrix.hpp:57-59).
//
// Parallel form (probe A.4): padding depends only on adjacent nonzeros.  For a
// zero column c with previous nonzero p (or -1) it is a padding entry iff (c - p) % 2^b == 0
// and a nonzero exists after c; a nonzero at c has delta ((c - p - 1) mod 2^b) + 1.  So every
// column is classified independently once p (an exclusive max-scan over the row) and the last
// nonzero column of the row are known:
//   K2a count_rows : warp per row, 16-B loads, nonzero bitmask, max-scan -> entries per row
//   K2b scan_counts: one CTA, exclusive u64 scan -> u32 row pointers + pad_nnz (overflow check)
//   K2c emit_rows  : warp per row, same classification, lane-prefix of entry counts -> values
//                    (2-B stores) and codewords staged per warp in shared memory and written as
//                    whole 32-bit words; words shared with a neighbouring row use atomicOr.
#include "common.cuh"
#include "compress.cuh"

#include <algorithm>

namespace mk {

namespace {

constexpr int kCompressWarpsPerCta = 8;
constexpr int kStageWords = 72;  // per chunk <= 256 entries x 8 bits or 512 x 4 bits = 64 words, + carry + spill

// The 8 columns [c, c+8) of a dense row (zeros past `cols`) as four fp16 pairs.  Loops issue
// the next chunk's fetch before working on the current one (one 16-byte load per lane in flight
// under the classification).
__device__ __forceinline__ uint4 fetch8(const uint16_t* row, uint32_t c, uint32_t cols, bool vec_ok) {
    if (vec_ok && c + 8 <= cols) return __ldg(reinterpret_cast<const uint4*>(row + c));
    uint32_t w[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const uint32_t lo = (c + 2 * m < cols) ? row[c + 2 * m] : 0u;
        const uint32_t hi = (c + 2 * m + 1 < cols) ? row[c + 2 * m + 1] : 0u;
        w[m] = lo | (hi << 16);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// Nonzero mask of 8 fetched columns (+-0 are zero); `h` receives the raw fp16 bits.
__device__ __forceinline__ uint32_t unpack8(const uint4 q, uint16_t h[8]) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        h[2 * m] = (uint16_t)(w[m] & 0xFFFFu);
        h[2 * m + 1] = (uint16_t)(w[m] >> 16);
    }
    uint32_t nz = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) nz |= ((h[k] & 0x7FFFu) != 0 ? 1u : 0u) << k;
    return nz;
}

// Previous nonzero column before this lane's first column (-1: none in the row so far), seeded
// with `carry` (the last nonzero column of the earlier chunks); carry becomes the chunk's last.
// One ballot finds the nearest lower lane holding a nonzero, one shuffle fetches its column.
__device__ __forceinline__ int prev_nonzero(int lane_last, int lane, int& carry) {
    const uint32_t bal = __ballot_sync(kFull, lane_last >= 0);
    const uint32_t below = bal & ((1u << lane) - 1u);
    const int from = __shfl_sync(kFull, lane_last, below ? 31 - __clz(below) : lane);
    const int p = below ? from : carry;
    const int last = __shfl_sync(kFull, lane_last, bal ? 31 - __clz(bal) : 0);
    if (bal) carry = last;
    return p;
}

// b_delta >= 4 (max delta >= 16 >= the kCols columns of a lane): a lane holds at most one padding entry,
// at the first column cc0 >= c with cc0 = p (mod 2^b), cc0 > p, before the lane's first nonzero
// (and before the row's last nonzero L); the nonzeros after the lane's first are never padded.
template <int kCols>
__device__ __forceinline__ uint32_t pad_bit(uint32_t nz, int c, int p, int L, uint32_t bits) {
    const int maxd = 1 << bits;
    const int cc0 = p + maxd * ((c - p + maxd - 1) >> bits);  // smallest p + k*maxd >= c (c > p)
    const int lim = min(nz ? c + __ffs(nz) - 1 : c + kCols, L);
    return cc0 < lim ? 1u << (cc0 - c) : 0u;
}

// kCols columns per lane per chunk (16 for b_delta = 4: gaps inside a lane stay < 2^b).
template <bool kFast, int kCols>
__global__ void __launch_bounds__(kCompressWarpsPerCta * kWarp, 4)
    count_rows(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, uint32_t bits,
               uint32_t* counts, int32_t* lastcol) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint32_t nwarps = gridDim.x * kCompressWarpsPerCta;
    const bool vec_base = ((reinterpret_cast<uintptr_t>(dense) | (ld * 2)) & 15u) == 0;
    constexpr uint32_t kStep = kWarp * kCols;
    for (uint32_t r = blockIdx.x * kCompressWarpsPerCta + (threadIdx.x >> 5); r < rows; r += nwarps) {
        const uint16_t* row = dense + (uint64_t)r * ld;
        int carry = -1;
        uint32_t cnt = 0;
        uint4 next[kCols / 8];  // the next chunk's load is in flight while this one is classified
#pragma unroll
        for (int q = 0; q < kCols / 8; ++q) next[q] = fetch8(row, kCols * lane + 8 * q, cols, vec_base);
        for (uint32_t c0 = 0; c0 < cols; c0 += kStep) {
            const uint32_t c = c0 + kCols * lane;
            uint16_t h[kCols];
            uint32_t nz = 0;
#pragma unroll
            for (int q = 0; q < kCols / 8; ++q) nz |= unpack8(next[q], h + 8 * q) << (8 * q);
            if (c0 + kStep < cols) {
#pragma unroll
                for (int q = 0; q < kCols / 8; ++q) next[q] = fetch8(row, c + kStep + 8 * q, cols, vec_base);
            }
            const int lane_last = nz ? (int)(c + 31 - __clz(nz)) : -1;
            int p = prev_nonzero(lane_last, lane, carry);
            cnt += __popc(nz);
            if constexpr (kFast) {
                // pads of the gap before the lane's first nonzero (the others are < 2^b apart)
                if (nz) cnt += (uint32_t)((int)c + __ffs(nz) - 2 - p) >> bits;
            } else {
                while (nz) {
                    const int k = __ffs(nz) - 1;
                    nz &= nz - 1;
                    const int cc = (int)c + k;
                    cnt += (uint32_t)(cc - p - 1) >> bits;
                    p = cc;
                }
            }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
        if (lane == 0) {
            counts[r] = cnt;
            lastcol[r] = carry;
        }
    }
}

__global__ void __launch_bounds__(1024) scan_counts(const uint32_t* counts, uint32_t rows, uint32_t* row_ptrs,
                                                     unsigned long long* total) {
    __shared__ unsigned long long warp_sums[32];
    const uint32_t t = threadIdx.x, nt = blockDim.x;
    const uint64_t lo = (uint64_t)rows * t / nt, hi = (uint64_t)rows * (t + 1) / nt;
    unsigned long long mine = 0;
    for (uint64_t i = lo; i < hi; ++i) mine += counts[i];
    // block exclusive scan of `mine`
    const int lane = t & 31, wid = t >> 5;
    unsigned long long incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long v = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += v;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        unsigned long long ws = lane < (int)(nt / 32) ? warp_sums[lane] : 0ull;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long v = __shfl_up_sync(kFull, ws, off);
            if (lane >= off) ws += v;
        }
        warp_sums[lane] = ws;
    }
    __syncthreads();
    unsigned long long run = incl - mine + (wid ? warp_sums[wid - 1] : 0ull);
    if (t == 0) row_ptrs[0] = 0;
    for (uint64_t i = lo; i < hi; ++i) {
        run += counts[i];
        row_ptrs[i + 1] = (uint32_t)run;
    }
    if (t == nt - 1) *total = run;
}

// kCols columns per lane per chunk: 16 for b_delta = 4 (a lane's <= 16 entries fit one 64-bit code
// word), else 8.
template <bool kFast, int kCols>
__global__ void __launch_bounds__(kCompressWarpsPerCta * kWarp, 4)
    emit_rows(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, uint32_t bits,
              const uint32_t* row_ptrs, const int32_t* lastcol, uint16_t* values, uint32_t* delta_words) {
    __shared__ uint32_t stage_all[kCompressWarpsPerCta][kStageWords];
    // a chunk's values (<= kWarp * kCols entries: a pad takes a zero column), written out coalesced
    __shared__ uint16_t vstage_all[kCompressWarpsPerCta][kWarp * kCols];
    // kFast: codes of the nonzeros after a lane's first one, per 8-column nonzero pattern (their
    // deltas are the gaps between set bits, < 8), packed at b_delta bits each
    __shared__ uint64_t gap_codes[kFast ? 256 : 1];
    const int lane = threadIdx.x & (kWarp - 1);
    if constexpr (kFast) {
        for (uint32_t pat = threadIdx.x; pat < 256; pat += blockDim.x) {
            uint64_t v = 0;
            uint32_t i = 0, rest = pat;
            int prev = -1;
            while (rest) {
                const int k = __ffs(rest) - 1;
                rest &= rest - 1;
                if (prev >= 0) v |= (uint64_t)(uint32_t)(k - prev - 1) << (bits * i++);
                prev = k;
            }
            gap_codes[pat] = v;
        }
        __syncthreads();
    }
    uint32_t* stage = stage_all[threadIdx.x >> 5];
    uint16_t* vstage = vstage_all[threadIdx.x >> 5];
    const uint32_t nwarps = gridDim.x * kCompressWarpsPerCta;
    const bool vec_base = ((reinterpret_cast<uintptr_t>(dense) | (ld * 2)) & 15u) == 0;
    const uint32_t maxd = 1u << bits;
    for (uint32_t r = blockIdx.x * kCompressWarpsPerCta + (threadIdx.x >> 5); r < rows; r += nwarps) {
        const uint32_t start = row_ptrs[r], end = row_ptrs[r + 1];
        if (start == end) continue;
        const int L = lastcol[r];
        const uint16_t* row = dense + (uint64_t)r * ld;
        const uint64_t row_first_word = ((uint64_t)start * bits) >> 5;
        const bool first_shared = (((uint64_t)start * bits) & 31u) != 0;
        for (int i = lane; i < kStageWords; i += kWarp) stage[i] = 0;
        __syncwarp();
        int carry = -1;
        uint32_t emitted = 0;                // entries of this row written so far
        uint64_t wb = row_first_word;        // global word held in stage[0]
        constexpr uint32_t kStep = kWarp * kCols;
        uint4 next[kCols / 8];
#pragma unroll
        for (int q = 0; q < kCols / 8; ++q) next[q] = fetch8(row, kCols * lane + 8 * q, cols, vec_base);
        for (uint32_t c0 = 0; c0 < cols && (int)c0 <= L; c0 += kStep) {
            const uint32_t c = c0 + kCols * lane;
            uint16_t h[kCols];
            uint32_t nz = 0;
#pragma unroll
            for (int q = 0; q < kCols / 8; ++q) nz |= unpack8(next[q], h + 8 * q) << (8 * q);
            if (c0 + kStep < cols && (int)(c0 + kStep) <= L) {
#pragma unroll
                for (int q = 0; q < kCols / 8; ++q) next[q] = fetch8(row, c + kStep + 8 * q, cols, vec_base);
            }
            const int lane_last = nz ? (int)(c + 31 - __clz(nz)) : -1;
            int p = prev_nonzero(lane_last, lane, carry);
            // classify the lane's 8 columns: nonzero entry, padding entry or nothing; codes of the
            // lane's entries packed in column order (entry i at bits [i*b, (i+1)*b))
            uint32_t em = 0;  // entry mask
            uint64_t codes = 0;
            if constexpr (kFast) {
                const uint32_t pb = pad_bit<kCols>(nz, (int)c, p, L, bits);
                em = nz | pb;
                const uint32_t sh = pb ? bits : 0u;  // the pad entry comes first
                codes = pb ? (uint64_t)(maxd - 1) : 0ull;
                if (nz) {
                    const uint32_t first = (uint32_t)((int)c + __ffs(nz) - 2 - p) & (maxd - 1);
                    uint64_t gaps;  // codes of the nonzeros after the lane's first, in order
                    if constexpr (kCols == 8) {
                        gaps = gap_codes[nz];
                    } else {  // two 8-column halves joined by the gap across them
                        const uint32_t lo = nz & 0xFFu, hi = nz >> 8;
                        gaps = lo ? gap_codes[lo] : 0ull;
                        uint32_t pos = lo ? bits * (__popc(lo) - 1) : 0u;
                        if (lo && hi) {
                            gaps |= (uint64_t)(uint32_t)(8 + __ffs(hi) - 1 - (31 - __clz(lo)) - 1) << pos;
                            pos += bits;
                        }
                        if (hi) gaps |= gap_codes[hi] << pos;
                    }
                    codes |= ((uint64_t)first << sh) | (gaps << (sh + bits));
                }
            } else {
                uint32_t code[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int cc = (int)c + k;
                    code[k] = 0;
                    if ((nz >> k) & 1u) {
                        code[k] = (uint32_t)(cc - p - 1) & (maxd - 1);  // delta - 1
                        em |= 1u << k;
                        p = cc;
                    } else if (cc < L && cc > p && (((uint32_t)(cc - p)) & (maxd - 1)) == 0) {
                        code[k] = maxd - 1;
                        em |= 1u << k;
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if ((em >> k) & 1u) codes |= (uint64_t)code[k] << (__popc(em & ((1u << k) - 1u)) * bits);
            }
            const uint32_t n = __popc(em);
            // lane offsets of the entries
            uint32_t incl = n;
#pragma unroll
            for (int off = 1; off < kWarp; off <<= 1) {
                const uint32_t t = __shfl_up_sync(kFull, incl, off);
                if (lane >= off) incl += t;
            }
            const uint32_t tot = __shfl_sync(kFull, incl, kWarp - 1);
            const uint64_t o = (uint64_t)start + emitted + (incl - n);
            {
                // the lane's entries into the warp's value stage (predicated, no branch per column),
                // then the chunk's values to global memory with lane-consecutive 2-byte stores: scattered
                // 2-byte global stores would cost a partial L2 sector write each
                const uint32_t vs = static_cast<uint32_t>(__cvta_generic_to_shared(vstage)) + 2u * (incl - n);
#pragma unroll
                for (int k = 0; k < kCols; ++k) {
                    const uint16_t val = ((nz >> k) & 1u) ? h[k] : (uint16_t)0;  // pads are +0
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u16 [%0], %1;\n\t}" ::"r"(
                                     vs + 2u * __popc(em & ((1u << k) - 1u))),
                                 "h"(val), "r"(em & (1u << k))
                                 : "memory");
                }
                __syncwarp();
                uint16_t* vdst = values + (uint64_t)start + emitted;
                for (uint32_t i = lane; i < tot; i += kWarp) vdst[i] = vstage[i];
            }
            if (n) {
                const uint64_t bit0 = o * bits;
                const uint32_t sh = (uint32_t)(bit0 & 31u);
                const int rel = (int)((bit0 >> 5) - wb);
                // codes (<= 64 bits) shifted left by sh (< 32) spans up to 3 words
                const uint64_t lo64 = codes << sh;
                const uint32_t hi_bits = sh ? (uint32_t)(codes >> (64 - sh)) : 0u;
                atomicOr(&stage[rel], (uint32_t)lo64);
                if ((uint32_t)(lo64 >> 32)) atomicOr(&stage[rel + 1], (uint32_t)(lo64 >> 32));
                if (hi_bits) atomicOr(&stage[rel + 2], hi_bits);
            }
            __syncwarp();
            emitted += tot;
            const uint64_t end_bit = ((uint64_t)start + emitted) * bits;
            const uint64_t wend = end_bit >> 5;  // words [wb, wend) are complete
            const int ncomplete = (int)(wend - wb);
            for (int i = lane; i < ncomplete; i += kWarp) {
                const uint64_t gw = wb + i;
                if (gw == row_first_word && first_shared)
                    atomicOr(delta_words + gw, stage[i]);
                else
                    delta_words[gw] = stage[i];
            }
            __syncwarp();
            // move the partial word (and anything after it, all zero) to the front
            const uint32_t partial = (end_bit & 31u) ? stage[ncomplete] : 0u;
            __syncwarp();
            for (int i = lane; i <= ncomplete; i += kWarp) stage[i] = 0;  // beyond: still zero
            __syncwarp();
            if (lane == 0) stage[0] = partial;
            __syncwarp();
            wb = wend;
        }
        // the row's last partial word is shared with the next row
        if (lane == 0 && ((((uint64_t)start + emitted) * bits) & 31u)) atomicOr(delta_words + wb, stage[0]);
        __syncwarp();
    }
}

// Nonzero mask of the 16 fp16 values in w[0..7] (bit k = value k; +-0 are zero), byte-SIMD: per
// word (v & 0x7FFF7FFF) + 0x7FFF7FFF sets bit 15 / 31 iff the low / high half is nonzero (no carry
// crosses bit 15), PRMT packs those bytes four at a time and one multiply gathers the four flags.
__device__ __forceinline__ uint32_t nz_mask16(const uint32_t (&w)[8]) {
    uint32_t m = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t t0 = (w[2 * q] & 0x7FFF7FFFu) + 0x7FFF7FFFu;
        const uint32_t t1 = (w[2 * q + 1] & 0x7FFF7FFFu) + 0x7FFF7FFFu;
        const uint32_t b = (__byte_perm(t0, t1, 0x7531) >> 7) & 0x01010101u;  // flags of values 4q..4q+3
        m |= ((b * 0x01020408u) >> 24) << (4 * q);  // flag k of the group -> bit 24 + k
    }
    return m;
}

// b_delta = 4 emitter (the benchmark width): the same classification as emit_rows<true, 16>, with
// the output path rebuilt around 16-byte stores.  Stage position q of a warp's value stage is
// global value vbase + q with vbase 8-aligned, so every complete 8-value group leaves as one
// 16-byte store; the partial group rolls to the front of the stage for the next 512 columns.  A
// lane's entries go to the stage with one predicated store each at a running address (no popc
// per column).  Codewords (nibbles) are OR-ed into a word stage the same way and complete words
// leave as plain 32-bit stores; the row's first and last words, shared with the neighbouring
// rows, are OR-ed into global memory.
constexpr int kE4Warps = 8;
constexpr uint32_t kE4Step = kWarp * 16;  // columns per warp step

#ifndef MACKO_E4_MINB
#define MACKO_E4_MINB 4
#endif
__global__ void __launch_bounds__(kE4Warps * kWarp, MACKO_E4_MINB)
    emit_rows4(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, const uint32_t* row_ptrs,
               const int32_t* lastcol, uint16_t* values, uint32_t* delta_words) {
    constexpr uint32_t bits = 4, maxd = 16;
    __shared__ __align__(16) uint16_t vst_all[kE4Warps][kE4Step + 16];
    __shared__ uint32_t cst_all[kE4Warps][kE4Step / 8 + 8];
    __shared__ uint64_t gap_codes[256];
    for (uint32_t pat = threadIdx.x; pat < 256; pat += blockDim.x) {
        uint64_t v = 0;
        uint32_t i = 0, rest = pat;
        int prev = -1;
        while (rest) {
            const int k = __ffs(rest) - 1;
            rest &= rest - 1;
            if (prev >= 0) v |= (uint64_t)(uint32_t)(k - prev - 1) << (bits * i++);
            prev = k;
        }
        gap_codes[pat] = v;
    }
    __syncthreads();
    const int lane = threadIdx.x & (kWarp - 1);
    uint16_t* vst = vst_all[threadIdx.x >> 5];
    uint32_t* cst = cst_all[threadIdx.x >> 5];
    const uint32_t vst_s = static_cast<uint32_t>(__cvta_generic_to_shared(vst));
    const uint32_t nwarps = gridDim.x * kE4Warps;
    const bool vec_base = ((reinterpret_cast<uintptr_t>(dense) | (ld * 2)) & 15u) == 0;
    for (uint32_t r = blockIdx.x * kE4Warps + (threadIdx.x >> 5); r < rows; r += nwarps) {
        const uint32_t start = row_ptrs[r], end = row_ptrs[r + 1];
        if (start == end) continue;
        const int L = lastcol[r];
        const uint16_t* row = dense + (uint64_t)r * ld;
        uint32_t vbase = start & ~7u, vlo = start & 7u, vP = vlo;  // value stage: q <-> vbase + q
        uint32_t wbase = start >> 3, cP = start & 7u;              // code stage: nibble q <-> 8 wbase + q
        const uint32_t first_word = wbase;
        bool first_open = (start & 7u) != 0;  // the row's first word still holds the previous row's nibbles
        for (int i = lane; i < (int)(kE4Step / 8 + 8); i += kWarp) cst[i] = 0;
        __syncwarp();
        int carry = -1;
        uint4 next[2];
        next[0] = fetch8(row, 16 * lane, cols, vec_base);
        next[1] = fetch8(row, 16 * lane + 8, cols, vec_base);
        for (uint32_t c0 = 0; c0 < cols && (int)c0 <= L; c0 += kE4Step) {
            const uint32_t c = c0 + 16 * lane;
            const uint32_t w[8] = {next[0].x, next[0].y, next[0].z, next[0].w, next[1].x, next[1].y, next[1].z, next[1].w};
            const uint32_t nz = nz_mask16(w);
            if (c0 + kE4Step < cols && (int)(c0 + kE4Step) <= L) {
                if (vec_base && c0 + 2 * kE4Step <= cols) {  // whole next step in bounds: plain 16-byte loads
                    next[0] = __ldg(reinterpret_cast<const uint4*>(row + c + kE4Step));
                    next[1] = __ldg(reinterpret_cast<const uint4*>(row + c + kE4Step + 8));
                } else {
                    next[0] = fetch8(row, c + kE4Step, cols, vec_base);
                    next[1] = fetch8(row, c + kE4Step + 8, cols, vec_base);
                }
            }
            const int lane_last = nz ? (int)(c + 31 - __clz(nz)) : -1;
            const int p = prev_nonzero(lane_last, lane, carry);
            const uint32_t pb = pad_bit<16>(nz, (int)c, p, L, bits);
            const uint32_t em = nz | pb;
            uint64_t codes = pb ? (uint64_t)(maxd - 1) : 0ull;
            if (nz) {
                const uint32_t sh = pb ? bits : 0u;
                const uint32_t first = (uint32_t)((int)c + __ffs(nz) - 2 - p) & (maxd - 1);
                const uint32_t lo = nz & 0xFFu, hi = nz >> 8;
                uint64_t gaps = lo ? gap_codes[lo] : 0ull;
                uint32_t pos = lo ? bits * (__popc(lo) - 1) : 0u;
                if (lo && hi) {
                    gaps |= (uint64_t)(uint32_t)(8 + __ffs(hi) - 1 - (31 - __clz(lo)) - 1) << pos;
                    pos += bits;
                }
                if (hi) gaps |= gap_codes[hi] << pos;
                codes |= ((uint64_t)first << sh) | (gaps << (sh + bits));
            }
            const uint32_t n = __popc(em);
            uint32_t incl = n;
#pragma unroll
            for (int off = 1; off < kWarp; off <<= 1) {
                const uint32_t t = __shfl_up_sync(kFull, incl, off);
                if (lane >= off) incl += t;
            }
            const uint32_t tot = __shfl_sync(kFull, incl, kWarp - 1);
            // values: the pad (+0; it precedes the lane's nonzeros) then one predicated 2-byte store
            // per nonzero at a running stage address, straight from the loaded words
            uint32_t va = vst_s + 2u * (vP + incl - n);
            if (pb) {
                asm volatile("st.shared.u16 [%0], %1;" ::"r"(va), "h"((uint16_t)0) : "memory");
                va += 2u;
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if ((nz >> k) & 1u) {
                    const uint32_t v32 = (k & 1) ? w[k >> 1] >> 16 : w[k >> 1];
                    asm volatile("st.shared.u16 [%0], %1;" ::"r"(va), "r"(v32) : "memory");
                    va += 2u;
                }
            }
            // codewords: nibble position cP + (incl - n); <= 16 nibbles span <= 3 words
            if (n) {
                const uint32_t np = cP + incl - n, wi = np >> 3, sh = (np & 7u) * 4u;
                const uint64_t lo64 = codes << sh;
                atomicOr(&cst[wi], (uint32_t)lo64);
                if ((uint32_t)(lo64 >> 32)) atomicOr(&cst[wi + 1], (uint32_t)(lo64 >> 32));
                if (sh && (uint32_t)(codes >> (64 - sh))) atomicOr(&cst[wi + 2], (uint32_t)(codes >> (64 - sh)));
            }
            __syncwarp();
            vP += tot;
            cP += tot;
            // complete 8-value groups -> 16-byte stores (the row's first group, shared with the
            // previous row, value by value)
            const uint32_t nfull = vP >> 3;
            uint32_t j0 = 0;
            if (vlo && nfull) {
                if ((uint32_t)lane >= vlo && lane < 8) values[vbase + lane] = vst[lane];
                j0 = 1;
                vlo = 0;
            }
            for (uint32_t j = j0 + lane; j < nfull; j += kWarp)
                *reinterpret_cast<uint4*>(values + vbase + 8u * j) = *reinterpret_cast<const uint4*>(vst + 8u * j);
            // complete code words
            const uint32_t nw = cP >> 3;
            for (uint32_t i = lane; i < nw; i += kWarp) {
                if (first_open && wbase + i == first_word)
                    atomicOr(delta_words + first_word, cst[i]);
                else
                    delta_words[wbase + i] = cst[i];
            }
            if (nw) first_open = false;
            __syncwarp();
            // roll the partial value group and the partial code word to the front
            const uint32_t rem = vP - 8u * nfull;
            const uint16_t tv = (uint32_t)lane < rem ? vst[8u * nfull + lane] : (uint16_t)0;
            const uint32_t tw = cst[nw];
            __syncwarp();
            for (uint32_t i = lane; i <= nw + 2u; i += kWarp) cst[i] = 0;
            __syncwarp();
            if ((uint32_t)lane < rem) vst[lane] = tv;
            if (lane == 0) cst[0] = tw;
            __syncwarp();
            vbase += 8u * nfull;
            vP = rem;
            wbase += nw;
            cP &= 7u;
        }
        // row end: the last partial value group value by value, the last partial word OR-ed (the
        // next row's entries share it)
        if ((uint32_t)lane >= vlo && (uint32_t)lane < vP) values[vbase + lane] = vst[lane];
        if (lane == 0 && cP) atomicOr(delta_words + wbase, cst[0]);
        __syncwarp();
    }
}

}  // namespace

cudaError_t launch_count_rows(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, uint32_t bits,
                              uint32_t* counts, int32_t* lastcol, int sms, cudaStream_t s) {
    const int grid = (int)std::min<uint64_t>((rows + kCompressWarpsPerCta - 1) / kCompressWarpsPerCta, (uint64_t)sms * 8);
    if (grid > 0) {
        const dim3 b(kCompressWarpsPerCta * kWarp);
        if (bits == 4)
            count_rows<true, 16><<<grid, b, 0, s>>>(dense, ld, rows, cols, bits, counts, lastcol);
        else if (bits == 8)
            count_rows<true, 8><<<grid, b, 0, s>>>(dense, ld, rows, cols, bits, counts, lastcol);
        else
            count_rows<false, 8><<<grid, b, 0, s>>>(dense, ld, rows, cols, bits, counts, lastcol);
    }
    return cudaGetLastError();
}

cudaError_t launch_scan_counts(const uint32_t* counts, uint32_t rows, uint32_t* row_ptrs, unsigned long long* total,
                               cudaStream_t s) {
    scan_counts<<<1, 1024, 0, s>>>(counts, rows, row_ptrs, total);
    return cudaGetLastError();
}

cudaError_t launch_emit_rows(const uint16_t* dense, uint64_t ld, uint32_t rows, uint32_t cols, uint32_t bits,
                             const uint32_t* row_ptrs, const int32_t* lastcol, uint16_t* values, uint32_t* delta_words,
                             int sms, cudaStream_t s) {
    const int grid = (int)std::min<uint64_t>((rows + kCompressWarpsPerCta - 1) / kCompressWarpsPerCta, (uint64_t)sms * 8);
    if (grid > 0) {
        const dim3 b(kCompressWarpsPerCta * kWarp);
        if (bits == 4)
            emit_rows4<<<grid, b, 0, s>>>(dense, ld, rows, cols, row_ptrs, lastcol, values, delta_words);
        else if (bits == 8)
            emit_rows<true, 8><<<grid, b, 0, s>>>(dense, ld, rows, cols, bits, row_ptrs, lastcol, values, delta_words);
        else
            emit_rows<false, 8><<<grid, b, 0, s>>>(dense, ld, rows, cols, bits, row_ptrs, lastcol, values, delta_words);
    }
    return cudaGetLastError();
}

}  // namespace mk
