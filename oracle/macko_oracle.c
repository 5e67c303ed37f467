/*
 * macko_oracle.c — CPU ORACLE (test infrastructure only; see macko_oracle.h).
 *
 * Plain-C restatement of the reference MACKO algorithm.  Each function names the reference
 * location it follows.  Reference paths are relative to /root/reference.
 */
#include "macko_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* mo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------------------------
 * fp16 — proj/src/fp16.hpp:9-17 (Half = raw bits, ±0 test), fp16.cpp:8-35 (half_to_float,
 * exact incl. subnormals, NaN payload kept without quieting), fp16.cpp:37-73 (float_to_half,
 * round-to-nearest-even, subnormals, overflow to ±inf, NaN -> quiet 0x200|man>>13).
 * ---------------------------------------------------------------------------------------- */
int mo_half_is_zero(uint16_t h) { return (h & 0x7FFFu) == 0; }

float mo_half_to_float(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const uint32_t ex = (h >> 10) & 0x1Fu, man = h & 0x3FFu;
    uint32_t bits;
    if (ex == 0x1Fu) {
        bits = sign | 0x7F800000u | (man << 13);
    } else if (ex == 0) {
        /* zero or subnormal: man * 2^-24 is exact in binary32 */
        float v = (float)man * 5.9604644775390625e-8f;
        memcpy(&bits, &v, 4);
        bits |= sign;
    } else {
        bits = sign | ((ex + 112u) << 23) | (man << 13);
    }
    float out;
    memcpy(&out, &bits, 4);
    return out;
}

uint16_t mo_float_to_half(float x) {
    uint32_t f;
    memcpy(&f, &x, 4);
    const uint16_t sign = (uint16_t)((f >> 16) & 0x8000u);
    const uint32_t a = f & 0x7FFFFFFFu;
    if (a >= 0x7F800000u) { /* inf / nan */
        if (a == 0x7F800000u) return sign | 0x7C00u;
        return (uint16_t)(sign | 0x7C00u | 0x200u | ((a & 0x7FFFFFu) >> 13));
    }
    if (a >= 0x477FF000u) return sign | 0x7C00u; /* >= 65520 rounds (ties-even) to inf */
    if (a <= 0x33000000u) return sign;           /* <= 2^-25 rounds to zero */
    const int e = (int)(a >> 23) - 127;
    const uint32_t mant = (a & 0x7FFFFFu) | 0x800000u; /* 24 significant bits */
    uint32_t q, rem, halfway;
    uint32_t h;
    if (e < -14) { /* binary16 subnormal: units of 2^-24 */
        const int shift = -e - 1;                /* 14..24 */
        q = mant >> shift;
        rem = mant & ((1u << shift) - 1u);
        halfway = 1u << (shift - 1);
        h = q;
    } else {
        q = mant >> 13;
        rem = mant & 0x1FFFu;
        halfway = 0x1000u;
        h = ((uint32_t)(e + 15) << 10) + (q - 0x400u);
    }
    if (rem > halfway || (rem == halfway && (h & 1u))) h += 1; /* carry may reach the exponent */
    return (uint16_t)(sign | h);
}

/* ------------------------------------------------------------------------------------------
 * Delta packing — proj/src/bitpack.hpp:9-25, bitpack.cpp:8-52: codeword = delta-1 stored in
 * `bits` bits, 8/bits codewords per byte, element i at bit (i mod (8/bits))*bits of byte
 * i/(8/bits) (least-significant first); bits in {1,2,4,8}; out-of-range deltas rejected.
 * ---------------------------------------------------------------------------------------- */
int mo_is_valid_delta_bits(unsigned bits) { return bits == 1 || bits == 2 || bits == 4 || bits == 8; }

static inline uint32_t code_at(const uint8_t* bytes, uint64_t i, unsigned bits) {
    const unsigned per = 8u / bits;
    const uint32_t mask = bits == 8 ? 0xFFu : ((1u << bits) - 1u);
    return (bytes[i / per] >> ((unsigned)(i % per) * bits)) & mask;
}

static inline void put_code(uint8_t* bytes, uint64_t i, unsigned bits, uint32_t code) {
    const unsigned per = 8u / bits;
    bytes[i / per] |= (uint8_t)(code << ((unsigned)(i % per) * bits));
}

int mo_pack_deltas(const uint32_t* deltas, uint64_t n, unsigned bits, uint8_t* out) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    const unsigned per = 8u / bits;
    const uint32_t maxd = 1u << bits;
    memset(out, 0, (size_t)((n + per - 1) / per));
    for (uint64_t i = 0; i < n; ++i) {
        if (deltas[i] < 1 || deltas[i] > maxd) return fail(MO_EINVAL, "delta out of range [1, 2^bits]");
        put_code(out, i, bits, deltas[i] - 1);
    }
    return MO_OK;
}

int mo_unpack_deltas(const uint8_t* bytes, uint64_t n, unsigned bits, uint32_t* out) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    for (uint64_t i = 0; i < n; ++i) out[i] = code_at(bytes, i, bits) + 1;
    return MO_OK;
}

/* ---- proj/src/matrix.hpp:73-81: payload sizes with 16-byte tail padding ---- */
uint64_t mo_align_up(uint64_t n, uint64_t a) { return (n + a - 1) / a * a; }
uint64_t mo_values_bytes(uint64_t pad_nnz) { return mo_align_up(pad_nnz * 2, 16); }
uint64_t mo_delta_bytes(uint64_t pad_nnz, unsigned bits) { return mo_align_up((pad_nnz * bits + 7) / 8, 16); }

/* ------------------------------------------------------------------------------------------
 * csr_from_dense — proj/src/convert.hpp:8-10 (declaration): exact nonzeros in
 * row-major order; anything equal to zero in binary16 (+0 or -0) is dropped.
 * ---------------------------------------------------------------------------------------- */
uint64_t mo_csr_count(const uint16_t* dense, uint64_t rows, uint64_t cols, uint32_t* rp) {
    uint64_t nnz = 0;
    rp[0] = 0;
    for (uint64_t r = 0; r < rows; ++r) {
        const uint16_t* row = dense + r * cols;
        for (uint64_t c = 0; c < cols; ++c) nnz += !mo_half_is_zero(row[c]);
        rp[r + 1] = (uint32_t)nnz;
    }
    return nnz;
}

void mo_csr_fill(const uint16_t* dense, uint64_t rows, uint64_t cols, const uint32_t* rp,
                 uint16_t* values, uint32_t* col_idx) {
    for (uint64_t r = 0; r < rows; ++r) {
        uint64_t o = rp[r];
        const uint16_t* row = dense + r * cols;
        for (uint64_t c = 0; c < cols; ++c)
            if (!mo_half_is_zero(row[c])) { values[o] = row[c]; col_idx[o] = (uint32_t)c; ++o; }
    }
}

/* ------------------------------------------------------------------------------------------
 * macko_from_csr — proj/src/convert.hpp:12-16, SPEC.md:64-72 and the design decisions at
 * SPEC.md:111-118.  Per row, prev starts at the virtual column -1; for each nonzero at column
 * c: while c - prev > 2^bits emit a padding entry (value +0, delta 2^bits) and advance prev by
 * 2^bits; then emit (value, c - prev).  No padding after the last nonzero of a row.  Row
 * pointers are u32 element offsets (SPEC.md:403 caps pad_nnz below 2^32).  Both payload
 * arrays are zero-padded to 16-byte multiples (proj/src/matrix.hpp:57-59).
 * ---------------------------------------------------------------------------------------- */
typedef struct {
    uint16_t* values; /* NULL in the count pass */
    uint8_t* deltas;
    uint64_t at;      /* next element offset */
    unsigned bits;
    int64_t prev;
    uint32_t maxd;
} row_encoder;

static inline void enc_emit(row_encoder* en, uint16_t v, uint32_t delta) {
    if (en->values) {
        en->values[en->at] = v;
        /* atomic OR: in the threaded encoder two row ranges may share a codeword byte */
        const unsigned per = 8u / en->bits;
        __atomic_fetch_or(&en->deltas[en->at / per], (uint8_t)((delta - 1) << ((unsigned)(en->at % per) * en->bits)),
                          __ATOMIC_RELAXED);
    }
    ++en->at;
}

/* Encode one nonzero at column c (caller guarantees c > prev). */
static inline void enc_push(row_encoder* en, int64_t c, uint16_t v) {
    while (c - en->prev > (int64_t)en->maxd) {
        enc_emit(en, 0, en->maxd);
        en->prev += en->maxd;
    }
    enc_emit(en, v, (uint32_t)(c - en->prev));
    en->prev = c;
}

static int encode_csr(uint64_t rows, uint64_t cols, const uint32_t* crp, const uint32_t* ccols,
                      const uint16_t* cvals, unsigned bits, uint32_t* mrp, uint16_t* values,
                      uint8_t* deltas, uint64_t* pad_nnz_out) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    row_encoder en = {values, deltas, 0, bits, -1, 1u << bits};
    if (mrp && !values) mrp[0] = 0;
    for (uint64_t r = 0; r < rows; ++r) {
        en.prev = -1;
        if (values) en.at = mrp[r];
        for (uint64_t k = crp[r]; k < crp[r + 1]; ++k) {
            const int64_t c = ccols[k];
            if ((uint64_t)c >= cols) return fail(MO_EINVAL, "column index out of range");
            if (c <= en.prev) return fail(MO_EINVAL, "columns not strictly increasing within a row");
            enc_push(&en, c, values ? cvals[k] : 0);
        }
        if (!values) {
            if (en.at > 0xFFFFFFFFull) return fail(MO_EINVAL, "pad_nnz does not fit u32 row pointers");
            mrp[r + 1] = (uint32_t)en.at;
        }
    }
    if (pad_nnz_out) *pad_nnz_out = en.at;
    return MO_OK;
}

int mo_macko_count(uint64_t rows, uint64_t cols, const uint32_t* crp, const uint32_t* ccols,
                   unsigned bits, uint32_t* mrp, uint64_t* pad_nnz) {
    return encode_csr(rows, cols, crp, ccols, NULL, bits, mrp, NULL, NULL, pad_nnz);
}

int mo_macko_fill(uint64_t rows, uint64_t cols, const uint32_t* crp, const uint32_t* ccols,
                  const uint16_t* cvals, unsigned bits, const uint32_t* mrp, uint16_t* values,
                  uint8_t* deltas) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    const uint64_t pad_nnz = rows ? mrp[rows] : 0;
    memset(values, 0, (size_t)mo_values_bytes(pad_nnz));
    memset(deltas, 0, (size_t)mo_delta_bytes(pad_nnz, bits));
    return encode_csr(rows, cols, crp, ccols, cvals, bits, (uint32_t*)mrp, values, deltas, NULL);
}

/* Dense -> MACKO without materialising CSR: identical output (same greedy loop fed by the
 * row-major nonzeros that csr_from_dense would produce). */
static int encode_dense(const uint16_t* dense, uint64_t rows, uint64_t cols, unsigned bits,
                        uint32_t* mrp, uint16_t* values, uint8_t* deltas, uint64_t* pad_nnz_out) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    row_encoder en = {values, deltas, 0, bits, -1, 1u << bits};
    if (!values) mrp[0] = 0;
    for (uint64_t r = 0; r < rows; ++r) {
        const uint16_t* row = dense + r * cols;
        en.prev = -1;
        if (values) en.at = mrp[r];
        for (uint64_t c = 0; c < cols; ++c)
            if (!mo_half_is_zero(row[c])) enc_push(&en, (int64_t)c, row[c]);
        if (!values) {
            if (en.at > 0xFFFFFFFFull) return fail(MO_EINVAL, "pad_nnz does not fit u32 row pointers");
            mrp[r + 1] = (uint32_t)en.at;
        }
    }
    if (pad_nnz_out) *pad_nnz_out = en.at;
    return MO_OK;
}

int mo_encode_dense_count(const uint16_t* dense, uint64_t rows, uint64_t cols, unsigned bits,
                          uint32_t* rp, uint64_t* pad_nnz) {
    return encode_dense(dense, rows, cols, bits, rp, NULL, NULL, pad_nnz);
}

int mo_encode_dense_fill(const uint16_t* dense, uint64_t rows, uint64_t cols, unsigned bits,
                         const uint32_t* rp, uint16_t* values, uint8_t* deltas) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    const uint64_t pad_nnz = rows ? rp[rows] : 0;
    memset(values, 0, (size_t)mo_values_bytes(pad_nnz));
    memset(deltas, 0, (size_t)mo_delta_bytes(pad_nnz, bits));
    return encode_dense(dense, rows, cols, bits, (uint32_t*)rp, values, deltas, NULL);
}

/* ------------------------------------------------------------------------------------------
 * Row decode — proj/src/convert.hpp:29-42 (for_each_row_element): col starts at -1 and adds
 * each decoded delta over [row_pointers[r], row_pointers[r+1]); the tail is never read.
 * ---------------------------------------------------------------------------------------- */

/* dense_from_macko — convert.hpp:18-20, SPEC.md:74-82 (decoded column >= C is corruption). */
int mo_dense_from_macko(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values,
                        const uint8_t* deltas, const uint32_t* rp, uint16_t* dense) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    memset(dense, 0, (size_t)(rows * cols * 2));
    for (uint64_t r = 0; r < rows; ++r) {
        int64_t col = -1;
        for (uint64_t e = rp[r]; e < rp[r + 1]; ++e) {
            col += code_at(deltas, e, bits) + 1;
            if ((uint64_t)col >= cols) return fail(MO_EFORMAT, "decoded column index past the column bound");
            dense[r * cols + (uint64_t)col] = values[e];
        }
    }
    return MO_OK;
}

/* validate_macko — convert.hpp:25-27, invariants SPEC.md:44-51. */
int mo_validate_macko(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values,
                      uint64_t n_values, const uint8_t* deltas, uint64_t n_delta_bytes,
                      const uint32_t* rp) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    if (rp[0] != 0) return fail(MO_EFORMAT, "row_pointers[0] must be 0");
    for (uint64_t r = 0; r < rows; ++r)
        if (rp[r + 1] < rp[r]) return fail(MO_EFORMAT, "row_pointers not monotone");
    const uint64_t pad_nnz = rp[rows];
    if (n_values < pad_nnz) return fail(MO_EFORMAT, "values shorter than pad_nnz");
    if (n_delta_bytes * 8 < pad_nnz * bits) return fail(MO_EFORMAT, "packed_deltas shorter than pad_nnz");
    for (uint64_t r = 0; r < rows; ++r) {
        int64_t col = -1;
        for (uint64_t e = rp[r]; e < rp[r + 1]; ++e) {
            col += code_at(deltas, e, bits) + 1;
            if ((uint64_t)col >= cols) return fail(MO_EFORMAT, "decoded column index past the column bound");
            if (values[e] == 0x8000u) return fail(MO_EFORMAT, "padding value must be +0");
        }
    }
    return MO_OK;
}

/* padding_count — convert.hpp:22-23: zero-valued non-tail entries. */
uint64_t mo_padding_count(uint64_t rows, const uint16_t* values, const uint32_t* rp) {
    uint64_t n = 0;
    const uint64_t pad_nnz = rows ? rp[rows] : 0;
    for (uint64_t e = 0; e < pad_nnz; ++e) n += mo_half_is_zero(values[e]);
    return n;
}

/* ------------------------------------------------------------------------------------------
 * Executors — SPEC.md:210-296.
 * ---------------------------------------------------------------------------------------- */

/* dense_mv — SPEC.md:225-233: fp16 products widened to fp32, sequential, one RNE. */
void mo_dense_mv(const uint16_t* dense, uint64_t rows, uint64_t cols, const uint16_t* x, uint16_t* y) {
    for (uint64_t r = 0; r < rows; ++r) {
        float acc = 0.0f;
        const uint16_t* row = dense + r * cols;
        for (uint64_t c = 0; c < cols; ++c) acc += mo_half_to_float(row[c]) * mo_half_to_float(x[c]);
        y[r] = mo_float_to_half(acc);
    }
}

typedef struct {
    uint64_t r0, r1, cols;
    unsigned bits;
    const uint16_t* values;
    const uint8_t* deltas;
    const uint32_t* rp;
    const float* xf;
    uint16_t* y;
    int status;
} spmv_job;

/* reference_spmv — SPEC.md:235-243: decode each row (convert.hpp:32-42), accumulate
 * value*x[col] left to right in fp32 with padding entries included, one RNE per row. */
static void* spmv_rows(void* arg) {
    spmv_job* j = (spmv_job*)arg;
    for (uint64_t r = j->r0; r < j->r1; ++r) {
        float acc = 0.0f;
        int64_t col = -1;
        for (uint64_t e = j->rp[r]; e < j->rp[r + 1]; ++e) {
            col += code_at(j->deltas, e, j->bits) + 1;
            if ((uint64_t)col >= j->cols) { j->status = MO_EFORMAT; return NULL; }
            acc += mo_half_to_float(j->values[e]) * j->xf[col];
        }
        j->y[r] = mo_float_to_half(acc);
    }
    return NULL;
}

int mo_reference_spmv(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values,
                      const uint8_t* deltas, const uint32_t* rp, const uint16_t* x, uint16_t* y,
                      int nthreads) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    float* xf = (float*)malloc((size_t)(cols ? cols : 1) * sizeof(float));
    if (!xf) return fail(MO_EINVAL, "out of memory");
    for (uint64_t c = 0; c < cols; ++c) xf[c] = mo_half_to_float(x[c]);
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > rows) nthreads = rows ? (int)rows : 1;
    spmv_job* jobs = (spmv_job*)calloc((size_t)nthreads, sizeof(spmv_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        spmv_job j = {rows * t / nthreads, rows * (t + 1) / nthreads, cols, bits, values, deltas, rp, xf, y, MO_OK};
        jobs[t] = j;
    }
    if (nthreads == 1) {
        spmv_rows(&jobs[0]);
    } else {
        for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, spmv_rows, &jobs[t]);
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    }
    int st = MO_OK;
    for (int t = 0; t < nthreads; ++t) if (jobs[t].status != MO_OK) st = jobs[t].status;
    free(jobs); free(th); free(xf);
    if (st != MO_OK) return fail(st, "decoded column index past the column bound");
    return MO_OK;
}

/* Algorithm 1 — PAPER.md:377-391: inclusive doubling scan by shfl_up with
 * offsets 1,2,4,8,16 (a lane below the offset keeps its value), minus the own local sum. */
void mo_warp_prefix_sum(const uint32_t* local, uint32_t* out) {
    uint32_t p[32], q[32];
    for (int l = 0; l < 32; ++l) p[l] = local[l];
    for (int off = 1; off < 32; off *= 2) {
        for (int l = 0; l < 32; ++l) q[l] = l >= off ? p[l] + p[l - off] : p[l];
        memcpy(p, q, sizeof p);
    }
    for (int l = 0; l < 32; ++l) out[l] = p[l] - local[l];
}

/* xor-butterfly over 32 lane accumulators (offsets 16,8,4,2,1); every lane ends with the same
 * bits, lane 0's value is returned.  This is the B200 kernel's reduction tree. */
static float lane_tree(const float* acc) {
    float a[32], b[32];
    memcpy(a, acc, sizeof a);
    for (int off = 16; off >= 1; off /= 2) {
        for (int l = 0; l < 32; ++l) b[l] = a[l] + a[l ^ off];
        memcpy(a, b, sizeof a);
    }
    return a[0];
}

/* warp_spmv — SPEC.md:255-264 with the design decisions at SPEC.md:281-287: one emulated warp
 * per row; ROMA aligns the row start down to 8 elements (16 B of values) and masks elements
 * before the row start; 256 elements per step (32 lanes x 8); columns reconstructed from
 * Algorithm 1's exclusive prefix of lane-local delta sums plus a running base that starts at
 * -1 and advances by lane 31's inclusive total; lanes past the row end contribute nothing;
 * lane accumulators reduced once after the row; one RNE. */
int mo_warp_spmv(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values,
                 const uint8_t* deltas, const uint32_t* rp, const uint16_t* x, uint16_t* y) {
    if (bits != 4 && bits != 1 && bits != 2 && bits != 8)
        return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    for (uint64_t r = 0; r < rows; ++r) {
        const uint64_t s = rp[r], e = rp[r + 1];
        float acc[32] = {0};
        int64_t base = -1;
        for (uint64_t a = s & ~(uint64_t)7; a < e; a += 256) {
            uint32_t local[32], excl[32];
            for (int l = 0; l < 32; ++l) {
                local[l] = 0;
                for (int k = 0; k < 8; ++k) {
                    const uint64_t i = a + 8 * (uint64_t)l + k;
                    if (i >= s && i < e) local[l] += code_at(deltas, i, bits) + 1;
                }
            }
            mo_warp_prefix_sum(local, excl);
            for (int l = 0; l < 32; ++l) {
                int64_t col = base + excl[l];
                for (int k = 0; k < 8; ++k) {
                    const uint64_t i = a + 8 * (uint64_t)l + k;
                    if (i < s || i >= e) continue;
                    col += code_at(deltas, i, bits) + 1;
                    if ((uint64_t)col >= cols) return fail(MO_EFORMAT, "decoded column index past the column bound");
                    acc[l] += mo_half_to_float(values[i]) * mo_half_to_float(x[col]);
                }
            }
            base += excl[31] + local[31];
        }
        y[r] = mo_float_to_half(lane_tree(acc));
    }
    return MO_OK;
}

/* The B200 kernel's order: as warp_spmv, but the row's steps (256 elements from
 * the ROMA-aligned start) are grouped into units of `unit_steps` steps, the last unit absorbing
 * a remainder shorter than `unit_steps` (a row of T steps has max(1, T / unit_steps) units).
 * At every unit end the lane accumulators are tree-reduced and the unit sum is added to a
 * sequential row accumulator that starts at +0.  unit_steps = 0 means "one unit per row"
 * (= warp_spmv). */
int mo_b200_order_spmv(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values,
                       const uint8_t* deltas, const uint32_t* rp, const uint16_t* x, uint16_t* y,
                       unsigned unit_steps) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    for (uint64_t r = 0; r < rows; ++r) {
        const uint64_t s = rp[r], e = rp[r + 1];
        const uint64_t a0 = s & ~(uint64_t)7;
        const uint64_t T = e > s ? (e - a0 + 255) / 256 : 0;
        uint64_t n_units = 1;
        if (unit_steps && T >= unit_steps) n_units = T / unit_steps;
        float row_acc = 0.0f;
        int64_t col = -1;
        uint64_t i = s;
        for (uint64_t j = 0; j < n_units && T; ++j) {
            float acc[32] = {0};
            const uint64_t t_end = (j + 1 == n_units) ? T : (j + 1) * unit_steps;
            for (uint64_t t = unit_steps ? j * unit_steps : 0; t < t_end; ++t) {
                const uint64_t a = a0 + 256 * t;
                const uint64_t hi = a + 256 < e ? a + 256 : e;
                for (; i < hi; ++i) {
                    col += code_at(deltas, i, bits) + 1;
                    if ((uint64_t)col >= cols) return fail(MO_EFORMAT, "decoded column index past the column bound");
                    acc[(i - a) / 8] += mo_half_to_float(values[i]) * mo_half_to_float(x[col]);
                }
            }
            row_acc += lane_tree(acc);
        }
        y[r] = mo_float_to_half(row_acc);
    }
    return MO_OK;
}

/* ------------------------------------------------------------------------------------------
 * Synthetic inputs.  gen_random leaves the magnitude distribution and RNG
 * undocumented (generate.cpp is absent), so this generator is ours and identical on CPU and
 * GPU: splitmix64 of seed ^ idx*K; entry kept iff the top 24 hash bits < round(d*2^24);
 * float mode: value (u-32768)*2^-15 rounded to fp16 (u = low 16 bits, u=32768 -> 32769 so
 * kept entries are never zero); integer mode: value in [-8,8]\{0}, vector in [-8,8].
 * ---------------------------------------------------------------------------------------- */
static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint32_t mo_density_threshold(double d) {
    if (!(d > 0)) return 0;
    if (d >= 1) return 1u << 24;
    return (uint32_t)floor(d * 16777216.0 + 0.5);
}

uint16_t mo_gen_value(uint64_t seed, uint64_t idx, uint32_t thr24, int int_mode) {
    const uint64_t h = mix64(seed ^ (idx * 0xD1B54A32D192ED03ull));
    if ((uint32_t)(h >> 40) >= thr24) return 0;
    if (int_mode) {
        int v = (int)(h & 15u) - 8;
        if (v >= 0) v += 1;
        return mo_float_to_half((float)v);
    }
    uint32_t u = (uint32_t)(h & 0xFFFFu);
    if (u == 32768u) u = 32769u;
    return mo_float_to_half((float)((int32_t)u - 32768) * (1.0f / 32768.0f));
}

void mo_gen_dense(uint64_t rows, uint64_t cols, uint32_t thr24, uint64_t seed, int int_mode, uint16_t* out) {
    const uint64_t n = rows * cols;
    for (uint64_t i = 0; i < n; ++i) out[i] = mo_gen_value(seed, i, thr24, int_mode);
}

void mo_gen_vector(uint64_t n, uint64_t seed, int int_mode, uint16_t* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t h = mix64(seed ^ (i * 0xD1B54A32D192ED03ull));
        if (int_mode) {
            out[i] = mo_float_to_half((float)((int)((h & 0xFFFFu) % 17u) - 8));
        } else {
            out[i] = mo_float_to_half((float)((int32_t)(h & 0xFFFFu) - 32768) * (1.0f / 32768.0f));
        }
    }
}

/* gen_worst_case — SPEC.md:171-179: runs of exactly `zero_run` zeros, each followed by one
 * nonzero (value 1.0) so that every run forces floor(zero_run/2^bits) pads. */
void mo_gen_worst_case(uint64_t rows, uint64_t cols, uint64_t zero_run, uint16_t* out) {
    for (uint64_t r = 0; r < rows; ++r)
        for (uint64_t c = 0; c < cols; ++c)
            out[r * cols + c] = (c % (zero_run + 1) == zero_run) ? 0x3C00u : 0;
}

/* spmv_traffic — SPEC.md:333-341: stored matrix arrays + 2C (x) + 2R (y). */
uint64_t mo_spmv_traffic_bytes(uint64_t rows, uint64_t cols, uint64_t pad_nnz, unsigned bits) {
    return mo_values_bytes(pad_nnz) + mo_delta_bytes(pad_nnz, bits) + 4 * (rows + 1) + 2 * cols + 2 * rows;
}

uint64_t mo_dense_traffic_bytes(uint64_t rows, uint64_t cols) { return 2 * rows * cols + 2 * rows + 2 * cols; }

/* Array forms for vectorised tests. */
void mo_float_to_half_array(const float* x, uint64_t n, uint16_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = mo_float_to_half(x[i]);
}

void mo_half_to_float_array(const uint16_t* h, uint64_t n, float* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = mo_half_to_float(h[i]);
}

/* ------------------------------------------------------------------------------------------
 * Threaded variants for full-size parity tests (36864x12288 ... 131072x32768): rows are
 * independent (convert.hpp:12-16: every row restarts at the virtual column -1), so a row
 * partition over pthreads gives byte-identical output.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
    uint64_t r0, r1, cols, row0;
    uint32_t thr24;
    uint64_t seed;
    int int_mode, status;
    unsigned bits, unit_steps;
    const uint16_t* dense;
    uint16_t* out;
    uint32_t* counts;
    const uint32_t* rp;
    uint16_t* values;
    uint8_t* deltas;
    const uint16_t* x;
} mt_job;

static void run_jobs(mt_job* jobs, int n, void* (*fn)(void*)) {
    pthread_t* th = (pthread_t*)calloc((size_t)n, sizeof(pthread_t));
    for (int t = 0; t < n; ++t) pthread_create(&th[t], NULL, fn, &jobs[t]);
    for (int t = 0; t < n; ++t) pthread_join(th[t], NULL);
    free(th);
}

static int clamp_threads(int nthreads, uint64_t rows) {
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > rows) nthreads = rows ? (int)rows : 1;
    return nthreads;
}

static void* gen_rows_job(void* arg) {
    mt_job* j = (mt_job*)arg;
    for (uint64_t r = j->r0; r < j->r1; ++r)
        for (uint64_t c = 0; c < j->cols; ++c)
            j->out[r * j->cols + c] = mo_gen_value(j->seed, (j->row0 + r) * j->cols + c, j->thr24, j->int_mode);
    return NULL;
}

void mo_gen_dense_rows_mt(uint64_t row0, uint64_t rows, uint64_t cols, uint32_t thr24, uint64_t seed, int int_mode,
                          uint16_t* out, int nthreads) {
    nthreads = clamp_threads(nthreads, rows);
    mt_job* jobs = (mt_job*)calloc((size_t)nthreads, sizeof(mt_job));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].r0 = rows * t / nthreads;
        jobs[t].r1 = rows * (t + 1) / nthreads;
        jobs[t].cols = cols;
        jobs[t].row0 = row0;
        jobs[t].thr24 = thr24;
        jobs[t].seed = seed;
        jobs[t].int_mode = int_mode;
        jobs[t].out = out;
    }
    run_jobs(jobs, nthreads, gen_rows_job);
    free(jobs);
}

static void* count_rows_job(void* arg) {
    mt_job* j = (mt_job*)arg;
    row_encoder en = {NULL, NULL, 0, j->bits, -1, 1u << j->bits};
    for (uint64_t r = j->r0; r < j->r1; ++r) {
        const uint16_t* row = j->dense + r * j->cols;
        en.prev = -1;
        en.at = 0;
        for (uint64_t c = 0; c < j->cols; ++c)
            if (!mo_half_is_zero(row[c])) enc_push(&en, (int64_t)c, row[c]);
        j->counts[r] = (uint32_t)en.at;
    }
    return NULL;
}

static void* fill_rows_job(void* arg) {
    mt_job* j = (mt_job*)arg;
    row_encoder en = {j->values, j->deltas, 0, j->bits, -1, 1u << j->bits};
    for (uint64_t r = j->r0; r < j->r1; ++r) {
        const uint16_t* row = j->dense + r * j->cols;
        en.prev = -1;
        en.at = j->rp[r];
        for (uint64_t c = 0; c < j->cols; ++c)
            if (!mo_half_is_zero(row[c])) enc_push(&en, (int64_t)c, row[c]);
    }
    return NULL;
}

/* encode_dense over a row partition: count pass (per-row entries), scan, fill pass. */
int mo_encode_dense_count_mt(const uint16_t* dense, uint64_t rows, uint64_t cols, unsigned bits, uint32_t* rp,
                             uint64_t* pad_nnz, int nthreads) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    nthreads = clamp_threads(nthreads, rows);
    mt_job* jobs = (mt_job*)calloc((size_t)nthreads, sizeof(mt_job));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].r0 = rows * t / nthreads;
        jobs[t].r1 = rows * (t + 1) / nthreads;
        jobs[t].cols = cols;
        jobs[t].bits = bits;
        jobs[t].dense = dense;
        jobs[t].counts = rp + 1;
    }
    run_jobs(jobs, nthreads, count_rows_job);
    free(jobs);
    uint64_t acc = 0;
    rp[0] = 0;
    for (uint64_t r = 0; r < rows; ++r) {
        acc += rp[r + 1];
        if (acc > 0xFFFFFFFFull) return fail(MO_EINVAL, "pad_nnz does not fit u32 row pointers");
        rp[r + 1] = (uint32_t)acc;
    }
    *pad_nnz = acc;
    return MO_OK;
}

int mo_encode_dense_fill_mt(const uint16_t* dense, uint64_t rows, uint64_t cols, unsigned bits, const uint32_t* rp,
                            uint16_t* values, uint8_t* deltas, int nthreads) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    const uint64_t pad_nnz = rows ? rp[rows] : 0;
    memset(values, 0, (size_t)mo_values_bytes(pad_nnz));
    memset(deltas, 0, (size_t)mo_delta_bytes(pad_nnz, bits));
    nthreads = clamp_threads(nthreads, rows);
    mt_job* jobs = (mt_job*)calloc((size_t)nthreads, sizeof(mt_job));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].r0 = rows * t / nthreads;
        jobs[t].r1 = rows * (t + 1) / nthreads;
        jobs[t].cols = cols;
        jobs[t].bits = bits;
        jobs[t].dense = dense;
        jobs[t].rp = rp;
        jobs[t].values = values;
        jobs[t].deltas = deltas;
    }
    run_jobs(jobs, nthreads, fill_rows_job);
    free(jobs);
    return MO_OK;
}

static void* order_rows_job(void* arg) {
    mt_job* j = (mt_job*)arg;
    /* the row range's own slice of row pointers (absolute offsets stay valid) */
    j->status = mo_b200_order_spmv(j->r1 - j->r0, j->cols, j->bits, j->values, j->deltas, j->rp + j->r0, j->x,
                                   j->out + j->r0, j->unit_steps);
    return NULL;
}

int mo_b200_order_spmv_mt(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values, const uint8_t* deltas,
                          const uint32_t* rp, const uint16_t* x, uint16_t* y, unsigned unit_steps, int nthreads) {
    if (!mo_is_valid_delta_bits(bits)) return fail(MO_EINVAL, "delta width must be one of 1, 2, 4, 8 bits");
    nthreads = clamp_threads(nthreads, rows);
    mt_job* jobs = (mt_job*)calloc((size_t)nthreads, sizeof(mt_job));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].r0 = rows * t / nthreads;
        jobs[t].r1 = rows * (t + 1) / nthreads;
        jobs[t].cols = cols;
        jobs[t].bits = bits;
        jobs[t].unit_steps = unit_steps;
        jobs[t].values = (uint16_t*)values;
        jobs[t].deltas = (uint8_t*)deltas;
        jobs[t].rp = rp;
        jobs[t].x = x;
        jobs[t].out = y;
    }
    run_jobs(jobs, nthreads, order_rows_job);
    int st = MO_OK;
    for (int t = 0; t < nthreads; ++t)
        if (jobs[t].status != MO_OK) st = jobs[t].status;
    free(jobs);
    return st == MO_OK ? MO_OK : fail(st, "decoded column index past the column bound");
}
