/*
 * macko_oracle.h — CPU ORACLE for the MACKO-SpMV hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This is a plain-C restatement of the reference's algorithm (arxiv 2511.13061,
 * /root/reference).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker or the CPU baseline.  The
 * product path (paper_2511_13061_b200/, libmacko_cuda.so) never links or calls it.
 *
 * Pinning: fp16 and bit packing are checked against the reference's own fp16.cpp /
 * bitpack.cpp compiled into oracle/_ref (see oracle/Makefile, tests/test_oracle.py), and
 * the encoder / SpMV against SPEC.md's golden vectors (tests/golden/) and the ref shim.
 * The encoder/decoder/SpMV bodies are absent from the reference tree;
 * they are restated from SPEC.md and cited function by function in macko_oracle.c.
 */
#ifndef MACKO_ORACLE_H
#define MACKO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { MO_OK = 0, MO_EINVAL = 1, MO_EFORMAT = 2, MO_EINFEASIBLE = 4 };

/* Last error message of the calling thread ("" if none). */
const char* mo_last_error(void);

/* ---- fp16 (reference fp16.hpp / fp16.cpp) ---- */
uint16_t mo_float_to_half(float x);
float mo_half_to_float(uint16_t h);
int mo_half_is_zero(uint16_t h);
void mo_float_to_half_array(const float* x, uint64_t n, uint16_t* out);
void mo_half_to_float_array(const uint16_t* h, uint64_t n, float* out);

/* ---- delta bit packing (reference bitpack.hpp / bitpack.cpp) ---- */
int mo_is_valid_delta_bits(unsigned bits);
/* out must hold ceil(n / (8/bits)) bytes; it is fully written (zeros included). */
int mo_pack_deltas(const uint32_t* deltas, uint64_t n, unsigned bits, uint8_t* out);
int mo_unpack_deltas(const uint8_t* bytes, uint64_t n, unsigned bits, uint32_t* out);

/* ---- storage sizes (reference matrix.hpp:73-81) ---- */
uint64_t mo_align_up(uint64_t n, uint64_t alignment);
uint64_t mo_values_bytes(uint64_t pad_nnz);
uint64_t mo_delta_bytes(uint64_t pad_nnz, unsigned bits);

/* ---- csr_from_dense: two phases, count then fill ---- */
uint64_t mo_csr_count(const uint16_t* dense, uint64_t rows, uint64_t cols, uint32_t* row_ptrs);
void mo_csr_fill(const uint16_t* dense, uint64_t rows, uint64_t cols, const uint32_t* row_ptrs,
                 uint16_t* values, uint32_t* col_idx);

/* ---- macko_from_csr: count (row pointers) then fill ----
 * values must hold mo_values_bytes(pad_nnz) bytes, deltas mo_delta_bytes(pad_nnz, bits);
 * both are fully written including the zero tail. */
int mo_macko_count(uint64_t rows, uint64_t cols, const uint32_t* csr_row_ptrs,
                   const uint32_t* csr_cols, unsigned bits, uint32_t* macko_row_ptrs,
                   uint64_t* pad_nnz);
int mo_macko_fill(uint64_t rows, uint64_t cols, const uint32_t* csr_row_ptrs,
                  const uint32_t* csr_cols, const uint16_t* csr_values, unsigned bits,
                  const uint32_t* macko_row_ptrs, uint16_t* values, uint8_t* deltas);

/* Dense -> MACKO in one call (csr_from_dense + macko_from_csr semantics, no CSR buffers).
 * Phase 1 fills row_ptrs (rows+1) and pad_nnz; phase 2 fills values/deltas. */
int mo_encode_dense_count(const uint16_t* dense, uint64_t rows, uint64_t cols, unsigned bits,
                          uint32_t* row_ptrs, uint64_t* pad_nnz);
int mo_encode_dense_fill(const uint16_t* dense, uint64_t rows, uint64_t cols, unsigned bits,
                         const uint32_t* row_ptrs, uint16_t* values, uint8_t* deltas);

/* ---- dense_from_macko / validate / padding_count ---- */
int mo_dense_from_macko(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values,
                        const uint8_t* deltas, const uint32_t* row_ptrs, uint16_t* dense);
int mo_validate_macko(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values,
                      uint64_t n_values, const uint8_t* deltas, uint64_t n_delta_bytes,
                      const uint32_t* row_ptrs);
uint64_t mo_padding_count(uint64_t rows, const uint16_t* values, const uint32_t* row_ptrs);

/* ---- executors ---- */
void mo_dense_mv(const uint16_t* dense, uint64_t rows, uint64_t cols, const uint16_t* x,
                 uint16_t* y);
/* Sequential fp32, pads included, one RNE per row; nthreads<=1 runs single-threaded. */
int mo_reference_spmv(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values,
                      const uint8_t* deltas, const uint32_t* row_ptrs, const uint16_t* x,
                      uint16_t* y, int nthreads);
/* Algorithm 1: exclusive prefix over 32 lanes by shfl_up doubling. */
void mo_warp_prefix_sum(const uint32_t* local, uint32_t* out);
/* SPEC.md:255-264 warp_spmv: 32 lanes x 8 elements per step, ROMA, reduce after the row. */
int mo_warp_spmv(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values,
                 const uint8_t* deltas, const uint32_t* row_ptrs, const uint16_t* x,
                 uint16_t* y);
/* The B200 kernel's canonical summation order: warp_spmv, but the 32 lane
 * accumulators are xor-tree reduced every `unit_steps` steps and the unit sums are added
 * sequentially into the row accumulator.  Lets tests check the GPU bit-exactly in float mode. */
int mo_b200_order_spmv(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values,
                       const uint8_t* deltas, const uint32_t* row_ptrs, const uint16_t* x,
                       uint16_t* y, unsigned unit_steps);

/* Threaded variants (row partitions; byte-identical to the single-threaded functions), for the
 * full-size parity tests. */
void mo_gen_dense_rows_mt(uint64_t row0, uint64_t rows, uint64_t cols, uint32_t thr24, uint64_t seed, int int_mode,
                          uint16_t* out, int nthreads);
int mo_encode_dense_count_mt(const uint16_t* dense, uint64_t rows, uint64_t cols, unsigned bits, uint32_t* rp,
                             uint64_t* pad_nnz, int nthreads);
int mo_encode_dense_fill_mt(const uint16_t* dense, uint64_t rows, uint64_t cols, unsigned bits, const uint32_t* rp,
                            uint16_t* values, uint8_t* deltas, int nthreads);
int mo_b200_order_spmv_mt(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values, const uint8_t* deltas,
                          const uint32_t* rp, const uint16_t* x, uint16_t* y, unsigned unit_steps, int nthreads);

/* ---- synthetic inputs (our counter-hash generator) ---- */
uint32_t mo_density_threshold(double density);
uint16_t mo_gen_value(uint64_t seed, uint64_t idx, uint32_t thr24, int int_mode);
void mo_gen_dense(uint64_t rows, uint64_t cols, uint32_t thr24, uint64_t seed, int int_mode,
                  uint16_t* out);
void mo_gen_vector(uint64_t n, uint64_t seed, int int_mode, uint16_t* out);
void mo_gen_worst_case(uint64_t rows, uint64_t cols, uint64_t zero_run, uint16_t* out);

/* ---- spmv_traffic: algorithmic bytes per SpMV ---- */
uint64_t mo_spmv_traffic_bytes(uint64_t rows, uint64_t cols, uint64_t pad_nnz, unsigned bits);
uint64_t mo_dense_traffic_bytes(uint64_t rows, uint64_t cols);

#ifdef __cplusplus
}
#endif
#endif
