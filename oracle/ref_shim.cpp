// ref_shim.cpp — TEST INFRASTRUCTURE: builds oracle/_ref/libmacko_ref.so from the reference's
// own sources where they lie (/root/reference/proj/src: fp16.cpp, bitpack.cpp and the headers
// fp16.hpp, bitpack.hpp, matrix.hpp, convert.hpp, errors.hpp — compiled, never copied).
//
// The reference tree ships declarations without bodies for csr_from_dense, macko_from_csr,
// dense_from_macko, padding_count, validate_* (convert.hpp:8-27) and no spmv.cpp at all
// (SURVEY.md §0.2).  This shim restates those bodies from SPEC.md on top of the reference's
// own types, bit packing (pack_deltas, bitpack.cpp:18-32), row decoder (for_each_row_element,
// convert.hpp:29-42) and fp16 LUT (half_table, fp16.cpp:75-82), and exports a C surface for
// ctypes.  It is the "reference" CPU arm of bench.py and the cross-check for oracle/*.c.
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "bitpack.hpp"
#include "convert.hpp"
#include "errors.hpp"
#include "fp16.hpp"
#include "matrix.hpp"

namespace macko {

// SPEC.md:54-62
CsrMatrix csr_from_dense(const DenseMatrix& m, unsigned index_width) {
    CsrMatrix out;
    out.rows = m.rows;
    out.cols = m.cols;
    out.index_width = index_width;
    out.row_pointers.reserve(m.rows + 1);
    out.row_pointers.push_back(0);
    for (size_t r = 0; r < m.rows; ++r) {
        for (size_t c = 0; c < m.cols; ++c) {
            const Half h = m.at(r, c);
            if (half_is_zero(h)) continue;
            out.values.push_back(h);
            out.column_indices.push_back(static_cast<uint32_t>(c));
        }
        out.row_pointers.push_back(static_cast<uint32_t>(out.values.size()));
    }
    return out;
}

// greedy padding, virtual column -1, no trailing pads, 16-B tails.
MackoMatrix macko_from_csr(const CsrMatrix& m, MackoParams params) {
    if (!is_valid_delta_bits(params.b_delta))
        throw std::invalid_argument("delta width must be one of 1, 2, 4, 8 bits; got " +
                                    std::to_string(params.b_delta));
    const long long maxd = params.max_delta();
    MackoMatrix out;
    out.rows = m.rows;
    out.cols = m.cols;
    out.params = params;
    std::vector<uint32_t> deltas;
    out.row_pointers.push_back(0);
    for (size_t r = 0; r < m.rows; ++r) {
        long long prev = -1;
        for (uint32_t k = m.row_pointers[r]; k < m.row_pointers[r + 1]; ++k) {
            const long long c = m.column_indices[k];
            if (c >= static_cast<long long>(m.cols) || c <= prev)
                throw std::invalid_argument("CSR column out of range or not increasing");
            while (c - prev > maxd) {
                out.values.push_back(half_zero());
                deltas.push_back(static_cast<uint32_t>(maxd));
                prev += maxd;
            }
            out.values.push_back(m.values[k]);
            deltas.push_back(static_cast<uint32_t>(c - prev));
            prev = c;
        }
        if (out.values.size() > 0xFFFFFFFFull) throw std::invalid_argument("pad_nnz exceeds u32");
        out.row_pointers.push_back(static_cast<uint32_t>(out.values.size()));
    }
    const size_t pad_nnz = out.values.size();
    out.packed_deltas = pack_deltas(deltas, params.b_delta);
    out.values.resize(macko_values_bytes(pad_nnz) / 2, half_zero());
    out.packed_deltas.resize(macko_delta_bytes(pad_nnz, params.b_delta), 0);
    return out;
}

// SPEC.md:74-82
DenseMatrix dense_from_macko(const MackoMatrix& m) {
    DenseMatrix d = DenseMatrix::zeros(m.rows, m.cols);
    for (size_t r = 0; r < m.rows; ++r)
        for_each_row_element(m, r, [&](size_t, size_t col, Half v) {
            if (col >= m.cols) throw FormatError("decoded column index past the column bound");
            d.at(r, col) = v;
        });
    return d;
}

// SPEC.md:95-102
size_t padding_count(const MackoMatrix& m) {
    size_t n = 0;
    for (size_t e = 0; e < m.pad_nnz(); ++e) n += half_is_zero(m.values[e]);
    return n;
}

void validate_csr(const CsrMatrix& m) {
    if (m.row_pointers.size() != m.rows + 1 || m.row_pointers[0] != 0)
        throw FormatError("bad CSR row pointers");
    for (size_t r = 0; r < m.rows; ++r) {
        long long prev = -1;
        for (uint32_t k = m.row_pointers[r]; k < m.row_pointers[r + 1]; ++k) {
            const long long c = m.column_indices[k];
            if (c <= prev || c >= static_cast<long long>(m.cols)) throw FormatError("bad CSR column");
            if (half_is_zero(m.values[k])) throw FormatError("stored zero in CSR");
            prev = c;
        }
    }
}

void validate_macko(const MackoMatrix& m) {
    if (!is_valid_delta_bits(m.params.b_delta)) throw std::invalid_argument("bad delta width");
    if (m.row_pointers.size() != m.rows + 1 || m.row_pointers[0] != 0)
        throw FormatError("bad row pointers");
    for (size_t r = 0; r < m.rows; ++r) {
        if (m.row_pointers[r + 1] < m.row_pointers[r]) throw FormatError("row pointers not monotone");
        for_each_row_element(m, r, [&](size_t, size_t col, Half) {
            if (col >= m.cols) throw FormatError("decoded column index past the column bound");
        });
    }
}

}  // namespace macko

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const macko::FormatError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// reference_spmv — SPEC.md:235-243, on the reference's decoder and fp16 LUT.
void spmv_rows(const macko::MackoMatrix& m, const macko::Half* x, macko::Half* y, size_t r0, size_t r1) {
    const float* lut = macko::half_table();
    for (size_t r = r0; r < r1; ++r) {
        float acc = 0.0f;
        macko::for_each_row_element(m, r, [&](size_t, size_t col, macko::Half v) {
            acc += lut[v.bits] * lut[x[col].bits];
        });
        y[r] = macko::float_to_half(acc);
    }
}

}  // namespace

struct ref_matrix {
    macko::MackoMatrix m;
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint16_t ref_float_to_half(float x) { return macko::float_to_half(x).bits; }
float ref_half_to_float(uint16_t h) { return macko::half_to_float(macko::Half{h}); }

void ref_half_to_float_array(const uint16_t* h, uint64_t n, float* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = macko::half_to_float(macko::Half{h[i]});
}

void ref_float_to_half_array(const float* x, uint64_t n, uint16_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = macko::float_to_half(x[i]).bits;
}

int ref_pack_deltas(const uint32_t* deltas, uint64_t n, unsigned bits, uint8_t* out, uint64_t out_len) {
    return guarded([&] {
        std::vector<uint32_t> d(deltas, deltas + n);
        std::vector<uint8_t> b = macko::pack_deltas(d, bits);
        if (b.size() > out_len) throw std::invalid_argument("output too small");
        std::memcpy(out, b.data(), b.size());
    });
}

int ref_unpack_deltas(const uint8_t* bytes, uint64_t n, unsigned bits, uint32_t* out) {
    return guarded([&] {
        std::vector<uint32_t> d = macko::unpack_deltas(bytes, n, bits);
        std::memcpy(out, d.data(), n * 4);
    });
}

int ref_encode_dense(const uint16_t* dense, uint64_t rows, uint64_t cols, unsigned bits, ref_matrix** out) {
    return guarded([&] {
        macko::DenseMatrix d = macko::DenseMatrix::zeros(rows, cols);
        std::memcpy(d.data.data(), dense, rows * cols * 2);
        auto* h = new ref_matrix;
        h->m = macko::macko_from_csr(macko::csr_from_dense(d), macko::MackoParams{16, bits});
        *out = h;
    });
}

int ref_from_arrays(uint64_t rows, uint64_t cols, unsigned bits, const uint16_t* values, uint64_t n_values,
                    const uint8_t* deltas, uint64_t n_delta_bytes, const uint32_t* rp, ref_matrix** out) {
    return guarded([&] {
        auto* h = new ref_matrix;
        h->m.rows = rows;
        h->m.cols = cols;
        h->m.params = macko::MackoParams{16, bits};
        h->m.values.resize(n_values);
        std::memcpy(h->m.values.data(), values, n_values * 2);
        h->m.packed_deltas.assign(deltas, deltas + n_delta_bytes);
        h->m.row_pointers.assign(rp, rp + rows + 1);
        *out = h;
    });
}

void ref_matrix_info(const ref_matrix* h, uint64_t* pad_nnz, uint64_t* n_values, uint64_t* n_delta_bytes) {
    *pad_nnz = h->m.pad_nnz();
    *n_values = h->m.values.size();
    *n_delta_bytes = h->m.packed_deltas.size();
}

void ref_matrix_copy(const ref_matrix* h, uint16_t* values, uint8_t* deltas, uint32_t* rp) {
    std::memcpy(values, h->m.values.data(), h->m.values.size() * 2);
    std::memcpy(deltas, h->m.packed_deltas.data(), h->m.packed_deltas.size());
    std::memcpy(rp, h->m.row_pointers.data(), h->m.row_pointers.size() * 4);
}

void ref_matrix_free(ref_matrix* h) { delete h; }

int ref_dense_from_macko(const ref_matrix* h, uint16_t* dense) {
    return guarded([&] {
        macko::DenseMatrix d = macko::dense_from_macko(h->m);
        std::memcpy(dense, d.data.data(), d.data.size() * 2);
    });
}

int ref_validate(const ref_matrix* h) { return guarded([&] { macko::validate_macko(h->m); }); }

uint64_t ref_padding_count(const ref_matrix* h) { return macko::padding_count(h->m); }

// reference_spmv over all host threads requested (row partition).
int ref_spmv(const ref_matrix* h, const uint16_t* x, uint16_t* y, int nthreads) {
    return guarded([&] {
        const auto* xh = reinterpret_cast<const macko::Half*>(x);
        auto* yh = reinterpret_cast<macko::Half*>(y);
        const size_t R = h->m.rows;
        if (nthreads <= 1 || R < 2) {
            spmv_rows(h->m, xh, yh, 0, R);
            return;
        }
        (void)macko::half_table();  // build the LUT before fanning out
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t)
            th.emplace_back(spmv_rows, std::cref(h->m), xh, yh, R * t / nthreads, R * (t + 1) / nthreads);
        for (auto& t : th) t.join();
    });
}

// dense_mv — SPEC.md:225-233 on the reference's fp16 LUT.
void ref_dense_mv(const uint16_t* dense, uint64_t rows, uint64_t cols, const uint16_t* x, uint16_t* y) {
    const float* lut = macko::half_table();
    for (uint64_t r = 0; r < rows; ++r) {
        float acc = 0.0f;
        for (uint64_t c = 0; c < cols; ++c) acc += lut[dense[r * cols + c]] * lut[x[c]];
        y[r] = macko::float_to_half(acc).bits;
    }
}

}  // extern "C"
