// macko_dropin.cpp — libmacko.so: the reference's C++ API (namespace macko, proj/src/*.hpp) backed
// by the B200 library.  A caller of the reference links this library instead of the reference's
// `macko` target (proj/src/CMakeLists.txt:1-19) and keeps its code and headers unchanged:
//
//   fp16.hpp    half_to_float / float_to_half / half_table        (host, bit-exact RNE; fp16.cpp:8-82)
//   bitpack.hpp is_valid_delta_bits / pack_deltas / unpack_deltas / pack_delta_at (host; bitpack.cpp)
//   convert.hpp csr_from_dense, macko_from_csr, dense_from_macko, padding_count, validate_macko
//               -> GPU kernels through the C-ABI (macko_csr_from_dense, macko_dev_from_csr,
//                  macko_dev_to_dense, macko_dev_padding_count, macko_dev_upload's device validation);
//               validate_csr on the host (convert.hpp:25)
//   spmv.hpp    dense_mv (host) and reference_spmv (GPU; include/macko/spmv.hpp)
//
// Errors keep the reference's taxonomy (errors.hpp:9-21, bitpack.cpp:14-15): the C-ABI status codes
// become std::invalid_argument / macko::FormatError / macko::IoError / macko::InfeasibleError.
// Built against the reference headers (-I proj/src); no reference source is compiled in.
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "bitpack.hpp"
#include "convert.hpp"
#include "errors.hpp"
#include "fp16.hpp"
#include "macko/spmv.hpp"
#include "macko_cuda.h"

namespace macko {

namespace {

void check(macko_status s) {
    if (s == MACKO_OK) return;
    const std::string msg = macko_last_error();
    switch (s) {
        case MACKO_EINVAL: throw std::invalid_argument(msg);
        case MACKO_EFORMAT: throw FormatError(msg);
        case MACKO_EIO: throw IoError(msg);
        case MACKO_EINFEASIBLE: throw InfeasibleError(msg);
        case MACKO_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error("libmacko_cuda: " + msg);
    }
}

// Device handle of a host MackoMatrix for one call (uploaded and validated on the device).
struct Uploaded {
    macko_dev_matrix* h = nullptr;
    explicit Uploaded(const MackoMatrix& m) {
        if (!is_valid_delta_bits(m.params.b_delta))
            throw std::invalid_argument("delta width must be one of 1, 2, 4, 8 bits; got " +
                                        std::to_string(m.params.b_delta));
        if (m.row_pointers.size() != m.rows + 1) throw FormatError("row_pointers must hold rows + 1 entries");
        static_assert(sizeof(Half) == 2, "Half is a raw 16-bit pattern");
        check(macko_dev_upload(0, m.rows, m.cols, m.params.b_delta, reinterpret_cast<const uint16_t*>(m.values.data()),
                               m.values.size(), m.packed_deltas.data(), m.packed_deltas.size(), m.row_pointers.data(),
                               nullptr, &h));
    }
    ~Uploaded() {
        if (h) macko_dev_free(h);
    }
    Uploaded(const Uploaded&) = delete;
    Uploaded& operator=(const Uploaded&) = delete;
};

uint32_t f32_bits(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    return u;
}

float bits_f32(uint32_t u) {
    float x;
    std::memcpy(&x, &u, 4);
    return x;
}

}  // namespace

// ---- fp16.hpp -------------------------------------------------------------------------------
// Exact widening: normals rebias the exponent, subnormals normalise, NaN payloads are carried
// (no quiet bit added, as fp16.cpp:8-35 does).
float half_to_float(Half h) {
    const uint32_t sign = (uint32_t)(h.bits & 0x8000u) << 16;
    const uint32_t exp = (h.bits >> 10) & 0x1Fu, man = h.bits & 0x3FFu;
    if (exp == 0x1Fu) return bits_f32(sign | 0x7F800000u | (man << 13));
    if (exp != 0) return bits_f32(sign | ((exp + 112u) << 23) | (man << 13));
    if (man == 0) return bits_f32(sign);
    int e = -1;
    uint32_t m = man;
    do {
        m <<= 1;
        ++e;
    } while (!(m & 0x400u));
    return bits_f32(sign | ((uint32_t)(112 - e) << 23) | ((m & 0x3FFu) << 13));
}

// Round to nearest, ties to even, on the integer representation: |x| >= 65520 -> inf, NaN ->
// quiet NaN with the top payload bits (fp16.cpp:37-73; equal to IEEE RNE on every input).
Half float_to_half(float x) {
    const uint32_t f = f32_bits(x);
    const uint16_t sign = (uint16_t)((f >> 16) & 0x8000u);
    const uint32_t a = f & 0x7FFFFFFFu;
    if (a > 0x7F800000u) return Half{(uint16_t)(sign | 0x7E00u | ((a >> 13) & 0x3FFu))};
    if (a >= 0x477FF000u) return Half{(uint16_t)(sign | 0x7C00u)};
    if (a >= 0x38800000u) {  // normal half: drop 13 mantissa bits with RNE (a carry rolls into the exponent)
        uint32_t hb = (a >> 13) - (112u << 10);
        const uint32_t rem = a & 0x1FFFu;
        if (rem > 0x1000u || (rem == 0x1000u && (hb & 1u))) ++hb;
        return Half{(uint16_t)(sign | hb)};
    }
    if (a <= 0x33000000u) return Half{sign};  // <= 2^-25: rounds to zero (the tie goes to even 0)
    const uint32_t e = a >> 23, m = (a & 0x7FFFFFu) | 0x800000u;
    const uint32_t shift = 126u - e;  // subnormal half: k = m * 2^(e - 126), unit 2^-24
    uint32_t k = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1u), half = 1u << (shift - 1u);
    if (rem > half || (rem == half && (k & 1u))) ++k;
    return Half{(uint16_t)(sign | k)};
}

const float* half_table() {
    static const std::vector<float> table = [] {
        std::vector<float> t(65536);
        for (uint32_t i = 0; i < 65536; ++i) t[i] = half_to_float(Half{(uint16_t)i});
        return t;
    }();
    return table.data();
}

// ---- bitpack.hpp ------------------------------------------------------------------------------
bool is_valid_delta_bits(unsigned bits) { return bits == 1 || bits == 2 || bits == 4 || bits == 8; }

namespace {
void require_bits(unsigned bits) {
    if (!is_valid_delta_bits(bits))
        throw std::invalid_argument("delta width must be one of 1, 2, 4, 8 bits; got " + std::to_string(bits));
}
void require_delta(uint32_t d, unsigned bits) {
    const uint32_t maxd = 1u << bits;
    if (d < 1 || d > maxd)
        throw std::invalid_argument("delta " + std::to_string(d) + " out of range [1, " + std::to_string(maxd) + "]");
}
}  // namespace

void pack_delta_at(uint8_t* bytes, size_t index, unsigned bits, uint32_t delta) {
    require_bits(bits);
    require_delta(delta, bits);
    const unsigned per = 8u / bits, shift = (unsigned)(index % per) * bits;
    const uint32_t mask = bits == 8 ? 0xFFu : ((1u << bits) - 1u);
    uint8_t& b = bytes[index / per];
    b = (uint8_t)((b & ~(mask << shift)) | ((delta - 1u) << shift));
}

std::vector<uint8_t> pack_deltas(const std::vector<uint32_t>& deltas, unsigned bits) {
    require_bits(bits);
    const unsigned per = 8u / bits;
    std::vector<uint8_t> out((deltas.size() + per - 1) / per, 0);
    for (size_t i = 0; i < deltas.size(); ++i) {
        require_delta(deltas[i], bits);
        out[i / per] |= (uint8_t)((deltas[i] - 1u) << ((unsigned)(i % per) * bits));
    }
    return out;
}

std::vector<uint32_t> unpack_deltas(const uint8_t* bytes, size_t count, unsigned bits) {
    require_bits(bits);
    std::vector<uint32_t> out(count);
    for (size_t i = 0; i < count; ++i) out[i] = unpack_delta_at(bytes, i, bits);
    return out;
}

// ---- convert.hpp ------------------------------------------------------------------------------
CsrMatrix csr_from_dense(const DenseMatrix& m, unsigned index_width) {
    if (m.data.size() != m.rows * m.cols) throw std::invalid_argument("dense data size != rows * cols");
    CsrMatrix c;
    c.rows = m.rows;
    c.cols = m.cols;
    c.index_width = index_width;
    c.row_pointers.assign(m.rows + 1, 0);
    if (m.rows == 0 || m.cols == 0) return c;
    const uint16_t* d = reinterpret_cast<const uint16_t*>(m.data.data());
    uint64_t nnz = 0;
    check(macko_csr_from_dense(0, d, m.rows, m.cols, m.cols, 0, c.row_pointers.data(), nullptr, nullptr, &nnz, nullptr));
    c.values.resize(nnz);
    c.column_indices.resize(nnz);
    if (nnz)
        check(macko_csr_from_dense(0, d, m.rows, m.cols, m.cols, 0, c.row_pointers.data(),
                                   reinterpret_cast<uint16_t*>(c.values.data()), c.column_indices.data(), &nnz, nullptr));
    return c;
}

void validate_csr(const CsrMatrix& m) {
    if (m.row_pointers.size() != m.rows + 1) throw std::invalid_argument("row_pointers must hold rows + 1 entries");
    if (m.row_pointers[0] != 0) throw std::invalid_argument("row_pointers[0] must be 0");
    if (m.values.size() != m.column_indices.size()) throw std::invalid_argument("values / column_indices size mismatch");
    if (m.row_pointers[m.rows] != m.values.size()) throw std::invalid_argument("row_pointers[rows] != nnz");
    for (size_t r = 0; r < m.rows; ++r) {
        if (m.row_pointers[r + 1] < m.row_pointers[r]) throw std::invalid_argument("row_pointers not monotone");
        long long prev = -1;
        for (size_t k = m.row_pointers[r]; k < m.row_pointers[r + 1]; ++k) {
            const long long c = m.column_indices[k];
            if (c >= (long long)m.cols) throw std::invalid_argument("column index out of range");
            if (c <= prev) throw std::invalid_argument("columns not strictly increasing within a row");
            if (half_is_zero(m.values[k])) throw std::invalid_argument("stored zero in a canonical CSR");
            prev = c;
        }
    }
}

MackoMatrix macko_from_csr(const CsrMatrix& m, MackoParams params) {
    require_bits(params.b_delta);
    if (params.b_val != 16) throw std::invalid_argument("b_val must be 16 (fp16 values)");
    if (m.row_pointers.size() != m.rows + 1) throw std::invalid_argument("row_pointers must hold rows + 1 entries");
    MackoMatrix out;
    out.rows = m.rows;
    out.cols = m.cols;
    out.params = params;
    if (m.rows == 0 || m.cols == 0) {
        out.row_pointers.assign(m.rows + 1, 0);
        return out;
    }
    macko_dev_matrix* h = nullptr;
    check(macko_dev_from_csr(0, m.rows, m.cols, params.b_delta, reinterpret_cast<const uint16_t*>(m.values.data()),
                             m.column_indices.data(), m.row_pointers.data(), m.values.size(), 0, nullptr, &h));
    macko_dev_info info{};
    macko_status st = macko_dev_get_info(h, &info);
    if (st == MACKO_OK) {
        out.values.resize(info.values_bytes / 2);
        out.packed_deltas.resize(info.delta_bytes);
        out.row_pointers.resize(m.rows + 1);
        st = macko_dev_download(h, reinterpret_cast<uint16_t*>(out.values.data()), out.packed_deltas.data(),
                                out.row_pointers.data(), nullptr);
    }
    macko_dev_free(h);
    check(st);
    return out;
}

DenseMatrix dense_from_macko(const MackoMatrix& m) {
    DenseMatrix d = DenseMatrix::zeros(m.rows, m.cols);
    if (m.rows == 0 || m.cols == 0) return d;
    Uploaded u(m);
    check(macko_dev_to_dense(u.h, reinterpret_cast<uint16_t*>(d.data.data()), m.cols, 0, nullptr));
    return d;
}

size_t padding_count(const MackoMatrix& m) {
    if (m.rows == 0 || m.cols == 0) return 0;
    Uploaded u(m);
    uint64_t n = 0;
    check(macko_dev_padding_count(u.h, &n, nullptr));
    return n;
}

void validate_macko(const MackoMatrix& m) {
    if (m.rows == 0 || m.cols == 0) return;
    Uploaded u(m);  // macko_dev_upload validates on the device: FormatError on any broken invariant
}

// ---- spmv.hpp ---------------------------------------------------------------------------------
Vector dense_mv(const DenseMatrix& m, const Vector& v) {
    if (v.size() != m.cols) throw std::invalid_argument("dimension mismatch: v must have cols entries");
    Vector y(m.rows);
    for (size_t r = 0; r < m.rows; ++r) {
        float acc = 0.0f;
        for (size_t c = 0; c < m.cols; ++c) acc += half_to_float(m.at(r, c)) * half_to_float(v[c]);
        y[r] = float_to_half(acc);
    }
    return y;
}

Vector reference_spmv(const MackoMatrix& m, const Vector& v) {
    if (v.size() != m.cols) throw std::invalid_argument("dimension mismatch: v must have cols entries");
    Vector y(m.rows);
    if (m.rows == 0) return y;
    if (m.cols == 0) return Vector(m.rows, half_zero());
    Uploaded u(m);
    check(macko_spmv_host(u.h, reinterpret_cast<const uint16_t*>(v.data()), reinterpret_cast<uint16_t*>(y.data()),
                          nullptr));
    return y;
}

}  // namespace macko
