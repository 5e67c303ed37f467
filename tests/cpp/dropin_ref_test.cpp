// dropin_ref_test.cpp — a reference C++ caller switched to libmacko.so (GPU).  Compiled against the
// reference's own headers (proj/src: matrix.hpp, convert.hpp, fp16.hpp, bitpack.hpp, errors.hpp)
// plus include/macko/spmv.hpp, linked against libmacko.so ONLY (no reference source, no
// oracle/_ref).  Checks the reference's worked examples and properties:
//   * fp16: float_to_half / half_to_float equal x86 F16C RNE (every half, 2^24 sampled floats),
//     half_table;
//   * bitpack KATs and its std::invalid_argument errors;
//   * Fig. 3: csr_from_dense -> macko_from_csr(b_delta 2) -> values
//     [1,2,0,3,4], packed deltas 0xB9 0x00, 16-byte tails; dense_from_macko roundtrip;
//     padding_count 1; reference_spmv(ones) = 10;
//   * random matrices, every b_delta: dense -> CSR -> MACKO -> dense roundtrip, padding_count,
//     reference_spmv == dense_mv bit-exactly in integer mode, the worst case
//     1x32;
//   * errors: validate_macko / dense_from_macko on a corrupt matrix -> macko::FormatError;
//     bad b_delta / non-canonical CSR -> std::invalid_argument; dimension mismatch.
// Prints "dropin_ref ok".  Built by `make cpptest`; run by tests/test_cpp_dropin.py.
#include <immintrin.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "bitpack.hpp"
#include "convert.hpp"
#include "errors.hpp"
#include "fp16.hpp"
#include "macko/spmv.hpp"
#include "matrix.hpp"

namespace {

int failures = 0;
#define EXPECT(cond)                                                        \
    do {                                                                    \
        if (!(cond)) {                                                      \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
            ++failures;                                                     \
        }                                                                   \
    } while (0)

template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

uint64_t lcg(uint64_t& s) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return s >> 33;
}

macko::Half H(int v) { return macko::half_from_int(v); }

void test_fp16() {
    for (uint32_t h = 0; h < 65536; ++h) {
        const bool snan = ((h & 0x7C00u) == 0x7C00u) && (h & 0x3FFu) && !(h & 0x200u);
        const float mine = macko::half_to_float(macko::Half{(uint16_t)h});
        const float hw = _cvtsh_ss((unsigned short)h);
        uint32_t a, b;
        std::memcpy(&a, &mine, 4);
        std::memcpy(&b, &hw, 4);
        if (snan) b &= ~0x00400000u;  // hardware quiets signalling NaNs; the reference does not
        EXPECT(a == b);
        if (a != b) break;
        EXPECT(macko::half_table()[h] == mine || mine != mine);
    }
    uint64_t s = 7;
    for (uint64_t i = 0; i < (1u << 24); ++i) {
        uint32_t u = (uint32_t)(i * 256u + (lcg(s) & 0xFFu));  // every 256-pattern block, one random low byte
        float f;
        std::memcpy(&f, &u, 4);
        const uint16_t mine = macko::float_to_half(f).bits, hw = (uint16_t)_cvtss_sh(f, _MM_FROUND_TO_NEAREST_INT);
        EXPECT(mine == hw);
        if (mine != hw) {
            std::printf("  float bits 0x%08x: mine 0x%04x hw 0x%04x\n", u, mine, hw);
            break;
        }
    }
    EXPECT(macko::float_to_half(65520.0f).bits == 0x7C00u);
    EXPECT(macko::float_to_half(65519.0f).bits == 0x7BFFu);
    EXPECT(macko::float_to_half(1.0f).bits == 0x3C00u);
}

void test_bitpack() {
    EXPECT(macko::pack_deltas({2, 3}, 4) == std::vector<uint8_t>{0x21});
    EXPECT(macko::pack_deltas({16}, 8) == std::vector<uint8_t>{0x0F});
    const std::vector<uint8_t> fig3 = macko::pack_deltas({2, 3, 4, 3, 1}, 2);
    EXPECT(fig3.size() == 2 && fig3[0] == 0xB9 && fig3[1] == 0x00);
    EXPECT(macko::unpack_deltas(fig3.data(), 5, 2) == (std::vector<uint32_t>{2, 3, 4, 3, 1}));
    EXPECT(throws<std::invalid_argument>([] { macko::pack_deltas({17}, 4); }));
    EXPECT(throws<std::invalid_argument>([] { macko::pack_deltas({1}, 3); }));
    uint8_t b[2] = {0, 0};
    macko::pack_delta_at(b, 3, 4, 9);
    EXPECT(b[1] == 0x80 && macko::unpack_delta_at(b, 3, 4) == 9);
}

void test_fig3() {
    // 1x14 row, values [1,2,3,4] at 1-based columns [2,5,12,13] (Fig. 3)
    macko::DenseMatrix d = macko::DenseMatrix::zeros(1, 14);
    d.at(0, 1) = H(1);
    d.at(0, 4) = H(2);
    d.at(0, 11) = H(3);
    d.at(0, 12) = H(4);
    const macko::CsrMatrix csr = macko::csr_from_dense(d);
    EXPECT(csr.nnz() == 4 && csr.column_indices == (std::vector<uint32_t>{1, 4, 11, 12}));
    macko::validate_csr(csr);
    macko::MackoParams p;
    p.b_delta = 2;
    const macko::MackoMatrix m = macko::macko_from_csr(csr, p);
    EXPECT(m.pad_nnz() == 5);
    EXPECT(m.values.size() == 8 && m.packed_deltas.size() == 16);  // 16-byte tails (matrix.hpp:77-81)
    const int want[5] = {1, 2, 0, 3, 4};
    for (int i = 0; i < 5; ++i) EXPECT(m.values[i] == H(want[i]));
    EXPECT(m.packed_deltas[0] == 0xB9 && m.packed_deltas[1] == 0x00);
    EXPECT(macko::dense_from_macko(m) == d);
    EXPECT(macko::padding_count(m) == 1);
    macko::validate_macko(m);
    const macko::Vector ones(14, H(1));
    const macko::Vector y = macko::reference_spmv(m, ones);
    EXPECT(y.size() == 1 && y[0] == H(10));
    EXPECT(macko::dense_mv(d, ones)[0] == H(10));
}

void test_random() {
    uint64_t s = 12345;
    for (unsigned bits : {1u, 2u, 4u, 8u}) {
        for (int trial = 0; trial < 3; ++trial) {
            const size_t R = 50 + lcg(s) % 300, C = 20 + lcg(s) % 3000;
            const uint32_t pct = (uint32_t)(lcg(s) % 100);
            macko::DenseMatrix d = macko::DenseMatrix::zeros(R, C);
            size_t nnz = 0;
            for (size_t i = 0; i < R * C; ++i)
                if (lcg(s) % 100 < pct) {
                    int v = (int)(lcg(s) % 16) - 8;
                    if (v >= 0) ++v;
                    d.data[i] = H(v);
                    ++nnz;
                }
            for (size_t r = 0; r < R; r += 7)
                for (size_t c = 0; c < C; ++c) d.at(r, c) = macko::half_zero();  // empty rows
            nnz = d.nnz();
            macko::MackoParams p;
            p.b_delta = bits;
            const macko::CsrMatrix csr = macko::csr_from_dense(d);
            EXPECT(csr.nnz() == nnz);
            const macko::MackoMatrix m = macko::macko_from_csr(csr, p);
            macko::validate_macko(m);
            EXPECT(macko::dense_from_macko(m) == d);
            EXPECT(macko::padding_count(m) == m.pad_nnz() - nnz);
            macko::Vector x(C);
            for (auto& v : x) v = H((int)(lcg(s) % 17) - 8);
            EXPECT(macko::reference_spmv(m, x) == macko::dense_mv(d, x));  // integer mode: exact
            // the stored elements decode, through the reference's own header decoder, to the nonzeros + pads
            size_t seen = 0;
            for (size_t r = 0; r < R; ++r)
                macko::for_each_row_element(m, r, [&](size_t, size_t col, macko::Half v) {
                    EXPECT(col < C && (macko::half_is_zero(v) || d.at(r, col) == v));
                    ++seen;
                });
            EXPECT(seen == m.pad_nnz());
        }
    }
    // 1x32, one nonzero at column 31, b_delta 4 -> one pad (column 15), delta 16
    macko::DenseMatrix w = macko::DenseMatrix::zeros(1, 32);
    w.at(0, 31) = H(1);
    const macko::MackoMatrix m = macko::macko_from_csr(macko::csr_from_dense(w), macko::MackoParams{});
    EXPECT(m.pad_nnz() == 2 && macko::padding_count(m) == 1);
    EXPECT(macko::unpack_delta_at(m.packed_deltas.data(), 0, 4) == 16 && macko::unpack_delta_at(m.packed_deltas.data(), 1, 4) == 16);
}

void test_errors() {
    macko::DenseMatrix d = macko::DenseMatrix::zeros(4, 64);
    for (size_t c = 0; c < 64; c += 3) d.at(1, c) = H(2);
    macko::MackoMatrix m = macko::macko_from_csr(macko::csr_from_dense(d), macko::MackoParams{});
    macko::MackoMatrix bad = m;
    for (auto& b : bad.packed_deltas) b = 0xFF;  // every delta 16: walks past the column bound
    EXPECT(throws<macko::FormatError>([&] { macko::validate_macko(bad); }));
    EXPECT(throws<macko::FormatError>([&] { macko::dense_from_macko(bad); }));
    EXPECT(throws<macko::FormatError>([&] { macko::reference_spmv(bad, macko::Vector(64, H(1))); }));
    macko::MackoParams p3;
    p3.b_delta = 3;
    EXPECT(throws<std::invalid_argument>([&] { macko::macko_from_csr(macko::csr_from_dense(d), p3); }));
    macko::CsrMatrix unsorted = macko::csr_from_dense(d);
    std::swap(unsorted.column_indices[0], unsorted.column_indices[1]);
    EXPECT(throws<std::invalid_argument>([&] { macko::validate_csr(unsorted); }));
    EXPECT(throws<std::invalid_argument>([&] { macko::macko_from_csr(unsorted, macko::MackoParams{}); }));
    EXPECT(throws<std::invalid_argument>([&] { macko::reference_spmv(m, macko::Vector(63)); }));
    EXPECT(throws<std::invalid_argument>([&] { macko::dense_mv(d, macko::Vector(65)); }));
}

}  // namespace

int main() {
    test_fp16();
    test_bitpack();
    test_fig3();
    test_random();
    test_errors();
    if (failures) {
        std::printf("dropin_ref FAILED (%d)\n", failures);
        return 1;
    }
    std::printf("dropin_ref ok\n");
    return 0;
}
