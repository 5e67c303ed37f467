// dropin_test.cpp — the C++ drop-in check (GPU): the reference's own types and encoder
// (/root/reference/proj/src headers; encoder bodies from oracle/ref_shim.cpp) feed
// libmacko_cuda.so through include/macko/macko_cuda.hpp with no conversion code.
//   1. macko::MackoMatrix from macko_from_csr -> DeviceMatrix::upload -> spmv_host must equal the
//      reference_spmv (sequential fp32, reference decoder + fp16 LUT) in integer mode, bit for bit;
//   2. DeviceMatrix::from_dense on the GPU -> download<macko::MackoMatrix>() must equal the
//      reference encoder's arrays byte for byte;
//   3. a corrupt matrix is rejected with a FormatError.
// Built by `make cpptest` (needs /root/reference for the headers); run by tests/test_cpp_dropin.py.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "convert.hpp"
#include "errors.hpp"
#include "fp16.hpp"
#include "matrix.hpp"
#include "macko/macko_cuda.hpp"

namespace {

macko::Vector reference_spmv(const macko::MackoMatrix& m, const macko::Vector& x) {
    macko::Vector y(m.rows);
    const float* lut = macko::half_table();
    for (size_t r = 0; r < m.rows; ++r) {
        float acc = 0.0f;
        macko::for_each_row_element(m, r, [&](size_t, size_t col, macko::Half v) { acc += lut[v.bits] * lut[x[col].bits]; });
        y[r] = macko::float_to_half(acc);
    }
    return y;
}

uint64_t lcg(uint64_t& s) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return s >> 33;
}

int fail(const char* what) {
    std::printf("FAIL: %s\n", what);
    return 1;
}

}  // namespace

int main() {
    const size_t R = 777, C = 3001;
    uint64_t seed = 12345;
    macko::DenseMatrix d = macko::DenseMatrix::zeros(R, C);
    for (auto& h : d.data)
        if (lcg(seed) % 2) h = macko::half_from_int((int)(lcg(seed) % 16) - 8);
    for (auto& h : d.data)
        if (macko::half_is_zero(h)) h = macko::Half{0};
    macko::Vector x(C);
    for (auto& h : x) h = macko::half_from_int((int)(lcg(seed) % 17) - 8);

    const macko::MackoMatrix m = macko::macko_from_csr(macko::csr_from_dense(d), macko::MackoParams{16, 4});

    // 1. upload + spmv_host == reference_spmv (integer mode: bit-exact)
    auto dm = macko::cuda::DeviceMatrix::upload(m);
    const macko::Vector y = dm.spmv_host(x);
    const macko::Vector y_ref = reference_spmv(m, x);
    if (!(y == y_ref)) return fail("spmv_host != reference_spmv");

    // 2. GPU compressor == reference encoder, byte for byte
    uint16_t* d_dense = nullptr;
    if (cudaMalloc(&d_dense, R * C * 2) != cudaSuccess) return fail("cudaMalloc");
    cudaMemcpy(d_dense, d.data.data(), R * C * 2, cudaMemcpyHostToDevice);
    auto dg = macko::cuda::DeviceMatrix::from_dense(d_dense, R, C, C, 4);
    const auto mg = dg.download<macko::MackoMatrix>();
    cudaFree(d_dense);
    if (mg.row_pointers != m.row_pointers) return fail("row_pointers differ");
    if (mg.values != m.values) return fail("values differ");
    if (mg.packed_deltas != m.packed_deltas) return fail("packed_deltas differ");
    if (!(dg.spmv_host(x) == y_ref)) return fail("compressed-on-GPU spmv differs");

    // 3. a decoded column past C is a FormatError
    macko::MackoMatrix bad = m;
    std::memset(bad.packed_deltas.data(), 0xFF, bad.packed_deltas.size() / 2);
    try {
        auto db = macko::cuda::DeviceMatrix::upload(bad);
        return fail("corrupt matrix accepted");
    } catch (const macko::cuda::FormatError&) {
    }
    std::printf("dropin ok: %zux%zu pad_nnz=%zu\n", R, C, m.pad_nnz());
    return 0;
}
