// macko_cuda.hpp — header-only C++ wrapper over the C-ABI (include/macko_cuda.h).
//
// The drop-in for C++ callers of the reference (proj/src/*.hpp): the wrapper is templated on
// the caller's matrix / vector types, so it accepts the reference's own macko::MackoMatrix,
// macko::DenseMatrix and macko::Vector (matrix.hpp:12-71) unchanged — any type with the same
// member names works (values / packed_deltas / row_pointers / rows / cols / params.b_delta,
// payloads of 2-byte fp16 bit patterns).  C-ABI status codes become exceptions with the
// reference's taxonomy: std::invalid_argument (bitpack.cpp:14-15) and FormatError / IoError /
// InfeasibleError (errors.hpp:9-21) — the reference's own types whenever its errors.hpp is on the
// include path.  The reference's free functions themselves (convert.hpp, fp16.hpp, bitpack.hpp and
// the SPEC executors in macko/spmv.hpp) are provided by libmacko.so (csrc/dropin/).
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../macko_cuda.h"

#if __has_include("errors.hpp")
#include "errors.hpp"  // the reference's exception taxonomy (proj/src/errors.hpp:9-21)
#endif

namespace macko {
namespace cuda {

// With the reference's errors.hpp on the include path (-I proj/src) the wrapper throws the
// reference's own exception types; otherwise equivalents with the same bases.
#if __has_include("errors.hpp")
using FormatError = ::macko::FormatError;
using IoError = ::macko::IoError;
using InfeasibleError = ::macko::InfeasibleError;
#else
struct FormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InfeasibleError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#endif
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <class FormatErrorT = FormatError, class IoErrorT = IoError, class InfeasibleErrorT = InfeasibleError>
inline void check(macko_status s) {
    if (s == MACKO_OK) return;
    const std::string msg = macko_last_error();
    switch (s) {
        case MACKO_EINVAL: throw std::invalid_argument(msg);
        case MACKO_EFORMAT: throw FormatErrorT(msg);
        case MACKO_EIO: throw IoErrorT(msg);
        case MACKO_EINFEASIBLE: throw InfeasibleErrorT(msg);
        case MACKO_ENOMEM: throw std::bad_alloc();
        default: throw CudaError(msg);
    }
}

// A MACKO matrix resident in HBM (owns the macko_dev_matrix handle).
class DeviceMatrix {
  public:
    DeviceMatrix() = default;
    explicit DeviceMatrix(macko_dev_matrix* h) : h_(h) {}
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
    DeviceMatrix(DeviceMatrix&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    DeviceMatrix& operator=(DeviceMatrix&& o) noexcept {
        if (this != &o) {
            reset();
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }
    ~DeviceMatrix() { reset(); }

    // Upload a host MackoMatrix (reference matrix.hpp:57-67 layout).
    template <class MackoMatrixT>
    static DeviceMatrix upload(const MackoMatrixT& m, int device = 0, void* stream = nullptr) {
        static_assert(sizeof(m.values[0]) == 2, "values must be 2-byte fp16 bit patterns");
        macko_dev_matrix* h = nullptr;
        check(macko_dev_upload(device, m.rows, m.cols, m.params.b_delta,
                               reinterpret_cast<const uint16_t*>(m.values.data()), m.values.size(),
                               reinterpret_cast<const uint8_t*>(m.packed_deltas.data()), m.packed_deltas.size(),
                               m.row_pointers.data(), stream, &h));
        return DeviceMatrix(h);
    }

    // GPU compressor from a dense fp16 matrix already in device memory.
    static DeviceMatrix from_dense(const uint16_t* d_dense, uint64_t rows, uint64_t cols, uint64_t ld,
                                   unsigned b_delta = 4, int device = 0, void* stream = nullptr) {
        macko_dev_matrix* h = nullptr;
        check(macko_dev_from_dense(device, d_dense, rows, cols, ld, b_delta, stream, &h));
        return DeviceMatrix(h);
    }

    macko_dev_info info() const {
        macko_dev_info i{};
        check(macko_dev_get_info(h_, &i));
        return i;
    }

    // Device -> host copy into a MackoMatrix-like value (bit-identical to the reference encoder).
    template <class MackoMatrixT>
    MackoMatrixT download(void* stream = nullptr) const {
        const macko_dev_info i = info();
        MackoMatrixT m;
        m.rows = i.rows;
        m.cols = i.cols;
        m.params.b_delta = i.b_delta;
        m.values.resize(i.values_bytes / 2);
        m.packed_deltas.resize(i.delta_bytes);
        m.row_pointers.resize(i.rows + 1);
        check(macko_dev_download(h_, reinterpret_cast<uint16_t*>(m.values.data()),
                                 reinterpret_cast<uint8_t*>(m.packed_deltas.data()), m.row_pointers.data(), stream));
        return m;
    }

    void validate(void* stream = nullptr) const { check(macko_dev_validate(h_, stream)); }

    // y = A*x on device buffers (stream ordered).
    // pdl: programmatic dependent launch after the previous kernel on the stream (SpMV chains)
    void spmv(const uint16_t* d_x, uint16_t* d_y, void* stream = nullptr, bool pdl = false) const {
        check(macko_dev_spmv_ex(h_, d_x, d_y, stream, pdl ? MACKO_SPMV_PDL : 0u));
    }

    // reference_spmv drop-in on host vectors: H2D x, kernel, D2H y.
    template <class VectorT>
    VectorT spmv_host(const VectorT& x, void* stream = nullptr) {
        static_assert(sizeof(x[0]) == 2, "vector entries must be 2-byte fp16 bit patterns");
        const macko_dev_info i = info();
        if (x.size() != i.cols) throw std::invalid_argument("dimension mismatch: x must have cols entries");
        VectorT y(i.rows);
        check(macko_spmv_host(h_, reinterpret_cast<const uint16_t*>(x.data()), reinterpret_cast<uint16_t*>(y.data()),
                              stream));
        return y;
    }

    macko_dev_matrix* handle() const { return h_; }

  private:
    void reset() {
        if (h_) macko_dev_free(h_);
        h_ = nullptr;
    }
    macko_dev_matrix* h_ = nullptr;
};

}  // namespace cuda
}  // namespace macko
