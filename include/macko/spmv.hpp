// spmv.hpp — the SPEC's executor operations as C++ free functions over the reference's own types
// (the reference lists spmv.cpp in proj/src/CMakeLists.txt but ships neither it
// nor a header).  Implemented by libmacko.so (paper_2511_13061_b200/csrc/dropin/), which runs them
// on the GPU through libmacko_cuda.so.  Include after the reference's matrix.hpp is on the path
// (-I proj/src).
#pragma once

#include "matrix.hpp"

namespace macko {

// dense_mv: Y[r] = sum_c M[r,c] V[c], fp16 products widened to fp32, sequential
// accumulation, one RNE.  Host computation (the correctness oracle of the dense path).
// Throws std::invalid_argument on a dimension mismatch.
Vector dense_mv(const DenseMatrix& m, const Vector& v);

// reference_spmv on the GPU: the matrix is uploaded (and validated) per call,
// y = A v with fp32 accumulation and one RNE per row.  Bit-exact with the sequential reference in
// integer mode; otherwise within |dy| <= ulp16(|y|) + 2 n 2^-24 sum|a x| (the kernel's summation
// order).  For repeated products keep the matrix resident instead:
// macko::cuda::DeviceMatrix (macko/macko_cuda.hpp).
// Throws std::invalid_argument on a dimension mismatch, macko::FormatError on a corrupt matrix.
Vector reference_spmv(const MackoMatrix& m, const Vector& v);

}  // namespace macko
