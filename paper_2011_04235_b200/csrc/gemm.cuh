// Internal interface of the FP64 DMMA GEMM (gemm.cu).
#pragma once
#include "common.cuh"

namespace fpi {
// C = alpha * op(A) op(B) + beta * C; row-major; op(A) is M x K, op(B) is K x N.
// sym: the caller asserts C is symmetric (A == B, exactly one of ta / tb): only the lower
// tiles are computed (half the flops) and mirrored.
void gemm(fpi_context* h, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
          int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, bool sym = false);
}  // namespace fpi
