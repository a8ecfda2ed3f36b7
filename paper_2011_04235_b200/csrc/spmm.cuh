// Internal interface of the CSR x dense kernels (spmm.cu).
#pragma once
#include "common.cuh"

namespace fpi {
// Y = alpha * diag(row_scale) * A * X + beta * Y  (row_scale may be null)
void spmm(fpi_context* h, int64_t p, int64_t q, int64_t k, const int64_t* indptr, const int32_t* indices,
          const double* values, const double* row_scale, double alpha, const double* X, int64_t ldx, double beta,
          double* Y, int64_t ldy);
}  // namespace fpi
