// Internal interfaces of the SVD engines (svd_engine.cu).
#pragma once
#include "common.cuh"

namespace fpi {
void dense_svd(fpi_context* h, int64_t p, int64_t q, const double* M, int64_t ldm, int64_t rank, double* U,
               double* sigma, double* Vt, fpi_svd_diag* diag);
void dense_svd_batched(fpi_context* h, int nb, const int64_t* p, const int64_t* q, const double* const* M,
                       const int64_t* ldm, const int64_t* rank, double* const* U, double* const* sigma,
                       double* const* Vt);
void complete_null_left(fpi_context* h, int64_t p, int64_t rank, double* U, int64_t ldu, const double* sigma,
                        fpi_svd_diag* diag);
}  // namespace fpi
