// Internal interfaces of the dense FP64 building blocks (linalg.cu).
#pragma once
#include "common.cuh"

namespace fpi {
void cholesky_lower(fpi_context* h, int64_t n, double* A, int64_t lda, int* h_info);
void trsm_lower_left(fpi_context* h, int64_t n, const double* L, int64_t ldl, double* X, int64_t ldx, int64_t nrhs);
// L (lower, upper zeroed) and L^-1 of an SPD matrix in one dataflow kernel; false if disabled
bool chol_inverse_dataflow(fpi_context* h, int64_t n, const double* G, int64_t ldg, double* L, int64_t ldl,
                           double* Linv, int64_t ldi, int* h_info);
void lower_inverse(fpi_context* h, int64_t n, const double* L, int64_t ldl, double* Linv, int64_t ldi);
// eigenvalues descending in w (n), eigenvectors as columns of V (n x n); returns Jacobi sweeps used
// Converged when every |a_pq| <= tol * sqrt(|a_pp a_qq|) (relative), or, with `absolute`,
// <= tol * max_i |a_ii|; also stops when the measure stagnates at rounding level.
int sym_eig(fpi_context* h, int64_t n, const double* A, int64_t lda, double* w, double* V, int64_t ldv,
            int max_sweeps, double tol = 1e-14, bool absolute = false);
// Independent eigenproblems in one cooperative launch (all solved concurrently).
void sym_eig_batched(fpi_context* h, int nprob, const int64_t* n, const double* const* A, const int64_t* lda,
                     double* const* w, double* const* V, const int64_t* ldv, int max_sweeps, double tol,
                     bool absolute, int* sweeps_out);
void transpose(fpi_context* h, int64_t M, int64_t N, const double* A, int64_t lda, double* B, int64_t ldb);
void col_sumsq(fpi_context* h, int64_t M, int64_t N, const double* A, int64_t lda, double* out);
void scale_cols(fpi_context* h, int64_t M, int64_t N, double* A, int64_t lda, const double* s, bool divide);
void scale_rows(fpi_context* h, int64_t M, int64_t N, double* A, int64_t lda, const double* s);
void canonical_signs_vt(fpi_context* h, int64_t r, int64_t q, double* Vt, int64_t ldvt, double* sign_out);
void canonical_signs(fpi_context* h, int64_t r, int64_t p, int64_t q, double* U, int64_t ldu, double* Vt,
                     int64_t ldvt);
}  // namespace fpi
