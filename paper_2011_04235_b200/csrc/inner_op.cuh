// Internal interface of the SVD engine's inner-matrix operator and the randomized-SVD pieces
// shared with the sharded engine (svd_engine.cu, sharded.cu).
#pragma once
#include "common.cuh"
#include "gram_route.cuh"
#include "sparse_core.cuh"

namespace fpi {

// inner-matrix operator: [D diag(dscale) | S] (horizontal) -- D may be null
struct InnerOp {
  int64_t p = 0, q = 0;
  const double* D = nullptr;
  int64_t ldd = 0, sd = 0;
  const double* dscale = nullptr;
  const int64_t* s_ptr = nullptr;
  const int32_t* s_idx = nullptr;
  const double* s_val = nullptr;  // p x (q - sd)
  const int64_t* st_ptr = nullptr;
  const int32_t* st_idx = nullptr;
  const double* st_val = nullptr;  // (q - sd) x p
  // optional: only nzr rows of D are nonzero (rows listed in nz_rows, gathered into Dnz)
  int64_t nzr = -1;
  const int32_t* nz_rows = nullptr;
  const double* Dnz = nullptr;
  int64_t s_nnz = 0;  // stored entries of the sparse part (cost model only)
  // optional: the heavy rows x heavy columns rectangle of the sparse part as a dense panel
  // (sparse_core.cu); apply / applyT then run the remainder SpMM plus a gathered DMMA product
  const SparseCore* core = nullptr;

  SparseGramIn gram_in() const {
    SparseGramIn g;
    g.p = p;
    g.sd = D ? sd : 0;
    g.q2 = q - g.sd;
    g.D = D;
    g.ldd = ldd;
    g.dscale = dscale;
    g.nzr = nzr;
    g.nz_rows = nz_rows;
    g.Dnz = Dnz;
    g.s_ptr = s_ptr;
    g.s_idx = s_idx;
    g.s_val = s_val;
    g.st_ptr = st_ptr;
    g.st_idx = st_idx;
    g.st_val = st_val;
    g.s_nnz = s_nnz;
    return g;
  }

  // flop-equivalent cost of apply() with k columns (a gathered SpMM byte ~ 10 flops on B200)
  double apply_cost(int64_t k) const {
    const double dense_rows = (double)(nzr >= 0 ? nzr : p);
    const double gathered = core ? (double)core->rem_nnz : (double)s_nnz;
    const double cells = core ? (double)core->nR * (double)core->nC : 0.0;
    return (D && sd > 0 ? 2.0 * dense_rows * (double)sd * (double)k : 0.0) + 10.0 * 8.0 * gathered * (double)k +
           2.0 * cells * (double)k;
  }

  // B (p x k) = inner * X (q x k)
  void apply(fpi_context* h, const double* X, int64_t k, double* B) const;
  // Z (q x k) = inner^T * B (p x k)
  void applyT(fpi_context* h, const double* B, int64_t k, double* Z) const;
  // sparse part only: B (+)= S * Xs (Xs: (q - sd) x k), Z2 = S^T * B (Z2: (q - sd) x k)
  void sparse_apply(fpi_context* h, const double* Xs, int64_t k, double beta, double* B) const;
  void sparse_applyT(fpi_context* h, const double* B, int64_t k, double* Z2) const;
  // dense copy (p x q)
  void densify(fpi_context* h, double* out) const;
};

// Q = B L^-T orthonormal from the Gram G = B^T B (k x k): CholeskyQR or an eigen-based factor
void orth_factor(fpi_context* h, int64_t k, const double* Gm, double* Linv, fpi_svd_diag* diag);
void sketch_normal(fpi_context* h, int64_t seed, int64_t rows, int64_t cols, double* d_out, int64_t ld);
void symmetrize(fpi_context* h, int64_t n, double* A, int64_t lda);

}  // namespace fpi
