// Internal interface of the inner-Gram route of the randomized SVD (gram_route.cu).
#pragma once
#include <vector>

#include "common.cuh"

namespace fpi {

// inner = [D diag(dscale) | S]  (p x (sd + q2)): the column update's [U Sigma | T] (pinv.py:202-203)
struct SparseGramIn {
  int64_t p = 0, sd = 0, q2 = 0;
  const double* D = nullptr;  // p x sd (ld ldd); rows outside nz_rows are zero when nzr >= 0
  int64_t ldd = 0;
  const double* dscale = nullptr;
  int64_t nzr = -1;                 // >= 0: only these rows of D are nonzero
  const int32_t* nz_rows = nullptr;
  const double* Dnz = nullptr;      // nzr x sd, ld sd
  const int64_t* s_ptr = nullptr;   // S: p x q2 CSR
  const int32_t* s_idx = nullptr;
  const double* s_val = nullptr;
  const int64_t* st_ptr = nullptr;  // S^T: q2 x p CSR (rows ascending within each row)
  const int32_t* st_idx = nullptr;
  const double* st_val = nullptr;
  int64_t s_nnz = 0;
};

struct GramPlan {
  bool use = false;
  double t_gram = 0.0, t_direct = 0.0;  // modelled seconds of the two ways to Z = inner^T inner X
  std::vector<int32_t> heavy;           // densified columns of S (ascending)
  std::vector<int32_t> light;           // the others (ascending)
  int64_t heavy_nnz = 0, light_nnz = 0;
};

// Decide between Z = inner^T (inner X) (two passes over inner with k columns) and Z = H X with
// H = inner^T inner formed once; env FPI_GRAM_ROUTE=0/1 forces the choice (when feasible).
GramPlan plan_inner_gram(fpi_context* h, const SparseGramIn& in, int64_t k);
// H = inner^T inner (q x q, q = sd + q2, row-major, ld ldh)
void inner_gram(fpi_context* h, const SparseGramIn& in, const GramPlan& plan, double* H, int64_t ldh);

}  // namespace fpi
