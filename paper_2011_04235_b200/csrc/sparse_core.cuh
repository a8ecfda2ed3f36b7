// Dense core of a skewed sparse block (sparse_core.cu): the heavy rows x heavy columns rectangle
// of T = [A12; A22] is nearly dense on Zipf inputs, so its share of T X / T^T B runs on DMMA from
// a dense panel and the gather SpMM keeps only the remainder.
#pragma once
#include "common.cuh"

namespace fpi {

struct SparseCore {
  bool use = false;
  int64_t nR = 0, nC = 0, core_nnz = 0, rem_nnz = 0;
  Scratch<int32_t> rows, cols;     // ascending ids of the core rows / columns of S
  Scratch<double> dense;           // nR x nC row-major: S[rows, cols]
  Scratch<int64_t> r_ptr, rt_ptr;  // remainder S' = S minus the core entries (p + 1), and S'^T (q2 + 1)
  Scratch<int32_t> r_idx, rt_idx;
  Scratch<double> r_val, rt_val;
};

// S: p x q2 CSR with nnz stored entries, St its transpose.  Leaves core.use false when the
// rectangle would not pay (small, or too sparse for the tensor pipe to beat the gathers).
void build_sparse_core(fpi_context* h, int64_t p, int64_t q2, int64_t nnz, const int64_t* s_ptr,
                       const int32_t* s_idx, const double* s_val, const int64_t* st_ptr, const int32_t* st_idx,
                       const double* st_val, SparseCore& core);

}  // namespace fpi
