// Internal interfaces of the sparse structure kernels (sparse.cu).
#pragma once
#include "common.cuh"
#include "cub_util.cuh"

namespace fpi {

struct PartOut {
  int64_t* a11_ptr; int32_t* a11_idx; double* a11_val;
  int64_t* t_ptr; int32_t* t_idx; double* t_val;
  int64_t* tt_ptr; int32_t* tt_idx; double* tt_val;
  int64_t* a21_ptr; int32_t* a21_idx; double* a21_val;
  int64_t* a21t_ptr; int32_t* a21t_idx; double* a21t_val;
};

void expand_rows(fpi_context* h, int64_t m, const int64_t* indptr, int32_t* rows);
void build_csr(fpi_context* h, CubTemp& tmp, int64_t cnt, const int32_t* major, const int32_t* minor,
               const double* vals, int64_t nmajor, int64_t nminor, int64_t* out_ptr, int32_t* out_idx,
               double* out_val);
void csr_transpose(fpi_context* h, int64_t p, int64_t q, int64_t nnz, const int64_t* indptr, const int32_t* indices,
                   const double* values, int64_t* t_ptr, int32_t* t_idx, double* t_val);
void partition(fpi_context* h, int64_t m, int64_t n, int64_t nnz, const int64_t* indptr, const int32_t* indices,
               const double* values, const int64_t* row_fwd, const int64_t* col_fwd, int64_t m1, int64_t n1,
               int64_t nspans, const int64_t* spans, fpi_partition_info* info, const PartOut* out);

}  // namespace fpi
