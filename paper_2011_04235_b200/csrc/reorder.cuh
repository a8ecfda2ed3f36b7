// Hub/spoke reordering (Algorithm 2, reference reorder.py:158-287): the two device drivers.
#pragma once
#include "common.cuh"

namespace fpi {

struct ReorderOut {
  int64_t m1, n1, m2, n2, T;
  // SURVEY 8(d) work accounting: sum over iterations of E_t (edges with both endpoints active at
  // the iteration's entry) and V_t (active nodes at entry); algorithmic bytes = 24 E + 32 V
  int64_t e_sum = 0, v_sum = 0;
};

// One persistent cooperative kernel for the whole iteration loop (reorder_persistent.cu).
// Returns false (nothing written) when the problem is outside its static limits (hub quota per
// side above the in-kernel cap, or no co-resident grid); the caller then uses the host loop.
bool run_reorder_persistent(fpi_context* h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                            const int32_t* d_indices, double k, int64_t* d_row_fwd, int64_t* d_col_fwd,
                            ReorderOut& out);

}  // namespace fpi
