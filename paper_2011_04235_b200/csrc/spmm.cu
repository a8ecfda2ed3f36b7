// CSR x dense-panel products (the sparse half of every sketch / projection):
//   Y = alpha * A * X + beta * Y        A: p x q CSR, X: q x k row-major
// which covers inner @ X (svd.py:133 via sparse.py:28) and, applied to the
// transposed CSR, inner^T @ Q (svd.py:135 via sparse.py:39) and Y^T U (pinv.py:75).
//
// One warp owns one output row and a 128-column slice (4 doubles per lane,
// vectorised double2 loads); grid.y walks the column slices so that a slice
// of X stays L2-resident while every row streams past it.  nnz are fetched 32
// at a time per warp and broadcast with shuffles.  Each output element is
// summed by one lane in CSR order: deterministic.
#include "common.cuh"
#include "capi_guard.cuh"
#include "spmm.cuh"
#include "instrument.cuh"

namespace fpi {
namespace {

constexpr int WARPS = 8;       // warps per CTA
constexpr int SLICE = 128;     // output columns per warp pass (4 per lane)

template <bool VEC>
__global__ void __launch_bounds__(WARPS * 32)
    k_spmm(int64_t p, int64_t k, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
           const double* __restrict__ values, const double* __restrict__ row_scale, double alpha,
           const double* __restrict__ X, int64_t ldx, double beta, double* __restrict__ Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t c0 = (int64_t)blockIdx.y * SLICE + lane * 4;
  for (int64_t row = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); row < p; row += (int64_t)gridDim.x * WARPS) {
    const int64_t b = indptr[row], e = indptr[row + 1];
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    for (int64_t base = b; base < e; base += 32) {
      const int64_t my = base + lane;
      int32_t col = 0;
      double val = 0.0;
      if (my < e) {
        col = indices[my];
        val = values[my];
      }
      const int cnt = (int)((e - base) < 32 ? (e - base) : 32);
      for (int j = 0; j < cnt; ++j) {
        const int32_t cj = __shfl_sync(0xffffffffu, col, j);
        const double vj = __shfl_sync(0xffffffffu, val, j);
        const double* xr = X + (int64_t)cj * ldx;
        if (VEC && c0 + 3 < k) {
          const double2 a = *reinterpret_cast<const double2*>(xr + c0);
          const double2 bb = *reinterpret_cast<const double2*>(xr + c0 + 2);
          acc0 = fma(vj, a.x, acc0);
          acc1 = fma(vj, a.y, acc1);
          acc2 = fma(vj, bb.x, acc2);
          acc3 = fma(vj, bb.y, acc3);
        } else {
          if (c0 < k) acc0 = fma(vj, xr[c0], acc0);
          if (c0 + 1 < k) acc1 = fma(vj, xr[c0 + 1], acc1);
          if (c0 + 2 < k) acc2 = fma(vj, xr[c0 + 2], acc2);
          if (c0 + 3 < k) acc3 = fma(vj, xr[c0 + 3], acc3);
        }
      }
    }
    double s = row_scale ? alpha * row_scale[row] : alpha;
    double* yr = Y + row * ldy;
    double acc[4] = {acc0, acc1, acc2, acc3};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (c0 + q < k) yr[c0 + q] = beta == 0.0 ? s * acc[q] : s * acc[q] + beta * yr[c0 + q];
    }
  }
}

}  // namespace

void spmm(fpi_context* h, int64_t p, int64_t q, int64_t k, const int64_t* indptr, const int32_t* indices,
          const double* values, const double* row_scale, double alpha, const double* X, int64_t ldx, double beta,
          double* Y, int64_t ldy) {
  if (p <= 0 || k <= 0) return;
  const int64_t slices = (k + SLICE - 1) / SLICE;
  FPI_REQUIRE(slices < 65536, FPI_ECAPACITY, "spmm: too many column slices");
  int64_t gx = (p + WARPS - 1) / WARPS;
  const int64_t cap = (int64_t)h->num_sms * 16;
  if (gx > cap) gx = cap;
  dim3 grid((unsigned)gx, (unsigned)slices);
  int64_t nnz = 0;
  if (h->timing_on) nnz = host_read(indptr + p, h->stream);
  // algorithmic bytes: 12 nnz + 4 (p + 1) + 8 q k + 8 p k
  KTimer kt(h, "spmm_csr", 2.0 * (double)nnz * (double)k,
            12.0 * nnz + 4.0 * (p + 1) + 8.0 * (double)q * k + 8.0 * (double)p * k);
  const bool vec = (ldx % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  if (vec)
    k_spmm<true><<<grid, WARPS * 32, 0, h->stream>>>(p, k, indptr, indices, values, row_scale, alpha, X, ldx, beta,
                                                     Y, ldy);
  else
    k_spmm<false><<<grid, WARPS * 32, 0, h->stream>>>(p, k, indptr, indices, values, row_scale, alpha, X, ldx, beta,
                                                      Y, ldy);
  FPI_LAUNCH_CHECK();
  note_launch(h);
}

}  // namespace fpi

extern "C" int fpi_spmm(fpi_handle h, int64_t p, int64_t q, int64_t k, const int64_t* d_indptr,
                        const int32_t* d_indices, const double* d_values, double alpha, const double* d_X,
                        int64_t ldx, double beta, double* d_Y, int64_t ldy) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(p >= 0 && q >= 0 && k >= 0 && ldx >= k && ldy >= k, FPI_EDOMAIN, "bad spmm shape");
  fpi::spmm(h, p, q, k, d_indptr, d_indices, d_values, nullptr, alpha, d_X, ldx, beta, d_Y, ldy);
  FPI_API_END(h)
}
