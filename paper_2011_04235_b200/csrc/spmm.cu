// CSR x dense-panel products (the sparse half of every sketch / projection):
//   Y = alpha * diag(row_scale) * A * X + beta * Y     A: p x q CSR, X: q x k row-major
// which covers inner @ X (svd.py:133 via sparse.py:28) and, applied to the
// transposed CSR, inner^T @ Q (svd.py:135 via sparse.py:39) and Y^T U (pinv.py:75).
//
// Short rows: one warp owns one output row and a 128-column slice (4 doubles
// per lane, 16-byte loads), nnz fetched 32 at a time and broadcast with
// shuffles, four X rows in flight per lane.  grid.y walks the column slices so
// a slice of X stays L2-resident while every row streams past it.
// Long rows (hub rows of T^T, popular labels of Y^T, ...): split into segments
// of SEG nonzeros, one warp per (segment, slice) writing a partial row, then
// an ordered per-row reduction of the segments -- balanced and deterministic
// (every output element is summed in a fixed order).
#include "common.cuh"
#include "capi_guard.cuh"
#include "cub_util.cuh"
#include "spmm.cuh"
#include "instrument.cuh"

namespace fpi {
namespace {

constexpr int WARPS = 8;       // warps per CTA
constexpr int SLICE = 128;     // output columns per warp pass (4 per lane)
constexpr int64_t SEG = 512;   // nonzeros per long-row segment (rows longer than this are split)

struct Acc4 {
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
};

template <bool VEC>
__device__ __forceinline__ void accumulate_range(int64_t b, int64_t e, const int32_t* __restrict__ indices,
                                                 const double* __restrict__ values, const double* __restrict__ X,
                                                 int64_t ldx, int64_t k, int64_t c0, int lane, Acc4& acc) {
  for (int64_t base = b; base < e; base += 32) {
    const int64_t my = base + lane;
    int32_t col = 0;
    double val = 0.0;
    if (my < e) {
      col = __ldg(indices + my);
      val = __ldg(values + my);
    }
    const int cnt = (int)((e - base) < 32 ? (e - base) : 32);
    int j = 0;
    if (VEC && c0 + 3 < k) {
      for (; j + 4 <= cnt; j += 4) {
        double2 xa[4], xb[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int32_t cj = __shfl_sync(0xffffffffu, col, j + u);
          v[u] = __shfl_sync(0xffffffffu, val, j + u);
          const double* xr = X + (int64_t)cj * ldx + c0;
          xa[u] = __ldg(reinterpret_cast<const double2*>(xr));
          xb[u] = __ldg(reinterpret_cast<const double2*>(xr + 2));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc.a0 = fma(v[u], xa[u].x, acc.a0);
          acc.a1 = fma(v[u], xa[u].y, acc.a1);
          acc.a2 = fma(v[u], xb[u].x, acc.a2);
          acc.a3 = fma(v[u], xb[u].y, acc.a3);
        }
      }
    }
    for (; j < cnt; ++j) {
      const int32_t cj = __shfl_sync(0xffffffffu, col, j);
      const double vj = __shfl_sync(0xffffffffu, val, j);
      const double* xr = X + (int64_t)cj * ldx;
      if (VEC && c0 + 3 < k) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(xr + c0));
        const double2 bb = __ldg(reinterpret_cast<const double2*>(xr + c0 + 2));
        acc.a0 = fma(vj, a.x, acc.a0);
        acc.a1 = fma(vj, a.y, acc.a1);
        acc.a2 = fma(vj, bb.x, acc.a2);
        acc.a3 = fma(vj, bb.y, acc.a3);
      } else {
        if (c0 < k) acc.a0 = fma(vj, xr[c0], acc.a0);
        if (c0 + 1 < k) acc.a1 = fma(vj, xr[c0 + 1], acc.a1);
        if (c0 + 2 < k) acc.a2 = fma(vj, xr[c0 + 2], acc.a2);
        if (c0 + 3 < k) acc.a3 = fma(vj, xr[c0 + 3], acc.a3);
      }
    }
  }
}

__device__ __forceinline__ void store4(double* yr, int64_t c0, int64_t k, double s, double beta, const Acc4& a) {
  const double acc[4] = {a.a0, a.a1, a.a2, a.a3};
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (c0 + q < k) yr[c0 + q] = beta == 0.0 ? s * acc[q] : s * acc[q] + beta * yr[c0 + q];
}

template <bool VEC>
__global__ void __launch_bounds__(WARPS * 32)
    k_spmm(int64_t p, int64_t k, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
           const double* __restrict__ values, const double* __restrict__ row_scale, double alpha,
           const double* __restrict__ X, int64_t ldx, double beta, double* __restrict__ Y, int64_t ldy,
           int64_t long_thresh) {
  const int lane = threadIdx.x & 31;
  const int64_t c0 = (int64_t)blockIdx.y * SLICE + lane * 4;
  for (int64_t row = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); row < p; row += (int64_t)gridDim.x * WARPS) {
    const int64_t b = indptr[row], e = indptr[row + 1];
    if (e - b > long_thresh) continue;  // handled by the segmented path
    Acc4 acc;
    accumulate_range<VEC>(b, e, indices, values, X, ldx, k, c0, lane, acc);
    const double s = row_scale ? alpha * row_scale[row] : alpha;
    store4(Y + row * ldy, c0, k, s, beta, acc);
  }
}

struct IsLong {
  const int64_t* indptr;
  int64_t thresh;
  __device__ bool operator()(int64_t r) const { return indptr[r + 1] - indptr[r] > thresh; }
};

__global__ void k_iota64(int64_t* a, int64_t n) {
  FPI_GRID_STRIDE(i, n) a[i] = i;
}

__global__ void k_seg_counts(const int64_t* __restrict__ rows, int64_t nl, const int64_t* __restrict__ indptr,
                             int64_t* __restrict__ nseg) {
  FPI_GRID_STRIDE(i, nl) {
    const int64_t r = rows[i];
    nseg[i] = (indptr[r + 1] - indptr[r] + SEG - 1) / SEG;
  }
}

// one warp per (segment, slice): partial row into P[seg][k]
template <bool VEC>
__global__ void __launch_bounds__(WARPS * 32)
    k_spmm_segments(const int64_t* __restrict__ rows, const int64_t* __restrict__ seg_off, int64_t nl,
                    int64_t nseg_total, int64_t k, const int64_t* __restrict__ indptr,
                    const int32_t* __restrict__ indices, const double* __restrict__ values,
                    const double* __restrict__ X, int64_t ldx, double* __restrict__ P) {
  const int lane = threadIdx.x & 31;
  const int64_t c0 = (int64_t)blockIdx.y * SLICE + lane * 4;
  for (int64_t sg = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); sg < nseg_total;
       sg += (int64_t)gridDim.x * WARPS) {
    // owning long row: last i with seg_off[i] <= sg
    int64_t lo = 0, hi = nl - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (seg_off[mid] <= sg) lo = mid; else hi = mid - 1;
    }
    const int64_t r = rows[lo];
    const int64_t b = indptr[r] + (sg - seg_off[lo]) * SEG;
    const int64_t e0 = indptr[r + 1];
    const int64_t e = b + SEG < e0 ? b + SEG : e0;
    Acc4 acc;
    accumulate_range<VEC>(b, e, indices, values, X, ldx, k, c0, lane, acc);
    store4(P + sg * k, c0, k, 1.0, 0.0, acc);
  }
}

__global__ void k_seg_reduce(const int64_t* __restrict__ rows, const int64_t* __restrict__ seg_off, int64_t nl,
                             int64_t k, const double* __restrict__ P, const double* __restrict__ row_scale,
                             double alpha, double beta, double* __restrict__ Y, int64_t ldy) {
  FPI_GRID_STRIDE(e, nl * k) {
    const int64_t i = e / k, c = e - i * k;
    const int64_t s0 = seg_off[i], s1 = seg_off[i + 1];
    double acc = 0.0;
    for (int64_t sg = s0; sg < s1; ++sg) acc += P[sg * k + c];
    const int64_t r = rows[i];
    const double s = row_scale ? alpha * row_scale[r] : alpha;
    double* y = Y + r * ldy + c;
    *y = beta == 0.0 ? s * acc : s * acc + beta * *y;
  }
}

}  // namespace

void spmm(fpi_context* h, int64_t p, int64_t q, int64_t k, const int64_t* indptr, const int32_t* indices,
          const double* values, const double* row_scale, double alpha, const double* X, int64_t ldx, double beta,
          double* Y, int64_t ldy) {
  if (p <= 0 || k <= 0) return;
  cudaStream_t s = h->stream;
  const int64_t slices = (k + SLICE - 1) / SLICE;
  FPI_REQUIRE(slices < 65536, FPI_ECAPACITY, "spmm: too many column slices");
  int64_t nnz = 0;
  if (h->timing_on) nnz = host_read(indptr + p, s);
  // algorithmic bytes: 12 nnz + 4 (p + 1) + 8 q k + 8 p k
  KTimer kt(h, "spmm_csr", 2.0 * (double)nnz * (double)k,
            12.0 * nnz + 4.0 * (p + 1) + 8.0 * (double)q * k + 8.0 * (double)p * k);
  const bool vec = (ldx % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  // long rows
  CubTemp tmp(s);
  Scratch<int64_t> ids(p, s), lrows(p, s);
  Scratch<int> nlong(1, s);
  k_iota64<<<grid_for(p, 256, (int64_t)h->num_sms * 8), 256, 0, s>>>(ids, p);
  select_if(tmp, ids.get(), lrows.get(), nlong.get(), p, IsLong{indptr, SEG}, s);
  const int64_t nl = host_read(nlong.get(), s);
  int64_t gx = (p + WARPS - 1) / WARPS;
  const int64_t cap = (int64_t)h->num_sms * 16;
  if (gx > cap) gx = cap;
  dim3 grid((unsigned)gx, (unsigned)slices);
  if (vec)
    k_spmm<true><<<grid, WARPS * 32, 0, s>>>(p, k, indptr, indices, values, row_scale, alpha, X, ldx, beta, Y, ldy,
                                             SEG);
  else
    k_spmm<false><<<grid, WARPS * 32, 0, s>>>(p, k, indptr, indices, values, row_scale, alpha, X, ldx, beta, Y, ldy,
                                              SEG);
  FPI_LAUNCH_CHECK();
  note_launch(h, 3);
  if (nl == 0) return;
  Scratch<int64_t> nseg(nl + 1, s), seg_off(nl + 1, s);
  FPI_CUDA(cudaMemsetAsync(nseg.get() + nl, 0, sizeof(int64_t), s));
  k_seg_counts<<<grid_for(nl, 256, cap), 256, 0, s>>>(lrows, nl, indptr, nseg);
  exclusive_sum(tmp, nseg.get(), seg_off.get(), nl + 1, s);
  const int64_t total = host_read(seg_off.get() + nl, s);
  Scratch<double> P(total * k, s);
  int64_t gs = (total + WARPS - 1) / WARPS;
  if (gs > cap) gs = cap;
  dim3 g2((unsigned)gs, (unsigned)slices);
  if (vec)
    k_spmm_segments<true><<<g2, WARPS * 32, 0, s>>>(lrows, seg_off, nl, total, k, indptr, indices, values, X, ldx, P);
  else
    k_spmm_segments<false><<<g2, WARPS * 32, 0, s>>>(lrows, seg_off, nl, total, k, indptr, indices, values, X, ldx,
                                                     P);
  k_seg_reduce<<<grid_for(nl * k, 256, cap), 256, 0, s>>>(lrows, seg_off, nl, k, P, row_scale, alpha, beta, Y, ldy);
  FPI_LAUNCH_CHECK();
  note_launch(h, 4);
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
