// CSR x dense-panel products (the sparse half of every sketch / projection):
//   Y = alpha * diag(row_scale) * A * X + beta * Y     A: p x q CSR, X: q x k row-major
// which covers inner @ X (svd.py:133 via sparse.py:28) and, applied to the
// transposed CSR, inner^T @ Q (svd.py:135 via sparse.py:39) and Y^T U (pinv.py:75).
//
// Short rows: one warp owns one output row and a 64-column slice (2 doubles
// per lane; one 16-byte load per lane covers 512 contiguous bytes of an X row),
// nnz fetched 32 at a time and broadcast with shuffles, eight X rows in flight
// per lane.  grid.y walks the column slices so
// a slice of X stays L2-resident while every row streams past it.
// Long rows (hub rows of T^T, popular labels of Y^T, ...): split into segments
// of SEG nonzeros, one warp per (segment, slice) writing a partial row, then
// an ordered per-row reduction of the segments -- balanced and deterministic
// (every output element is summed in a fixed order).
#include <cstdlib>

#include "common.cuh"
#include "capi_guard.cuh"
#include "cub_util.cuh"
#include "spmm.cuh"
#include "instrument.cuh"

namespace fpi {
namespace {

constexpr int WARPS = 8;       // warps per CTA
constexpr int SLICE = 64;      // output columns per warp pass (2 per lane)
#ifndef FPI_SPMM_UNROLL
#define FPI_SPMM_UNROLL 8
#endif
#ifndef FPI_SPMM_MINB
#define FPI_SPMM_MINB 3
#endif
constexpr int UNROLL = FPI_SPMM_UNROLL;  // gathered X rows in flight per lane
constexpr int64_t SEG = 512;   // nonzeros per long-row segment (rows longer than this are split)

// Column ownership inside a 64-column slice starting at c0:
//   VEC   : lane owns c0 + 2 lane, c0 + 2 lane + 1   (one 16-byte load, 512 contiguous bytes per warp)
//   scalar: lane owns c0 + lane,   c0 + 32 + lane    (two 8-byte loads, 256 contiguous bytes each)
// Lanes past column k load column 0 (always valid) and never store, so the gathers carry no
// predicates.  In VEC mode an odd k leaves the last lane's pair half outside the row: the 16-byte
// load stays inside the aligned 16-byte block that holds column k - 1 (ldx is even).
template <bool VEC>
struct Cols {
  int64_t a, b;      // owned columns
  int32_t la, lb;    // load offsets
  Cols() = default;
  __device__ __forceinline__ Cols(int64_t c0, int lane, int64_t k)
      : a(VEC ? c0 + 2 * lane : c0 + lane), b(VEC ? c0 + 2 * lane + 1 : c0 + 32 + lane) {
    la = a < k ? (int32_t)a : 0;
    lb = b < k ? (int32_t)b : 0;
  }
};

#ifndef FPI_SPMM_LOAD
#define FPI_SPMM_LOAD 0
#endif
// gather of one X row slice: 0 = ld.global.nc (L1-allocating), 1 = ld.global.cg (L2 only),
// 2 = ld.global.nc.L1::no_allocate
__device__ __forceinline__ double2 ldx2(const double* p) {
#if FPI_SPMM_LOAD == 1
  return __ldcg(reinterpret_cast<const double2*>(p));
#elif FPI_SPMM_LOAD == 2
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
#else
  return __ldg(reinterpret_cast<const double2*>(p));
#endif
}
__device__ __forceinline__ double ldx1(const double* p) {
#if FPI_SPMM_LOAD == 1
  return __ldcg(p);
#else
  return __ldg(p);
#endif
}

template <bool VEC>
__device__ __forceinline__ double2 load2(const double* __restrict__ xr, const Cols<VEC>& c) {
  if (VEC) return ldx2(xr + c.la);
  return make_double2(ldx1(xr + c.la), ldx1(xr + c.lb));
}

// acc += sum_{j in [b, e)} values[j] * X[indices[j], cols]; nonzeros fetched 32 at a time and
// broadcast with shuffles, UNROLL gathered rows in flight per lane.
template <bool VEC>
__device__ __forceinline__ void accumulate_range(int64_t b, int64_t e, const int32_t* __restrict__ indices,
                                                 const double* __restrict__ values, const double* __restrict__ X,
                                                 int64_t ldx, int64_t k, const Cols<VEC>& c, int lane,
                                                 double2& acc) {
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
    for (; j + UNROLL <= cnt; j += UNROLL) {
      double2 x[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int32_t cj = __shfl_sync(0xffffffffu, col, j + u);
        x[u] = load2<VEC>(X + (int64_t)cj * ldx, c);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const double v = __shfl_sync(0xffffffffu, val, j + u);
        acc.x = fma(v, x[u].x, acc.x);
        acc.y = fma(v, x[u].y, acc.y);
      }
    }
    if (j < cnt) {  // tail: up to UNROLL - 1 rows, still issued together
      double2 x[UNROLL - 1];
#pragma unroll
      for (int u = 0; u < UNROLL - 1; ++u) {
        const int32_t cj = __shfl_sync(0xffffffffu, col, (j + u) & 31);
        x[u] = j + u < cnt ? load2<VEC>(X + (int64_t)cj * ldx, c) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < UNROLL - 1; ++u) {
        const double v = __shfl_sync(0xffffffffu, val, (j + u) & 31);
        if (j + u < cnt) {
          acc.x = fma(v, x[u].x, acc.x);
          acc.y = fma(v, x[u].y, acc.y);
        }
      }
    }
  }
}

// NSL consecutive 64-column slices per warp (VEC layout): the nonzeros are fetched and shuffled
// once for all NSL slices, NSL 512-byte gathers per nonzero in flight.
template <int NSL>
__device__ __forceinline__ void accumulate_range_multi(int64_t b, int64_t e, const int32_t* __restrict__ indices,
                                                       const double* __restrict__ values, const double* __restrict__ X,
                                                       int64_t ldx, const Cols<true> (&c)[NSL], int lane,
                                                       double2 (&acc)[NSL]) {
  constexpr int U = (UNROLL / NSL) > 1 ? (UNROLL / NSL) : 1;
  for (int64_t base = b; base < e; base += 32) {
    const int64_t my = base + lane;
    int32_t col = 0;
    double val = 0.0;
    if (my < e) {
      col = __ldg(indices + my);
      val = __ldg(values + my);
    }
    const int cnt = (int)((e - base) < 32 ? (e - base) : 32);
    for (int j = 0; j < cnt; j += U) {
      double2 x[U][NSL];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int32_t cj = __shfl_sync(0xffffffffu, col, (j + u) & 31);
        const double* xr = X + (int64_t)cj * ldx;
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl)
          x[u][sl] = (j + u < cnt) ? ldx2(xr + c[sl].la) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double v = __shfl_sync(0xffffffffu, val, (j + u) & 31);
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) {
          acc[sl].x = fma(v, x[u][sl].x, acc[sl].x);
          acc[sl].y = fma(v, x[u][sl].y, acc[sl].y);
        }
      }
    }
  }
}

template <bool VEC>
__device__ __forceinline__ void store2(double* yr, const Cols<VEC>& c, int64_t k, double s, double beta,
                                       const double2& a) {
  if (c.a < k) yr[c.a] = beta == 0.0 ? s * a.x : s * a.x + beta * yr[c.a];
  if (c.b < k) yr[c.b] = beta == 0.0 ? s * a.y : s * a.y + beta * yr[c.b];
}

template <bool VEC>
__global__ void __launch_bounds__(WARPS * 32, 2)
    k_spmm(int64_t p, int64_t k, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
           const double* __restrict__ values, const double* __restrict__ row_scale, double alpha,
           const double* __restrict__ X, int64_t ldx, double beta, double* __restrict__ Y, int64_t ldy,
           int64_t long_thresh) {
  const int lane = threadIdx.x & 31;
  const Cols<VEC> c((int64_t)blockIdx.y * SLICE, lane, k);
  for (int64_t row = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); row < p; row += (int64_t)gridDim.x * WARPS) {
    const int64_t b = indptr[row], e = indptr[row + 1];
    if (e - b > long_thresh) continue;  // handled by the segmented path
    double2 acc = make_double2(0.0, 0.0);
    accumulate_range<VEC>(b, e, indices, values, X, ldx, k, c, lane, acc);
    const double s = row_scale ? alpha * row_scale[row] : alpha;
    store2<VEC>(Y + row * ldy, c, k, s, beta, acc);
  }
}

template <int NSL>
__global__ void __launch_bounds__(WARPS * 32, FPI_SPMM_MINB)
    k_spmm_multi(int64_t p, int64_t k, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                 const double* __restrict__ values, const double* __restrict__ row_scale, double alpha,
                 const double* __restrict__ X, int64_t ldx, double beta, double* __restrict__ Y, int64_t ldy,
                 int64_t long_thresh) {
  const int lane = threadIdx.x & 31;
  Cols<true> c[NSL];
#pragma unroll
  for (int sl = 0; sl < NSL; ++sl) c[sl] = Cols<true>(((int64_t)blockIdx.y * NSL + sl) * SLICE, lane, k);
  for (int64_t row = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); row < p; row += (int64_t)gridDim.x * WARPS) {
    const int64_t b = indptr[row], e = indptr[row + 1];
    if (e - b > long_thresh) continue;  // handled by the segmented path
    double2 acc[NSL];
#pragma unroll
    for (int sl = 0; sl < NSL; ++sl) acc[sl] = make_double2(0.0, 0.0);
    accumulate_range_multi<NSL>(b, e, indices, values, X, ldx, c, lane, acc);
    const double s = row_scale ? alpha * row_scale[row] : alpha;
#pragma unroll
    for (int sl = 0; sl < NSL; ++sl) store2<true>(Y + row * ldy, c[sl], k, s, beta, acc[sl]);
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
__global__ void __launch_bounds__(WARPS * 32, 2)
    k_spmm_segments(const int64_t* __restrict__ rows, const int64_t* __restrict__ seg_off, int64_t nl,
                    int64_t nseg_total, int64_t k, const int64_t* __restrict__ indptr,
                    const int32_t* __restrict__ indices, const double* __restrict__ values,
                    const double* __restrict__ X, int64_t ldx, double* __restrict__ P) {
  const int lane = threadIdx.x & 31;
  const Cols<VEC> c((int64_t)blockIdx.y * SLICE, lane, k);
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
    double2 acc = make_double2(0.0, 0.0);
    accumulate_range<VEC>(b, e, indices, values, X, ldx, k, c, lane, acc);
    store2<VEC>(P + sg * k, c, k, 1.0, 0.0, acc);
  }
}

template <int NSL>
__global__ void __launch_bounds__(WARPS * 32, FPI_SPMM_MINB)
    k_spmm_segments_multi(const int64_t* __restrict__ rows, const int64_t* __restrict__ seg_off, int64_t nl,
                          int64_t nseg_total, int64_t k, const int64_t* __restrict__ indptr,
                          const int32_t* __restrict__ indices, const double* __restrict__ values,
                          const double* __restrict__ X, int64_t ldx, double* __restrict__ P) {
  const int lane = threadIdx.x & 31;
  Cols<true> c[NSL];
#pragma unroll
  for (int sl = 0; sl < NSL; ++sl) c[sl] = Cols<true>(((int64_t)blockIdx.y * NSL + sl) * SLICE, lane, k);
  for (int64_t sg = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); sg < nseg_total;
       sg += (int64_t)gridDim.x * WARPS) {
    int64_t lo = 0, hi = nl - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (seg_off[mid] <= sg) lo = mid; else hi = mid - 1;
    }
    const int64_t r = rows[lo];
    const int64_t b = indptr[r] + (sg - seg_off[lo]) * SEG;
    const int64_t e0 = indptr[r + 1];
    const int64_t e = b + SEG < e0 ? b + SEG : e0;
    double2 acc[NSL];
#pragma unroll
    for (int sl = 0; sl < NSL; ++sl) acc[sl] = make_double2(0.0, 0.0);
    accumulate_range_multi<NSL>(b, e, indices, values, X, ldx, c, lane, acc);
#pragma unroll
    for (int sl = 0; sl < NSL; ++sl) store2<true>(P + sg * k, c[sl], k, 1.0, 0.0, acc[sl]);
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
  // two 64-column slices per warp (measured: tools/spmm_variants3.sh), FPI_SPMM_NSL overrides
  static const int nsl_env = getenv("FPI_SPMM_NSL") ? atoi(getenv("FPI_SPMM_NSL")) : 2;
  if (vec && nsl_env > 1) {
    const int nsl = nsl_env >= 4 ? 4 : 2;
    dim3 gm((unsigned)gx, (unsigned)((slices + nsl - 1) / nsl));
    if (nsl == 4)
      k_spmm_multi<4><<<gm, WARPS * 32, 0, s>>>(p, k, indptr, indices, values, row_scale, alpha, X, ldx, beta, Y, ldy,
                                               SEG);
    else
      k_spmm_multi<2><<<gm, WARPS * 32, 0, s>>>(p, k, indptr, indices, values, row_scale, alpha, X, ldx, beta, Y, ldy,
                                               SEG);
  } else if (vec)
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
  if (vec && nsl_env > 1) {
    dim3 g3((unsigned)gs, (unsigned)((slices + 1) / 2));
    k_spmm_segments_multi<2><<<g3, WARPS * 32, 0, s>>>(lrows, seg_off, nl, total, k, indptr, indices, values, X, ldx,
                                                       P);
  } else if (vec)
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
