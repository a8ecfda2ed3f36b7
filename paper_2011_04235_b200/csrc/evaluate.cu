// Precision@k of the regression harness (regression.py:89-124) on the GPU: for
// every row of a dense score block, the top-kmax labels in the reference's order
// (score descending, ties by ascending label index -- np.argsort(-s,
// kind="stable")) and whether each is a positive of that row's label set.
//
// One warp per row.  Pass j selects the best label strictly after pass j-1's
// pick in that total order (no marking, so any kmax works); lanes scan the
// row with stride 32 and the warp reduces (score, index) pairs.  A hit is a
// binary search in the row's sorted label CSR.  The output is the 0/1 hit
// matrix (rows x kmax, uint8), from which the host forms the reference's
// per-chunk sums hits[:, :k].sum() / k with the same chunk boundaries.
#include "common.cuh"
#include "capi_guard.cuh"

namespace fpi {
namespace {

// a precedes b in the reference's order
__device__ __forceinline__ bool before(double sa, int64_t ia, double sb, int64_t ib) {
  return sa > sb || (sa == sb && ia < ib);
}

__global__ void k_topk_hits(int64_t rows, int64_t L, const double* __restrict__ S, int64_t lds,
                            const int64_t* __restrict__ lab_ptr, const int32_t* __restrict__ lab_idx, int kmax,
                            uint8_t* __restrict__ hits) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const double* s = S + r * lds;
    const int64_t b = lab_ptr[r], e = lab_ptr[r + 1];
    double ps = INFINITY;  // previous pick (none yet): everything is after (+inf, -1)
    int64_t pi = -1;
    for (int j = 0; j < kmax; ++j) {
      double bs = -INFINITY;
      int64_t bi = INT64_MAX;
      for (int64_t c = lane; c < L; c += 32) {
        const double v = s[c];
        if (before(ps, pi, v, c) && before(v, c, bs, bi)) { bs = v; bi = c; }
      }
      for (int o = 16; o; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (before(os, oi, bs, bi)) { bs = os; bi = oi; }
      }
      if (bi == INT64_MAX) break;  // fewer than kmax labels (cannot happen: kmax <= L)
      if (lane == 0) {
        int64_t lo = b, hi = e;  // labels of the row are sorted ascending
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (lab_idx[mid] < bi) lo = mid + 1; else hi = mid;
        }
        hits[r * kmax + j] = (lo < e && lab_idx[lo] == bi) ? 1 : 0;
      }
      ps = bs;
      pi = bi;
    }
  }
}

}  // namespace
}  // namespace fpi

extern "C" int fpi_topk_hits(fpi_handle h, int64_t rows, int64_t L, const double* d_S, int64_t lds,
                             const int64_t* d_lab_ptr, const int32_t* d_lab_idx, int32_t kmax, uint8_t* d_hits) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(kmax >= 1 && kmax <= L, FPI_EDOMAIN,
              "k=" + std::to_string(kmax) + " must be in [1, " + std::to_string(L) + "]");
  if (rows > 0) {
    const unsigned G = fpi::grid_for(rows * 32, 256, (int64_t)h->num_sms * 16);
    fpi::k_topk_hits<<<G, 256, 0, h->stream>>>(rows, L, d_S, lds, d_lab_ptr, d_lab_idx, kmax, d_hits);
    FPI_LAUNCH_CHECK();
    fpi::note_launch(h);
  }
  FPI_API_END(h)
}
