// Sharded FastPI stages: one rank per GPU, the handle's communicator
// (comm.cu: NCCL over NVLink / NVSwitch) for the exchanges, everything else local.
//
// Ownership (fpi_shard_plan): the A11 diagonal blocks in contiguous block ranges balanced by
// cost -- rank i owns blocks [b_lo, b_hi), hence spoke rows [r_lo, r_hi) and spoke columns
// [c_lo, c_hi) --, plus a contiguous chunk [h_lo, h_hi) of the m2 hub rows and [hc_lo, hc_hi) of
// the n2 hub columns.  Rank i's rows of every row-indexed panel (U, T, A21, Y) are its spoke rows
// then its hub rows; its columns of every column-indexed panel (Vt, Z) are its spoke columns then
// its hub columns.
//
//   block SVD (svd.py:141-193)  own blocks only (fpi_block_svd_range); nothing exchanged: the later
//                               stages need only the owner's blocks
//   row update (pinv.py:131-171) inner rows = own kept rows of Sigma Vt11 + own A21 rows.
//                               B_i = inner_i X; G = sum B_i^T B_i (all-reduce k x k);
//                               Z = inner^T B reduced onto the owner of each spoke-column range
//                               (one ncclReduce per rank: the reduce-scatter of Y^T);
//                               Gram of Y^T = sum Z_i^T Z_i (all-reduce k x k); eigensolve
//                               replicated; V rows (= Vt columns) and U rows local
//   column update (pinv.py:174-208) inner rows = own rows of [U Sigma | T]; Z = sum M_i^T B_i
//                               (all-reduce q x k); G = X^T Z split over the ranks (all-reduce k x k);
//                               small SVD replicated; U rows local, Vt columns local
//   apply (pinv.py:72-81)       W = sum_i Y_i^T U_i (all-reduce L x r); Z rows of the own columns
//                               = V_i diag(sigma+) W^T (each rank its V-row slice)
//
// All-reduce results are bitwise identical on every rank, and everything after them is
// deterministic, so sigma and every replicated quantity agree bit for bit across ranks.
#include <algorithm>
#include <vector>

#include "capi_guard.cuh"
#include "comm.cuh"
#include "common.cuh"
#include "cub_util.cuh"
#include "gemm.cuh"
#include "inner_op.cuh"
#include "instrument.cuh"
#include "linalg.cuh"
#include "sparse.cuh"
#include "spmm.cuh"

namespace fpi {
namespace {

constexpr int PLAN_FIELDS = 10;  // b_lo b_hi r_lo r_hi c_lo c_hi h_lo h_hi hc_lo hc_hi

__global__ void k_row_cost(int64_t m, const int64_t* __restrict__ t_ptr, int64_t* __restrict__ cost) {
  FPI_GRID_STRIDE(i, m) cost[i] = 8 + (t_ptr ? t_ptr[i + 1] - t_ptr[i] : 0);
}

// block cost: its rows' cost (row-indexed work of the updates) + columns + the block SVD's h w min(h, w)
__global__ void k_block_cost(int64_t nspans, const int64_t* __restrict__ spans, const int64_t* __restrict__ rowpref,
                             int64_t* __restrict__ bc) {
  FPI_GRID_STRIDE(b, nspans) {
    const int64_t rs = spans[4 * b], hh = spans[4 * b + 1], ww = spans[4 * b + 3];
    const int64_t rows = hh > 0 ? rowpref[rs + hh - 1] - (rs > 0 ? rowpref[rs - 1] : 0) : 0;
    const int64_t mn = hh < ww ? hh : ww;
    bc[b] = rows + ww + (hh * ww / 32) * mn;
  }
}

// out[j] (j = 0..world): number of items whose inclusive prefix (minus base) is <= total * j / world
__global__ void k_split_points(int64_t n, const int64_t* __restrict__ pref, int64_t base, int world,
                               int64_t* __restrict__ out) {
  const int j = threadIdx.x;
  if (j > world) return;
  if (n == 0) {
    out[j] = 0;
    return;
  }
  const int64_t total = pref[n - 1] - base;
  if (j == world) {
    out[j] = n;
    return;
  }
  const double target = (double)total * (double)j / (double)world;
  int64_t lo = 0, hi = n;  // first index with pref - base > target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((double)(pref[mid] - base) > target) hi = mid; else lo = mid + 1;
  }
  out[j] = lo;
}

__global__ void k_plan_fields(int world, int64_t nspans, const int64_t* __restrict__ spans, int64_t m1, int64_t n1,
                              int64_t n2, const int64_t* __restrict__ bsplit, const int64_t* __restrict__ hsplit,
                              int64_t* __restrict__ out) {
  const int j = threadIdx.x;
  if (j >= world) return;
  int64_t* o = out + PLAN_FIELDS * j;
  const int64_t b0 = bsplit[j], b1 = bsplit[j + 1];
  o[0] = b0;
  o[1] = b1;
  o[2] = b0 < nspans ? spans[4 * b0] : m1;
  o[3] = b1 < nspans ? spans[4 * b1] : m1;
  o[4] = b0 < nspans ? spans[4 * b0 + 2] : n1;
  o[5] = b1 < nspans ? spans[4 * b1 + 2] : n1;
  o[6] = hsplit[j];
  o[7] = hsplit[j + 1];
  o[8] = n2 * j / world;
  o[9] = n2 * (j + 1) / world;
}

// rows [0, k) of the inner CSR: Vt11 rows scaled by sigma; rows after: A21 (pinv.py:161-163)
__global__ void k_inner_ptr(int64_t k, int64_t m2, const int64_t* __restrict__ vptr, const int64_t* __restrict__ aptr,
                            int64_t nnz_v, int64_t* __restrict__ iptr) {
  FPI_GRID_STRIDE(i, k + m2 + 1) iptr[i] = i <= k ? vptr[i] - vptr[0] : nnz_v + aptr[i - k] - aptr[0];
}
__global__ void k_inner_fill(int64_t k, const int64_t* __restrict__ vptr, const int32_t* __restrict__ vidx,
                             const double* __restrict__ vval, const double* __restrict__ sig, int64_t nnz_v,
                             int64_t nnz_a, const int32_t* __restrict__ aidx, const double* __restrict__ aval,
                             int32_t* __restrict__ iidx, double* __restrict__ ival) {
  const int64_t v0 = k ? vptr[0] : 0;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < k; r += nw) {
    const double s = sig[r];
    for (int64_t e = vptr[r] + lane; e < vptr[r + 1]; e += 32) {
      iidx[e - v0] = vidx[e];
      ival[e - v0] = s * vval[e];
    }
  }
  FPI_GRID_STRIDE(e, nnz_a) {
    iidx[nnz_v + e] = aidx[e];
    ival[nnz_v + e] = aval[e];
  }
}

__global__ void k_gather_vt_rows(int64_t q, int64_t K, const double* __restrict__ V, int64_t ldv,
                                 const int32_t* __restrict__ ord, const double* __restrict__ sv,
                                 double* __restrict__ Vt, int64_t ldvt) {
  FPI_GRID_STRIDE(e, K * q) {
    const int64_t k = e / q, j = e - k * q;
    const double d = sv ? sv[k] : 1.0;
    const double v = V[j * ldv + ord[k]];
    Vt[k * ldvt + j] = sv ? (d > 0.0 ? v / d : 0.0) : v;
  }
}

// rows [0, rows) of a CSR slice: ptr - p0, column indices - c0
__global__ void k_rebase_csr(int64_t rows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                             int64_t p0, int64_t n, int64_t c0, int64_t* __restrict__ optr,
                             int32_t* __restrict__ oidx) {
  FPI_GRID_STRIDE(i, rows + 1) optr[i] = ptr[i] - p0;
  FPI_GRID_STRIDE(e, n) oidx[e] = (int32_t)(idx[p0 + e] - c0);
}

__global__ void k_sqrt_vec(int64_t n, double* v) {
  FPI_GRID_STRIDE(i, n) v[i] = v[i] > 0.0 ? sqrt(v[i]) : 0.0;
}
__global__ void k_iota_ord(int32_t* a, int64_t n) {
  FPI_GRID_STRIDE(i, n) a[i] = (int32_t)i;
}

// per row of the local Vt slice: (max |v|, global column of the first max, signed value)
__global__ void k_canon_local(int64_t r, int64_t q, const double* __restrict__ Vt, int64_t ldvt, int64_t col0,
                              double* __restrict__ out) {
  __shared__ double bv_s[32];
  __shared__ int64_t bi_s[32];
  for (int64_t j = blockIdx.x; j < r; j += gridDim.x) {
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t c = threadIdx.x; c < q; c += blockDim.x) {
      const double a = fabs(Vt[j * ldvt + c]);
      if (a > bv) { bv = a; bi = c; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { bv_s[w] = bv; bi_s[w] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
        if (bv_s[k] > bv_s[0] || (bv_s[k] == bv_s[0] && bi_s[k] < bi_s[0])) { bv_s[0] = bv_s[k]; bi_s[0] = bi_s[k]; }
      const bool any = q > 0 && bi_s[0] != INT64_MAX;
      out[3 * j] = any ? bv_s[0] : -1.0;
      out[3 * j + 1] = any ? (double)(col0 + bi_s[0]) : 1e300;
      out[3 * j + 2] = any ? Vt[j * ldvt + bi_s[0]] : 1.0;
    }
    __syncthreads();
  }
}

// the canonical sign of every row from all ranks' candidates (largest |v|, then smallest column)
__global__ void k_canon_pick(int64_t r, int world, const double* __restrict__ all, double* __restrict__ sgn) {
  FPI_GRID_STRIDE(j, r) {
    double bv = -2.0, bi = 1e301, val = 1.0;
    for (int w = 0; w < world; ++w) {
      const double* c = all + ((int64_t)w * r + j) * 3;
      if (c[0] > bv || (c[0] == bv && c[1] < bi)) { bv = c[0]; bi = c[1]; val = c[2]; }
    }
    sgn[j] = val < 0.0 ? -1.0 : 1.0;
  }
}

__global__ void k_scale_rows_by(int64_t M, int64_t N, double* __restrict__ A, int64_t lda,
                                const double* __restrict__ s) {
  FPI_GRID_STRIDE(e, M * N) {
    const int64_t i = e / N, j = e - i * N;
    A[i * lda + j] *= s[i];
  }
}

__global__ void k_copy_cols(int64_t M, int64_t N, const double* __restrict__ A, int64_t lda, double* __restrict__ B,
                            int64_t ldb) {
  FPI_GRID_STRIDE(e, M * N) {
    const int64_t i = e / N, j = e - i * N;
    B[i * ldb + j] = A[i * lda + j];
  }
}

// local row of reordered row i: spoke rows [r_lo, r_hi) first, then hub rows [m1 + h_lo, m1 + h_hi)
__device__ __forceinline__ int64_t local_row(int64_t i, int64_t m1, int64_t r_lo, int64_t r_hi, int64_t h_lo,
                                             int64_t h_hi) {
  if (i >= r_lo && i < r_hi) return i - r_lo;
  if (i >= m1 + h_lo && i < m1 + h_hi) return (r_hi - r_lo) + (i - m1 - h_lo);
  return -1;
}

// entries of Y (original rows) whose reordered row is local: flag + (label, local row) pairs
__global__ void k_y_local(int64_t nnz, const int32_t* __restrict__ rows, const int64_t* __restrict__ row_fwd,
                          int64_t m1, int64_t r_lo, int64_t r_hi, int64_t h_lo, int64_t h_hi,
                          int32_t* __restrict__ lrow) {
  FPI_GRID_STRIDE(e, nnz) lrow[e] = (int32_t)local_row(row_fwd[rows[e]], m1, r_lo, r_hi, h_lo, h_hi);
}
struct NonNeg {
  const int32_t* v;
  __device__ bool operator()(int32_t e) const { return v[e] >= 0; }
};
__global__ void k_pick_y(int64_t cnt, const int32_t* __restrict__ picked, const int32_t* __restrict__ yidx,
                         const int32_t* __restrict__ lrow, const double* __restrict__ yval, int32_t* __restrict__ maj,
                         int32_t* __restrict__ mnr, double* __restrict__ val) {
  FPI_GRID_STRIDE(e, cnt) {
    const int32_t i = picked[e];
    maj[e] = yidx[i];
    mnr[e] = lrow[i];
    val[e] = yval[i];
  }
}

__global__ void k_scale_cols_by(int64_t M, int64_t N, double* __restrict__ A, int64_t lda,
                                const double* __restrict__ s) {
  FPI_GRID_STRIDE(e, M * N) {
    const int64_t i = e / N, j = e - i * N;
    A[i * lda + j] *= s[j];
  }
}

struct FlagNZ {
  const int32_t* f;
  __device__ bool operator()(int32_t i) const { return f[i] != 0; }
};
__global__ void k_row_nz(int64_t m, int64_t sd, const double* __restrict__ D, int32_t* __restrict__ flag) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < m; i += nw) {
    bool nz = false;
    for (int64_t c = lane; c < sd; c += 32) nz |= D[i * sd + c] != 0.0;
    nz = __any_sync(0xffffffffu, nz);
    if (lane == 0) flag[i] = nz ? 1 : 0;
  }
}
__global__ void k_gather_rows_i32(int64_t nr, int64_t k, const double* __restrict__ src, const int32_t* __restrict__ rows,
                                  double* __restrict__ dst) {
  FPI_GRID_STRIDE(e, nr * k) {
    const int64_t i = e / k, c = e - i * k;
    dst[e] = src[(int64_t)rows[i] * k + c];
  }
}

Comm& need_comm(fpi_context* h) {
  FPI_REQUIRE(h->comm != nullptr, FPI_EDOMAIN, "sharded call on a handle without a communicator");
  return *h->comm;
}

// ---------------------------------------------------------------------------------------------
// Randomized SVD (svd.py:120-138) of an inner matrix whose rows are spread over the ranks; this
// rank holds rows op (op.p local rows of q columns).  zoff (world + 1 offsets over q) assigns row
// ranges of Z = inner^T B (= columns of Y):
//   z_sharded: Z is reduced onto the owner of each range; this rank's Vt columns are its range;
//   otherwise: Z is all-reduced; Vt (rank x q) is complete on every rank (zoff only splits the
//   Gram work).
// U (op.p x rank) = this rank's rows of the left factor.
void rsvd_sharded(fpi_context* h, const InnerOp& op, int64_t p_global, int64_t rank, int64_t seed,
                  const std::vector<int64_t>& zoff, bool z_sharded, double* U, double* sigma, double* Vt,
                  fpi_svd_diag* diag) {
  Comm& c = need_comm(h);
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  const int me = c.rank, world = c.world;
  const int64_t p = op.p, q = op.q, k = 2 * rank;
  FPI_REQUIRE(p_global > k, FPI_EDOMAIN, "sharded randomized SVD needs more rows than the sketch width");
  if (diag) {
    *diag = fpi_svd_diag{};
    diag->engine = 1;
  }
  Scratch<double> X(q * k, s), B(p * k + 1, s), Zp(q * k, s), Gm(k * k, s), Linv(k * k, s);
  sketch_normal(h, seed, q, k, X, k);  // svd.py:131-132: the same sketch on every rank
  if (p > 0) {
    op.apply(h, X, k, B);   // B_i = inner_i X           (svd.py:133)
    op.applyT(h, B, k, Zp); // inner_i^T B_i             (svd.py:135's Q^T inner, before L^-T)
  } else {
    FPI_CUDA(cudaMemsetAsync(Zp.get(), 0, sizeof(double) * q * k, s));
  }
  const int64_t z0 = zoff[me], zn = zoff[me + 1] - zoff[me];
  Scratch<double> Zs;
  const double* Z = Zp.get();  // z_sharded: rows [z0, z0 + zn) only (ld k)
  if (z_sharded) {
    Zs.alloc(zn * k + 1, s);
    c.group_begin();
    for (int j = 0; j < world; ++j)
      c.reduce(Zp.get() + zoff[j] * k, j == me ? Zs.get() : Zp.get() + zoff[j] * k, (zoff[j + 1] - zoff[j]) * k, j, s);
    c.group_end();
    Z = Zs.get();
  } else {
    c.allreduce(Zp.get(), q * k, 0, s);
  }
  // rows of Z this rank's share of every Z-row product covers
  const double* Zmine = z_sharded ? Z : Z + z0 * k;
  // CholeskyQR Gram (svd.py:134): X^T Z for a tall inner, sum B_i^T B_i otherwise
  if (2 * q < p_global) {
    if (zn) gemm(h, true, false, k, k, zn, 1.0, X.get() + z0 * k, k, Zmine, k, 0.0, Gm, k);
    else FPI_CUDA(cudaMemsetAsync(Gm.get(), 0, sizeof(double) * k * k, s));
    c.allreduce(Gm.get(), k * k, 0, s);
    symmetrize(h, k, Gm, k);
  } else {
    if (p) gemm(h, true, false, k, k, p, 1.0, B, k, B, k, 0.0, Gm, k, /*sym=*/true);
    else FPI_CUDA(cudaMemsetAsync(Gm.get(), 0, sizeof(double) * k * k, s));
    c.allreduce(Gm.get(), k * k, 0, s);
  }
  fpi_svd_diag dd{};
  orth_factor(h, k, Gm, Linv, &dd);
  if (diag) {
    diag->cond_estimate = dd.cond_estimate;
    diag->cholqr_passes = dd.cholqr_passes;
  }
  B.release();
  // small SVD of Y^T = Z L^-T (svd.py:136) through the Gram of its rows, summed over the ranks
  const bool implicit = q >= k && dd.cond_estimate > 0.0 && dd.cond_estimate < 8.0;
  const int64_t mrows = z_sharded ? zn : q;  // rows of M this rank materialises
  const double* M = z_sharded ? Z : Z;
  Scratch<double> Mexp;
  if (!implicit) {
    Mexp.alloc(mrows * k + 1, s);
    if (mrows) gemm(h, false, true, mrows, k, k, 1.0, M, k, Linv, k, 0.0, Mexp, k);
    M = Mexp.get();
  }
  const double* Mmine = z_sharded ? M : M + z0 * k;
  Scratch<double> C(k * k, s), W0(k * k, s), w0(k, s);
  if (zn) gemm(h, true, false, k, k, zn, 1.0, Mmine, k, Mmine, k, 0.0, Gm, k, /*sym=*/true);
  else FPI_CUDA(cudaMemsetAsync(Gm.get(), 0, sizeof(double) * k * k, s));
  c.allreduce(Gm.get(), k * k, 0, s);
  if (implicit) {
    gemm(h, false, false, k, k, k, 1.0, Linv, k, Gm, k, 0.0, C, k);
    gemm(h, false, true, k, k, k, 1.0, C, k, Linv, k, 0.0, Gm, k);
    symmetrize(h, k, Gm, k);
  }
  const int sw0 = sym_eig(h, k, Gm, k, w0, W0, k, 60, 1e-15, true);
  double lam[2];
  FPI_CUDA(cudaMemcpyAsync(&lam[0], w0.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaMemcpyAsync(&lam[1], w0.get() + (rank - 1), sizeof(double), cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  const bool refine = !(lam[0] > 0.0) || lam[1] < 1e-6 * lam[0];
  // left vectors of Y^T: Uraw = M (R^T W)[:, :rank]  (R = L^-1 when implicit), or the refined pass
  Scratch<double> RW(k * k, s), Uraw(mrows * rank + 1, s), Vfin;
  const double* Vsel = W0.get();
  int sw1 = 0;
  if (implicit) gemm(h, true, false, k, k, k, 1.0, Linv, k, W0, k, 0.0, RW, k);
  else FPI_CUDA(cudaMemcpyAsync(RW.get(), W0.get(), sizeof(double) * k * k, cudaMemcpyDeviceToDevice, s));
  if (refine) {
    // M1 = M (R^T W0) has nearly orthogonal columns; the Jacobi solve of its Gram (summed over the
    // ranks) is relatively accurate (svd_engine.cu dense_svd_tall)
    Scratch<double> M1(mrows * k + 1, s), W1(k * k, s), w1(k, s);
    if (mrows) gemm(h, false, false, mrows, k, k, 1.0, M, k, RW, k, 0.0, M1, k);
    const double* M1mine = z_sharded ? M1.get() : M1.get() + z0 * k;
    if (zn) gemm(h, true, false, k, k, zn, 1.0, M1mine, k, M1mine, k, 0.0, Gm, k, /*sym=*/true);
    else FPI_CUDA(cudaMemsetAsync(Gm.get(), 0, sizeof(double) * k * k, s));
    c.allreduce(Gm.get(), k * k, 0, s);
    sw1 = sym_eig(h, k, Gm, k, w1, W1, k, 60, 1e-14, false);
    Vfin.alloc(k * k, s);
    gemm(h, false, false, k, k, k, 1.0, W0, k, W1, k, 0.0, Vfin, k);
    if (mrows) gemm(h, false, false, mrows, rank, k, 1.0, M1, k, W1, k, 0.0, Uraw, rank);
    Vsel = Vfin.get();
  } else {
    if (mrows) gemm(h, false, false, mrows, rank, k, 1.0, M, k, RW, k, 0.0, Uraw, rank);
  }
  // sigma = column norms of Uraw over all rows of Y^T
  Scratch<double> ss(rank, s), ss2(rank, s), sgn(rank, s);
  if (z_sharded) {
    if (zn) col_sumsq(h, zn, rank, Uraw, rank, ss);
    else FPI_CUDA(cudaMemsetAsync(ss.get(), 0, sizeof(double) * rank, s));
    c.allreduce(ss.get(), rank, 0, s);
  } else {
    col_sumsq(h, q, rank, Uraw, rank, ss);
  }
  k_sqrt_vec<<<grid_for(rank, 256, G), 256, 0, s>>>(rank, ss);
  Scratch<int32_t> ord(rank, s), ord2(rank, s);
  k_iota_ord<<<grid_for(rank, 256, G), 256, 0, s>>>(ord, rank);
  CubTemp tmp(s);
  sort_pairs(tmp, ss.get(), ss2.get(), ord.get(), ord2.get(), rank, true, 0, 64, s);
  FPI_CUDA(cudaMemcpyAsync(sigma, ss2.get(), sizeof(double) * rank, cudaMemcpyDeviceToDevice, s));
  double smin = 0.0;
  FPI_CUDA(cudaMemcpyAsync(&smin, ss2.get() + rank - 1, sizeof(double), cudaMemcpyDeviceToHost, s));
  // right vectors (of inner) = left vectors of Y^T, sorted and normalised: Vt (rank x cols)
  const int64_t vcols = z_sharded ? zn : q;
  if (vcols)
    k_gather_vt_rows<<<grid_for(rank * vcols, 256, G), 256, 0, s>>>(vcols, rank, Uraw, rank, ord2, ss2, Vt, vcols);
  FPI_LAUNCH_CHECK();
  note_launch(h, 4);
  FPI_CUDA(cudaStreamSynchronize(s));
  FPI_REQUIRE(smin > 0.0, FPI_ENUMERIC,
              "sharded randomized SVD: the inner matrix has fewer than `rank` nonzero singular values");
  // canonical signs: largest-|.| entry of each right vector positive (over all ranks' columns)
  if (z_sharded) {
    Scratch<double> loc(3 * rank, s), all(3 * rank * world, s);
    k_canon_local<<<(unsigned)std::min<int64_t>(rank, 4096), 256, 0, s>>>(rank, zn, Vt, zn, z0, loc);
    c.allgather(loc, all, 3 * rank, s);
    k_canon_pick<<<grid_for(rank, 256, G), 256, 0, s>>>(rank, world, all, sgn);
    if (zn) k_scale_rows_by<<<grid_for(rank * zn, 256, G), 256, 0, s>>>(rank, zn, Vt, zn, sgn);
    FPI_LAUNCH_CHECK();
    note_launch(h, 3);
  } else {
    canonical_signs_vt(h, rank, q, Vt, q, sgn);
  }
  // U = Q U~ = B L^-T U~ = inner (X L^-T U~)   (svd.py:137), U~ columns = Vsel[:, ord]
  Scratch<double> Uy(rank * k, s), Mx(k * rank, s);
  k_gather_vt_rows<<<grid_for(rank * k, 256, G), 256, 0, s>>>(k, rank, Vsel, k, ord2, nullptr, Uy, k);
  FPI_LAUNCH_CHECK();
  note_launch(h);
  gemm(h, true, true, k, rank, k, 1.0, Linv, k, Uy, k, 0.0, Mx, rank);
  scale_cols(h, k, rank, Mx, rank, sgn, false);
  if (p > 0) {
    Scratch<double> XM(q * rank, s);
    gemm(h, false, false, q, rank, k, 1.0, X, k, Mx, rank, 0.0, XM, rank);
    op.apply(h, XM, rank, U);
  }
  if (diag) {
    diag->eig_sweeps[0] = sw0;
    diag->eig_sweeps[1] = sw1;
  }
}

}  // namespace
}  // namespace fpi

using namespace fpi;

extern "C" {

/* Ownership plan of a sharded solve: h_out[world][10] = b_lo, b_hi, r_lo, r_hi, c_lo, c_hi, h_lo, h_hi,
 * hc_lo, hc_hi (block range, spoke rows, spoke columns, hub-row chunk within [0, m2), hub-column
 * chunk within [0, n2)).  Block ranges are contiguous and balanced by rows' work (8 + T row nnz)
 * plus each block's columns and h w min(h, w); hub rows by the same row cost; hub columns evenly. */
int fpi_shard_plan(fpi_handle h, int64_t m, int64_t m1, int64_t n1, int64_t n2, int64_t n_spans,
                   const int64_t* d_spans, const int64_t* d_t_ptr, int world, int64_t* h_out) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(world >= 1 && world <= 1024 && m >= m1, FPI_EDOMAIN, "bad shard plan arguments");
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  Scratch<int64_t> cost(m + 1, s), pref(m + 1, s), bc(n_spans + 1, s), bpref(n_spans + 1, s);
  Scratch<int64_t> bsplit(world + 1, s), hsplit(world + 1, s), out(PLAN_FIELDS * world, s);
  CubTemp tmp(s);
  if (m) {
    k_row_cost<<<grid_for(m, 256, G), 256, 0, s>>>(m, d_t_ptr, cost);
    inclusive_sum(tmp, cost.get(), pref.get(), m, s);
  }
  if (n_spans) {
    k_block_cost<<<grid_for(n_spans, 256, G), 256, 0, s>>>(n_spans, d_spans, pref, bc);
    inclusive_sum(tmp, bc.get(), bpref.get(), n_spans, s);
  }
  k_split_points<<<1, 1024, 0, s>>>(n_spans, bpref, 0, world, bsplit);
  // hub rows: prefix of the rows after m1, rebased
  const int64_t base = m1 > 0 ? host_read(pref.get() + m1 - 1, s) : 0;
  k_split_points<<<1, 1024, 0, s>>>(m - m1, pref.get() + m1, base, world, hsplit);
  k_plan_fields<<<1, 1024, 0, s>>>(world, n_spans, d_spans, m1, n1, n2, bsplit, hsplit, out);
  FPI_LAUNCH_CHECK();
  note_launch(h, 6);
  FPI_CUDA(cudaMemcpyAsync(h_out, out.get(), sizeof(int64_t) * PLAN_FIELDS * world, cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  FPI_API_END(h)
}

/* Row update (pinv.py:131-171) on this rank's rows of inner = [Sigma Vt11 ; A21]: the block factors'
 * kept rows [k_lo, k_lo + k_loc) (sigma11 and Vt11 rows, Vt11 as the global CSR), the U11 rows of
 * its spoke rows [r_lo, r_lo + r_rows) (U11 as the global CSR; their columns lie in the kept range)
 * and its A21 rows [h_lo, h_lo + m2_loc) (A21 as the global CSR).  p_global = rank11 + m2.  zoff
 * (host, world + 1): the spoke-column ranges owned by the ranks (fpi_shard_plan's c_lo / c_hi).
 * Out: U_loc ((r_rows + m2_loc) x s: spoke rows then hub rows), sigma (s, identical on every rank),
 * Vt_loc (s x (zoff[me+1] - zoff[me]): own columns).  The randomized engine only (s < thr * n1); the
 * caller replicates small, dense-engine problems. */
int fpi_row_update_shard(fpi_handle h, int64_t n1, const double* d_sigma11, const int64_t* vt_ptr,
                         const int32_t* vt_idx, const double* vt_val, int64_t k_lo, int64_t k_loc,
                         const int64_t* u_ptr, const int32_t* u_idx, const double* u_val, int64_t r_lo, int64_t r_rows,
                         const int64_t* a_ptr, const int32_t* a_idx, const double* a_val, int64_t h_lo,
                         int64_t m2_loc, int64_t p_global, int64_t s_rank, double thr, int64_t seed,
                         const int64_t* h_zoff, double* d_U, double* d_sigma, double* d_Vt) {
  FPI_API_BEGIN(h)
  Comm& c = need_comm(h);
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  FPI_REQUIRE(s_rank >= 1 && (double)s_rank < thr * (double)n1, FPI_EDOMAIN,
              "sharded row update: the randomized engine only (s < thr * n1)");
  std::vector<int64_t> zoff(h_zoff, h_zoff + c.world + 1);
  const int64_t p = k_loc + m2_loc;
  if (k_loc) vt_ptr += k_lo;
  if (m2_loc) a_ptr += h_lo;
  const int64_t nnz_v = k_loc ? host_read(vt_ptr + k_loc, s) - host_read(vt_ptr, s) : 0;
  const int64_t nnz_a = m2_loc ? host_read(a_ptr + m2_loc, s) - host_read(a_ptr, s) : 0;
  const int64_t nnz = nnz_v + nnz_a;
  Scratch<int64_t> iptr(p + 1, s), itptr(n1 + 1, s), zero(1, s);
  Scratch<int32_t> iidx(nnz + 1, s), itidx(nnz + 1, s);
  Scratch<double> ival(nnz + 1, s), itval(nnz + 1, s);
  FPI_CUDA(cudaMemsetAsync(zero.get(), 0, sizeof(int64_t), s));
  k_inner_ptr<<<grid_for(p + 1, 256, G), 256, 0, s>>>(k_loc, m2_loc, k_loc ? vt_ptr : zero.get(),
                                                      m2_loc ? a_ptr : zero.get(), nnz_v, iptr);
  const int64_t a0 = m2_loc ? host_read(a_ptr, s) : 0;
  k_inner_fill<<<grid_for(k_loc * 32 + nnz_a, 256, G), 256, 0, s>>>(k_loc, k_loc ? vt_ptr : zero.get(), vt_idx, vt_val,
                                                                   d_sigma11 + k_lo, nnz_v, nnz_a, a_idx + a0,
                                                                   a_val + a0,
                                                                   iidx, ival);
  FPI_LAUNCH_CHECK();
  note_launch(h, 2);
  csr_transpose(h, p, n1, nnz, iptr, iidx, ival, itptr, itidx, itval);
  InnerOp op;
  op.p = p;
  op.q = n1;
  op.s_nnz = nnz;
  op.s_ptr = iptr;
  op.s_idx = iidx;
  op.s_val = ival;
  op.st_ptr = itptr;
  op.st_idx = itidx;
  op.st_val = itval;
  Scratch<double> Ui(p * s_rank + 1, s);
  rsvd_sharded(h, op, p_global, s_rank, seed, zoff, /*z_sharded=*/true, Ui, d_sigma, d_Vt, &h->diag);
  // lift: U = [U11 Ui[:k_loc] ; Ui[k_loc:]]   (pinv.py:168-170), this rank's rows: the U11 rows
  // [r_lo, r_lo + r_rows) as a local CSR with column indices rebased to k_lo
  if (r_rows) {
    const int64_t u0 = host_read(u_ptr + r_lo, s), u1 = host_read(u_ptr + r_lo + r_rows, s);
    if (k_loc && u1 > u0) {
      Scratch<int64_t> lptr(r_rows + 1, s);
      Scratch<int32_t> lidx(u1 - u0, s);
      k_rebase_csr<<<grid_for(std::max<int64_t>(r_rows + 1, u1 - u0), 256, G), 256, 0, s>>>(
          r_rows, u_ptr + r_lo, u_idx, u0, u1 - u0, k_lo, lptr, lidx);
      FPI_LAUNCH_CHECK();
      note_launch(h);
      const int64_t ldp = (s_rank + 1) & ~(int64_t)1;
      Scratch<double> Up(k_loc * ldp, s);
      FPI_CUDA(cudaMemcpy2DAsync(Up.get(), ldp * sizeof(double), Ui.get(), s_rank * sizeof(double),
                                 s_rank * sizeof(double), k_loc, cudaMemcpyDeviceToDevice, s));
      spmm(h, r_rows, k_loc, s_rank, lptr, lidx, u_val + u0, nullptr, 1.0, Up, ldp, 0.0, d_U, s_rank);
    } else {
      FPI_CUDA(cudaMemsetAsync(d_U, 0, sizeof(double) * r_rows * s_rank, s));
    }
  }
  if (m2_loc)
    FPI_CUDA(cudaMemcpyAsync(d_U + r_rows * s_rank, Ui.get() + k_loc * s_rank, sizeof(double) * m2_loc * s_rank,
                             cudaMemcpyDeviceToDevice, s));
  FPI_API_END(h)
}

/* Column update (pinv.py:174-208) on this rank's m_loc rows of inner = [U Sigma | T]: U_loc
 * (m_loc x s_prev), sigma_prev, T_loc (m_loc x n2 CSR) and its transpose (n2 x m_loc), this rank's
 * columns of the previous Vt (s_prev x nc_loc, its spoke columns) and its hub-column chunk
 * [hc_lo, hc_hi).  m_global = m.  Out: U_out (m_loc x r), sigma (r, identical on every rank),
 * Vt_out (r x (nc_loc + hc_hi - hc_lo)): [Vt~[:, :s] Vt_prev_loc | Vt~[:, s + hc_lo : s + hc_hi]]. */
int fpi_column_update_shard(fpi_handle h, int64_t m_loc, int64_t s_prev, const double* d_U_prev,
                            const double* d_sigma_prev, const double* d_Vt_prev, int64_t nc_loc, int64_t n2,
                            const int64_t* t_ptr, const int32_t* t_idx, const double* t_val, const int64_t* tt_ptr,
                            const int32_t* tt_idx, const double* tt_val, int64_t m_global, int64_t hc_lo,
                            int64_t hc_hi, int64_t r, double thr, int64_t seed, double* d_U, double* d_sigma,
                            double* d_Vt) {
  FPI_API_BEGIN(h)
  Comm& c = need_comm(h);
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  const int64_t q = s_prev + n2;
  FPI_REQUIRE(r >= 1 && (double)r < thr * (double)q, FPI_EDOMAIN,
              "sharded column update: the randomized engine only (r < thr * (s + n2))");
  std::vector<int64_t> zoff(c.world + 1);
  for (int j = 0; j <= c.world; ++j) zoff[j] = q * j / c.world;
  InnerOp op;
  op.p = m_loc;
  op.q = q;
  op.D = s_prev ? d_U_prev : nullptr;
  op.ldd = s_prev;
  op.sd = s_prev;
  op.dscale = d_sigma_prev;
  op.s_ptr = t_ptr;
  op.s_idx = t_idx;
  op.s_val = t_val;
  op.st_ptr = tt_ptr;
  op.st_idx = tt_idx;
  op.st_val = tt_val;
  op.s_nnz = (n2 && m_loc) ? host_read(t_ptr + m_loc, s) : 0;
  // rows of U_prev that are zero (spoke rows of column-free blocks) skipped in the dense products
  Scratch<int32_t> flag, ids, nzl, cntd;
  Scratch<double> Dnz;
  if (s_prev > 0 && m_loc > 0) {
    flag.alloc(m_loc, s);
    ids.alloc(m_loc, s);
    nzl.alloc(m_loc, s);
    cntd.alloc(1, s);
    k_row_nz<<<grid_for(m_loc * 32, 256, G), 256, 0, s>>>(m_loc, s_prev, d_U_prev, flag);
    k_iota_ord<<<grid_for(m_loc, 256, G), 256, 0, s>>>(ids, m_loc);
    CubTemp tmp(s);
    select_if(tmp, ids.get(), nzl.get(), cntd.get(), m_loc, FlagNZ{flag.get()}, s);
    const int64_t nzr = host_read(cntd.get(), s);
    if (nzr < (m_loc * 6) / 10) {
      Dnz.alloc(nzr * s_prev + 1, s);
      if (nzr) k_gather_rows_i32<<<grid_for(nzr * s_prev, 256, G), 256, 0, s>>>(nzr, s_prev, d_U_prev, nzl, Dnz);
      FPI_LAUNCH_CHECK();
      op.nzr = nzr;
      op.nz_rows = nzl.get();
      op.Dnz = Dnz.get();
    }
  }
  // this rank's rows of T: their heavy rows x heavy columns rectangle on the tensor pipe (sparse_core.cu)
  SparseCore core;
  if (n2 > 0 && m_loc > 0) {
    build_sparse_core(h, m_loc, n2, op.s_nnz, t_ptr, t_idx, t_val, tt_ptr, tt_idx, tt_val, core);
    if (core.use) op.core = &core;
  }
  Scratch<double> Vti(r * q, s);
  rsvd_sharded(h, op, m_global, r, seed, zoff, /*z_sharded=*/false, d_U, d_sigma, Vti, &h->diag);
  // lift (pinv.py:205-207) on this rank's columns
  const int64_t nh = hc_hi - hc_lo, w = nc_loc + nh;
  if (nc_loc) {
    if (s_prev) gemm(h, false, false, r, nc_loc, s_prev, 1.0, Vti, q, d_Vt_prev, nc_loc, 0.0, d_Vt, w);
    else FPI_CUDA(cudaMemset2DAsync(d_Vt, w * sizeof(double), 0, nc_loc * sizeof(double), r, s));
  }
  if (nh) {
    k_copy_cols<<<grid_for(r * nh, 256, G), 256, 0, s>>>(r, nh, Vti.get() + s_prev + hc_lo, q, d_Vt + nc_loc, w);
    FPI_LAUNCH_CHECK();
    note_launch(h);
  }
  FPI_API_END(h)
}

/* Z rows of this rank's columns (pinv.py:72-81): W = sum over ranks of Y_i^T U_loc (all-reduce,
 * L x r), then Z_loc (n_loc x L) = Vt_loc^T diag(sigma+) W^T.  Y: m x L CSR in original row order;
 * row_fwd maps original rows to reordered ones; this rank's rows are [r_lo, r_hi) then
 * [m1 + h_lo, m1 + h_hi) (U_loc's row order).  Z_loc rows follow Vt_loc's columns. */
int fpi_pinv_apply_shard(fpi_handle h, int64_t m, int64_t m1, int64_t r_lo, int64_t r_hi, int64_t h_lo,
                         int64_t h_hi, int64_t r, const double* d_U_loc, const double* d_sdag, const double* d_Vt_loc,
                         int64_t n_loc, const int64_t* d_row_fwd, int64_t L, int64_t nnz, const int64_t* y_ptr,
                         const int32_t* y_idx, const double* y_val, double* d_Z_loc) {
  FPI_API_BEGIN(h)
  Comm& c = need_comm(h);
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  if (L == 0) return FPI_OK;
  const int64_t m_loc = (r_hi - r_lo) + (h_hi - h_lo);
  Scratch<double> W(L * r + 1, s);
  FPI_CUDA(cudaMemsetAsync(W.get(), 0, sizeof(double) * L * r, s));
  if (nnz > 0 && m_loc > 0 && r > 0) {
    CubTemp tmp(s);
    Scratch<int32_t> rows(nnz, s), lrow(nnz, s), ids(nnz, s), picked(nnz, s);
    Scratch<int> dcnt(1, s);
    expand_rows(h, m, y_ptr, rows);
    k_y_local<<<grid_for(nnz, 256, G), 256, 0, s>>>(nnz, rows, d_row_fwd, m1, r_lo, r_hi, h_lo, h_hi, lrow);
    k_iota_ord<<<grid_for(nnz, 256, G), 256, 0, s>>>(ids, nnz);
    select_if(tmp, ids.get(), picked.get(), dcnt.get(), nnz, NonNeg{lrow.get()}, s);
    const int64_t cnt = host_read(dcnt.get(), s);
    if (cnt) {
      Scratch<int32_t> maj(cnt, s), mnr(cnt, s);
      Scratch<double> val(cnt, s);
      k_pick_y<<<grid_for(cnt, 256, G), 256, 0, s>>>(cnt, picked, y_idx, lrow, y_val, maj, mnr, val);
      Scratch<int64_t> yt_ptr(L + 1, s);
      Scratch<int32_t> yt_idx(cnt, s);
      Scratch<double> yt_val(cnt, s);
      build_csr(h, tmp, cnt, maj, mnr, val, L, m_loc, yt_ptr, yt_idx, yt_val);
      spmm(h, L, m_loc, r, yt_ptr, yt_idx, yt_val, nullptr, 1.0, d_U_loc, r, 0.0, W, r);  // W = Y_i^T U_i
    }
    FPI_LAUNCH_CHECK();
    note_launch(h, 3);
  }
  c.allreduce(W.get(), L * r, 0, s);
  if (n_loc && r) {
    k_scale_cols_by<<<grid_for(L * r, 256, G), 256, 0, s>>>(L, r, W, r, d_sdag);
    FPI_LAUNCH_CHECK();
    note_launch(h);
    gemm(h, true, true, n_loc, L, r, 1.0, d_Vt_loc, n_loc, W, r, 0.0, d_Z_loc, L);  // V_loc diag(s+) W^T
  } else if (n_loc) {
    FPI_CUDA(cudaMemsetAsync(d_Z_loc, 0, sizeof(double) * n_loc * L, s));
  }
  FPI_API_END(h)
}

}  // extern "C"
