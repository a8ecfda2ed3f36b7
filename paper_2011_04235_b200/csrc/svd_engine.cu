// SVD engines and the FastPI stages built on them.
//
//  dense_svd        svd.py:86-117 (dense_svd + truncate).  Exact SVD of a dense
//                   p x q panel via the Gram matrix of its short side, refined
//                   once: G = M^T M -> eig -> M1 = M W0 (columns now nearly
//                   orthogonal) -> G1 = M1^T M1 -> eig (converges in a couple of
//                   Jacobi sweeps, relatively accurate) -> sigma = ||M1 w1_j||.
//  randomized_svd   svd.py:120-138.  X = numpy-exact sketch; B = inner X;
//                   CholeskyQR of B without forming Q (Q = B L^-T):
//                   Y^T = (inner^T B) L^-T; SVD of the q x 2r panel Y^T;
//                   U = B (L^-T U~).  An eigen-based orthonormalisation
//                   replaces Cholesky when B^T B is not numerically PD.
//  row_update       pinv.py:131-171  (inner [diag(s) Vt11 ; A21] as one CSR)
//  column_update    pinv.py:174-208  (inner [U diag(s) | T], dense + CSR)
//  pinv_assemble    pinv.py:211-231  (cutoff, sigma^+)
//  unfold           pinv.py:271-275  (+ the V / Ut transposes of pinv.py:226-228)
//  pinv_apply       pinv.py:72-81    (Z = V diag(s+) U^T Y, Y sparse or dense)
#include <cmath>
#include <vector>

#include "common.cuh"
#include "capi_guard.cuh"
#include "cub_util.cuh"
#include "gemm.cuh"
#include "linalg.cuh"
#include "instrument.cuh"
#include "sparse.cuh"
#include "spmm.cuh"
#include "svd_engine.cuh"
#include "gram_route.cuh"
#include "inner_op.cuh"

namespace fpi {


namespace {

// A <- (A + A^T) / 2 (upper and lower from the same pair of reads)
__global__ void k_symmetrize(int64_t n, double* A, int64_t lda) {
  FPI_GRID_STRIDE(e, n * n) {
    const int64_t i = e / n, j = e - i * n;
    if (j <= i) continue;
    const double v = 0.5 * (A[i * lda + j] + A[j * lda + i]);
    A[i * lda + j] = v;
    A[j * lda + i] = v;
  }
}

__global__ void k_sqrt_clamp(int64_t n, double* v) {
  FPI_GRID_STRIDE(i, n) v[i] = v[i] > 0.0 ? sqrt(v[i]) : 0.0;
}

__global__ void k_copy2d(int64_t M, int64_t N, const double* __restrict__ A, int64_t lda, double* __restrict__ B,
                         int64_t ldb) {
  FPI_GRID_STRIDE(e, M * N) {
    int64_t i = e / N, j = e - i * N;
    B[i * ldb + j] = A[i * lda + j];
  }
}

// cols of A (M x N) selected by ord[0..K) and divided by s[k]  -> B (M x K)
// B[:, k] = sign[k] A[:, ord[k]] / s[k] (0 where s[k] == 0): sorted, normalised and sign-fixed left
// vectors in one pass (sign may be null)
__global__ void k_gather_cols_div(int64_t M, int64_t K, const double* __restrict__ A, int64_t lda,
                                  const int32_t* __restrict__ ord, const double* __restrict__ s,
                                  const double* __restrict__ sign, double* __restrict__ B, int64_t ldb) {
  FPI_GRID_STRIDE(e, M * K) {
    int64_t i = e / K, k = e - i * K;
    double d = s[k];
    const double v = d > 0.0 ? A[i * lda + ord[k]] / d : 0.0;
    B[i * ldb + k] = sign ? sign[k] * v : v;
  }
}

// Vt[k][j] = V[j][ord[k]]   (V is q x q, Vt is K x q)
__global__ void k_gather_vt(int64_t q, int64_t K, const double* __restrict__ V, int64_t ldv,
                            const int32_t* __restrict__ ord, double* __restrict__ Vt, int64_t ldvt) {
  FPI_GRID_STRIDE(e, K * q) {
    int64_t k = e / q, j = e - k * q;
    Vt[k * ldvt + j] = V[j * ldv + ord[k]];
  }
}

// Vt[k][j] = V[j][ord[k]] / s[k]   (0 where s[k] == 0)
__global__ void k_gather_vt_div(int64_t q, int64_t K, const double* __restrict__ V, int64_t ldv,
                                const int32_t* __restrict__ ord, const double* __restrict__ sv,
                                double* __restrict__ Vt, int64_t ldvt) {
  FPI_GRID_STRIDE(e, K * q) {
    int64_t k = e / q, j = e - k * q;
    const double d = sv[k];
    Vt[k * ldvt + j] = d > 0.0 ? V[j * ldv + ord[k]] / d : 0.0;
  }
}

__global__ void k_iota32(int32_t* a, int64_t n) {
  FPI_GRID_STRIDE(i, n) a[i] = (int32_t)i;
}

// The finish of many small dense SVDs at once (dense_svd_batched), one CTA per panel: sigma =
// column norms of Uraw = M W[:, :r], sorted descending (stable: ties keep index order), Vt = the
// matching eigenvector columns with the canonical sign (largest-|.| entry positive, first index on
// ties), U = sign * Uraw[:, ord] / sigma; zero_flag[i] = 1 when a sigma is at rounding level (the
// caller completes those left vectors).  Same results as the per-panel kernel sequence.
struct PanelDesc {
  int64_t p, q, r;
  const double* Uraw;  // p x r
  const double* W;     // q x q eigenvectors (columns)
  double* U;           // p x r
  double* sigma;       // r
  double* Vt;          // r x q
};

__global__ void __launch_bounds__(256) k_panel_finish(const PanelDesc* __restrict__ desc, int nb,
                                                      int* __restrict__ zero_flag) {
  extern __shared__ double psm[];
  __shared__ double rbv[8];
  __shared__ int64_t rbi[8];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = blockIdx.x; i < nb; i += gridDim.x) {
    const PanelDesc P = desc[i];
    const int64_t p = P.p, q = P.q, r = P.r;
    double* ss = psm;
    double* ssd = psm + r;
    double* sgn = psm + 2 * r;
    int* ord = reinterpret_cast<int*>(psm + 3 * r);
    for (int64_t j = tid; j < r; j += blockDim.x) {
      double a = 0.0;
      for (int64_t row = 0; row < p; ++row) {
        const double v = P.Uraw[row * r + j];
        a = fma(v, v, a);
      }
      ss[j] = a > 0.0 ? sqrt(a) : 0.0;
    }
    __syncthreads();
    for (int64_t j = tid; j < r; j += blockDim.x) {
      const double v = ss[j];
      int64_t rk = 0;
      for (int64_t l = 0; l < r; ++l) rk += (ss[l] > v) || (ss[l] == v && l < j);
      ord[rk] = (int)j;
      ssd[rk] = v;
    }
    __syncthreads();
    for (int64_t k = tid; k < r; k += blockDim.x) P.sigma[k] = ssd[k];
    for (int64_t k = 0; k < r; ++k) {
      const int c = ord[k];
      double bv = -1.0;
      int64_t bi = 0;
      for (int64_t jj = tid; jj < q; jj += blockDim.x) {
        const double a = fabs(P.W[jj * q + c]);
        if (a > bv) { bv = a; bi = jj; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { rbv[wid] = bv; rbi[wid] = bi; }
      __syncthreads();
      if (tid == 0) {
        for (int w2 = 1; w2 < (int)(blockDim.x >> 5); ++w2)
          if (rbv[w2] > rbv[0] || (rbv[w2] == rbv[0] && rbi[w2] < rbi[0])) { rbv[0] = rbv[w2]; rbi[0] = rbi[w2]; }
        sgn[k] = (q > 0 && P.W[rbi[0] * q + c] < 0.0) ? -1.0 : 1.0;
      }
      __syncthreads();
      const double sk = sgn[k];
      for (int64_t jj = tid; jj < q; jj += blockDim.x) P.Vt[k * q + jj] = sk * P.W[jj * q + c];
    }
    __syncthreads();
    for (int64_t e = tid; e < p * r; e += blockDim.x) {
      const int64_t row = e / r, k = e - row * r;
      const double d = ssd[k];
      const double v = d > 0.0 ? P.Uraw[row * r + ord[k]] / d : 0.0;
      P.U[row * r + k] = sgn[k] * v;
    }
    if (tid == 0) {
      const double tol = 2.220446049250313e-16 * (ssd[0] > 0.0 ? ssd[0] : 1.0) * (double)(p > r ? p : r);
      int z = 0;
      for (int64_t k = 0; k < r; ++k) z |= !(ssd[k] > tol);
      zero_flag[i] = z;
    }
    __syncthreads();
  }
}

// lam[2 i] = w_i[0], lam[2 i + 1] = w_i[r_i - 1] (the wide-spectrum test of every panel at once)
__global__ void k_lam_pairs(int nb, const double* const* __restrict__ w, const int64_t* __restrict__ r,
                            double* __restrict__ lam) {
  FPI_GRID_STRIDE(i, nb) {
    lam[2 * i] = w[i][0];
    lam[2 * i + 1] = w[i][r[i] - 1];
  }
}

// rows [0, rank11) of the inner CSR: Vt11 rows scaled by sigma; rows after: A21
__global__ void k_inner_rows(int64_t rank11, int64_t m2, const int64_t* __restrict__ vptr,
                             const int64_t* __restrict__ aptr, int64_t nnz_v, int64_t* __restrict__ iptr) {
  FPI_GRID_STRIDE(i, rank11 + m2 + 1) {
    iptr[i] = i <= rank11 ? vptr[i] : nnz_v + aptr[i - rank11];
  }
}

__global__ void k_inner_vals(int64_t rank11, const int64_t* __restrict__ vptr, const int32_t* __restrict__ vidx,
                             const double* __restrict__ vval, const double* __restrict__ sig, int64_t nnz_v,
                             int64_t nnz_a, const int32_t* __restrict__ aidx, const double* __restrict__ aval,
                             int32_t* __restrict__ iidx, double* __restrict__ ival) {
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = warp; k < rank11; k += nw) {
    double s = sig[k];
    for (int64_t p = vptr[k] + lane; p < vptr[k + 1]; p += 32) {
      iidx[p] = vidx[p];
      ival[p] = s * vval[p];
    }
  }
  FPI_GRID_STRIDE(e, nnz_a) {
    iidx[nnz_v + e] = aidx[e];
    ival[nnz_v + e] = aval[e];
  }
}

// dense copy of a CSR (rows x cols) into D (ld), D pre-zeroed
__global__ void k_csr_to_dense(int64_t rows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                               const double* __restrict__ val, double* __restrict__ D, int64_t ld, int64_t col0) {
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nw)
    for (int64_t p = ptr[r] + lane; p < ptr[r + 1]; p += 32) D[r * ld + col0 + idx[p]] = val[p];
}

// 1 if row i of D (m x s) has a nonzero entry
__global__ void k_row_nonzero(int64_t m, int64_t sd, const double* __restrict__ D, int64_t ldd,
                              int32_t* __restrict__ flag) {
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < m; r += nw) {
    bool nz = false;
    for (int64_t c = lane; c < sd; c += 32) nz |= D[r * ldd + c] != 0.0;
    nz = __any_sync(0xffffffffu, nz);
    if (lane == 0) flag[r] = nz ? 1 : 0;
  }
}

struct FlagSet {
  const int32_t* f;
  __device__ bool operator()(int32_t i) const { return f[i] != 0; }
};

__global__ void k_gather_rows32(int64_t nr, int64_t k, const double* __restrict__ src, int64_t lds,
                                const int32_t* __restrict__ rows, double* __restrict__ dst, int64_t ldd) {
  FPI_GRID_STRIDE(e, nr * k) {
    const int64_t i = e / k, c = e - i * k;
    dst[i * ldd + c] = src[(int64_t)rows[i] * lds + c];
  }
}

__global__ void k_scatter_add_rows32(int64_t nr, int64_t k, const double* __restrict__ src, int64_t lds,
                                     const int32_t* __restrict__ rows, double* __restrict__ dst, int64_t ldd) {
  FPI_GRID_STRIDE(e, nr * k) {
    const int64_t i = e / k, c = e - i * k;
    dst[(int64_t)rows[i] * ldd + c] += src[i * lds + c];
  }
}

__global__ void k_iota_i32(int32_t* a, int64_t n) {
  FPI_GRID_STRIDE(i, n) a[i] = (int32_t)i;
}

__global__ void k_fill(int64_t n, double* a, double v) {
  FPI_GRID_STRIDE(i, n) a[i] = v;
}

__global__ void k_pinv(int64_t r, const double* __restrict__ sigma, double cutoff, int64_t maxpq,
                       double* __restrict__ sdag, double* __restrict__ tol_out, int* __restrict__ all_filtered) {
  if (blockIdx.x != 0) return;
  const double smax = r ? sigma[0] : 0.0;
  const double tol = cutoff * smax * (double)maxpq;  // pinv.py:217-218
  __shared__ int any_keep;
  if (threadIdx.x == 0) any_keep = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < r; i += blockDim.x) {
    const bool keep = sigma[i] > tol;
    sdag[i] = keep ? 1.0 / sigma[i] : 0.0;
    if (keep) any_keep = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *tol_out = tol;
    *all_filtered = (r > 0 && !any_keep) ? 1 : 0;
  }
}

// Ut[k][i] = U[idx[i]][k]    (U: m x r row-major; Ut: r x m)
__global__ void k_gather_rows_T(int64_t m, int64_t r, const double* __restrict__ U, int64_t ldu,
                                const int64_t* __restrict__ idx, double* __restrict__ Ut, int64_t ldt) {
  __shared__ double t[32][33];
  for (int64_t by = blockIdx.y; by * 32 < m; by += gridDim.y)
    for (int64_t bx = blockIdx.x; bx * 32 < r; bx += gridDim.x) {
      for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        int64_t row = by * 32 + i, c = bx * 32 + threadIdx.x;
        t[i][threadIdx.x] = (row < m && c < r) ? U[idx[row] * ldu + c] : 0.0;
      }
      __syncthreads();
      for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        int64_t k = bx * 32 + i, c = by * 32 + threadIdx.x;
        if (k < r && c < m) Ut[k * ldt + c] = t[threadIdx.x][i];
      }
      __syncthreads();
    }
}

// V[j][k] = Vt[k][idx[j]]     (Vt: r x n; V: n x r)
__global__ void k_gather_cols_T(int64_t n, int64_t r, const double* __restrict__ Vt, int64_t ldvt,
                                const int64_t* __restrict__ idx, double* __restrict__ V, int64_t ldv) {
  FPI_GRID_STRIDE(e, n * r) {
    int64_t j = e / r, k = e - j * r;
    V[j * ldv + k] = Vt[k * ldvt + idx[j]];
  }
}

// dst[j][:] = src[idx[j]][:]

// dst[idx[i]][:] = src[i][:]
__global__ void k_scatter_rows(int64_t m, int64_t L, const double* __restrict__ src, int64_t lds,
                               const int64_t* __restrict__ idx, double* __restrict__ dst, int64_t ldd) {
  FPI_GRID_STRIDE(e, m * L) {
    int64_t i = e / L, l = e - i * L;
    dst[idx[i] * ldd + l] = src[i * lds + l];
  }
}

__global__ void k_remap_rows_i32(int64_t nnz, const int32_t* __restrict__ rows, const int64_t* __restrict__ fwd,
                                 int32_t* __restrict__ out) {
  FPI_GRID_STRIDE(e, nnz) out[e] = (int32_t)fwd[rows[e]];
}

__global__ void k_rows_in_range(int64_t nnz, const int32_t* __restrict__ rr, int64_t r0, int64_t len,
                                int32_t* __restrict__ flag) {
  FPI_GRID_STRIDE(e, nnz) flag[e] = (rr[e] >= r0 && rr[e] < r0 + len) ? 1 : 0;
}

__global__ void k_gather_triplets(int64_t cnt, const int32_t* __restrict__ picked, const int32_t* __restrict__ major,
                                  const int32_t* __restrict__ minor, const double* __restrict__ val, int64_t r0,
                                  int32_t* __restrict__ omaj, int32_t* __restrict__ omin, double* __restrict__ oval) {
  FPI_GRID_STRIDE(e, cnt) {
    const int32_t i = picked[e];
    omaj[e] = major[i];
    omin[e] = (int32_t)(minor[i] - r0);
    oval[e] = val[i];
  }
}

// max / min |L_ii| (CholeskyQR condition estimate), one block
__global__ void k_diag_ratio(int64_t n, const double* __restrict__ L, int64_t ld, double* out) {
  __shared__ double smx[256], smn[256];
  double mx = 0.0, mn = 1e308;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = fabs(L[i * ld + i]);
    mx = fmax(mx, d);
    mn = fmin(mn, d);
  }
  smx[threadIdx.x] = mx;
  smn[threadIdx.x] = mn;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) {
      smx[threadIdx.x] = fmax(smx[threadIdx.x], smx[threadIdx.x + o]);
      smn[threadIdx.x] = fmin(smn[threadIdx.x], smn[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = smn[0] > 0 ? smx[0] / smn[0] : 1e308;
}

// Linv <- diag(lambda^-1/2) W^T over kept eigenpairs (others zero)
__global__ void k_eig_orth(int64_t k, const double* __restrict__ w, const double* __restrict__ W, double tolrel,
                           double* __restrict__ Linv) {
  FPI_GRID_STRIDE(e, k * k) {
    int64_t i = e / k, j = e - i * k;
    double lam = w[i], lmax = w[0];
    Linv[i * k + j] = (lam > tolrel * lmax && lam > 0.0) ? W[j * k + i] / sqrt(lam) : 0.0;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// dense SVD of a tall panel (p >= q): the top `rank` triplets.
// With R (q x q) the panel is the implicit product M R^T: its Gram is R (M^T M) R^T and every
// product with it goes through the small R first, so the p x q product is never formed (the
// randomized SVD's Y^T = Z L^-T, svd.py:135).
static void dense_svd_tall(fpi_context* h, int64_t p, int64_t q, const double* M, int64_t ldm, int64_t rank,
                           double* U, double* sigma, double* Vt, fpi_svd_diag* diag, const double* R = nullptr) {
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  Scratch<double> Gm(q * q, s), W0(q * q, s), w0(q, s);
  gemm(h, true, false, q, q, p, 1.0, M, ldm, M, ldm, 0.0, Gm, q, /*sym=*/true);
  if (R) {
    Scratch<double> T1(q * q, s);
    gemm(h, false, false, q, q, q, 1.0, R, q, Gm, q, 0.0, T1, q);   // R C
    gemm(h, false, true, q, q, q, 1.0, T1, q, R, q, 0.0, Gm, q);    // (R C) R^T
    k_symmetrize<<<grid_for(q * q, 256, G), 256, 0, s>>>(q, Gm, q);
    FPI_LAUNCH_CHECK();
    note_launch(h);
  }
  // Gram entries are accurate to eps * ||G|| in absolute terms: converge to that (absolute criterion)
  int sw0 = sym_eig(h, q, Gm, q, w0, W0, q, 60, 1e-15, true);
  int sw1 = 0;
  // sigma_i from the Gram eigenpairs carries absolute error ~eps sigma_1^2 / sigma_i; when the kept
  // spectrum is wide (sigma_r / sigma_1 < 1e-3) refine once: M1 = M W0 has nearly orthogonal
  // columns, and the Jacobi solve of its Gram then converges to relative accuracy in a few sweeps.
  double lam[2];
  FPI_CUDA(cudaMemcpyAsync(&lam[0], w0.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaMemcpyAsync(&lam[1], w0.get() + (rank - 1), sizeof(double), cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  const bool refine = !(lam[0] > 0.0) || lam[1] < 1e-6 * lam[0];
  const double* Mr = M;  // columns whose directions are refined
  int64_t ldr = ldm;
  Scratch<double> M1, W1, w1, V;
  const double* Vfin = W0.get();
  const double* Wsel = W0.get();  // maps Mr's columns to the candidate left vectors
  if (refine) {
    M1.alloc(p * q, s);
    W1.alloc(q * q, s);
    w1.alloc(q, s);
    V.alloc(q * q, s);
    if (R) {
      Scratch<double> T0(q * q, s);
      gemm(h, true, false, q, q, q, 1.0, R, q, W0, q, 0.0, T0, q);  // R^T W0
      gemm(h, false, false, p, q, q, 1.0, M, ldm, T0, q, 0.0, M1, q);
    } else {
      gemm(h, false, false, p, q, q, 1.0, M, ldm, W0, q, 0.0, M1, q);
    }
    gemm(h, true, false, q, q, p, 1.0, M1, q, M1, q, 0.0, Gm, q, /*sym=*/true);
    sw1 = sym_eig(h, q, Gm, q, w1, W1, q, 60, 1e-14, false);
    gemm(h, false, false, q, q, q, 1.0, W0, q, W1, q, 0.0, V, q);
    Mr = M1.get();
    ldr = q;
    Vfin = V.get();
    Wsel = W1.get();
  }
  // candidate left vectors for the top `rank` and their norms (= sigma)
  Scratch<double> Uraw(p * rank, s), ss(rank, s), ss2(rank, s);
  Scratch<int32_t> ord(rank, s), ord2(rank, s);
  if (R && !refine) {
    Scratch<double> Wt2(q * rank, s);
    gemm(h, true, false, q, rank, q, 1.0, R, q, Wsel, q, 0.0, Wt2, rank);  // R^T W[:, :rank]
    gemm(h, false, false, p, rank, q, 1.0, M, ldm, Wt2, rank, 0.0, Uraw, rank);
  } else {
    gemm(h, false, false, p, rank, q, 1.0, Mr, ldr, Wsel, q, 0.0, Uraw, rank);
  }
  col_sumsq(h, p, rank, Uraw, rank, ss);
  k_sqrt_clamp<<<grid_for(rank, 256, G), 256, 0, s>>>(rank, ss);
  // sort the kept sigma descending (ties keep order) so factors are flagged sorted
  k_iota32<<<grid_for(rank, 256, G), 256, 0, s>>>(ord, rank);
  CubTemp tmp(s);
  sort_pairs(tmp, ss.get(), ss2.get(), ord.get(), ord2.get(), rank, true, 0, 64, s);
  FPI_CUDA(cudaMemcpyAsync(sigma, ss2.get(), sizeof(double) * rank, cudaMemcpyDeviceToDevice, s));
  // right vectors first: their canonical signs ride along with the gather of the left ones
  Scratch<double> sgn(rank, s);
  k_gather_vt<<<grid_for(rank * q, 256, G), 256, 0, s>>>(q, rank, Vfin, q, ord2, Vt, q);
  canonical_signs_vt(h, rank, q, Vt, q, sgn);
  k_gather_cols_div<<<grid_for(p * rank, 256, G), 256, 0, s>>>(p, rank, Uraw, rank, ord2, ss2, sgn, U, rank);
  FPI_LAUNCH_CHECK();
  note_launch(h, 5);
  complete_null_left(h, p, rank, U, rank, sigma, diag);
  if (diag) {
    // slots 0/1: the first dense SVD of a stage, slots 2/3: the next one (sweeps of pass 1 / pass 2)
    const int slot = diag->eig_sweeps[0] ? 2 : 0;
    diag->eig_sweeps[slot] = sw0;
    diag->eig_sweeps[slot + 1] = sw1;
  }
}

// Many tall panels (p_i >= q_i) at once: Grams -> one batched eigensolve -> per-panel finish.
// Panels whose kept spectrum is wide fall back to the refined single-panel path.
void dense_svd_batched(fpi_context* h, int nb, const int64_t* p, const int64_t* q, const double* const* M,
                       const int64_t* ldm, const int64_t* rank, double* const* U, double* const* sigma,
                       double* const* Vt) {
  if (nb <= 0) return;
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  int64_t tq2 = 0, tq = 0;
  for (int i = 0; i < nb; ++i) {
    tq2 += q[i] * q[i];
    tq += q[i];
  }
  Scratch<double> Gall(tq2, s), Wall(tq2, s), wall(tq, s);
  std::vector<const double*> Gp(nb);
  std::vector<double*> Wp(nb), wp(nb);
  std::vector<int64_t> ldq(nb);
  int64_t o2 = 0, o1 = 0;
  for (int i = 0; i < nb; ++i) {
    double* Gi = Gall.get() + o2;
    gemm(h, true, false, q[i], q[i], p[i], 1.0, M[i], ldm[i], M[i], ldm[i], 0.0, Gi, q[i], /*sym=*/true);
    Gp[i] = Gi;
    Wp[i] = Wall.get() + o2;
    wp[i] = wall.get() + o1;
    ldq[i] = q[i];
    o2 += q[i] * q[i];
    o1 += q[i];
  }
  std::vector<int> sw(nb);
  sym_eig_batched(h, nb, q, Gp.data(), ldq.data(), wp.data(), Wp.data(), ldq.data(), 60, 1e-15, true, sw.data());
  // wide-spectrum test of every panel in one copy
  std::vector<double> hl(2 * nb);
  {
    Scratch<const double*> dw(nb, s);
    Scratch<int64_t> dr(nb, s);
    Scratch<double> dl(2 * nb, s);
    std::vector<const double*> wpc(wp.begin(), wp.end());
    FPI_CUDA(cudaMemcpyAsync(dw.get(), wpc.data(), sizeof(double*) * nb, cudaMemcpyHostToDevice, s));
    FPI_CUDA(cudaMemcpyAsync(dr.get(), rank, sizeof(int64_t) * nb, cudaMemcpyHostToDevice, s));
    k_lam_pairs<<<grid_for(nb, 256, G), 256, 0, s>>>(nb, dw, dr, dl);
    FPI_LAUNCH_CHECK();
    FPI_CUDA(cudaMemcpyAsync(hl.data(), dl.get(), sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, s));
    FPI_CUDA(cudaStreamSynchronize(s));
  }
  // panels with a narrow kept spectrum: Uraw GEMMs, then one batched finish; wide ones: refined path
  std::vector<int> fin;
  int64_t tot_u = 0, rmax = 0;
  for (int i = 0; i < nb; ++i) {
    if (!(hl[2 * i] > 0.0) || hl[2 * i + 1] < 1e-6 * hl[2 * i]) {  // wide spectrum: refined path
      dense_svd(h, p[i], q[i], M[i], ldm[i], rank[i], U[i], sigma[i], Vt[i], nullptr);
      continue;
    }
    fin.push_back(i);
    tot_u += p[i] * rank[i];
    rmax = std::max(rmax, rank[i]);
  }
  if (fin.empty()) return;
  const int nf = (int)fin.size();
  Scratch<double> Uraw_all(tot_u + 1, s);
  std::vector<PanelDesc> pd(nf);
  int64_t ou = 0;
  for (int f = 0; f < nf; ++f) {
    const int i = fin[f];
    double* Uraw = Uraw_all.get() + ou;
    gemm(h, false, false, p[i], rank[i], q[i], 1.0, M[i], ldm[i], Wp[i], q[i], 0.0, Uraw, rank[i]);
    pd[f] = PanelDesc{p[i], q[i], rank[i], Uraw, Wp[i], U[i], sigma[i], Vt[i]};
    ou += p[i] * rank[i];
  }
  Scratch<PanelDesc> dpd(nf, s);
  Scratch<int> zf(nf, s);
  FPI_CUDA(cudaMemcpyAsync(dpd.get(), pd.data(), sizeof(PanelDesc) * nf, cudaMemcpyHostToDevice, s));
  const size_t psmem = (size_t)rmax * (3 * sizeof(double) + sizeof(int)) + 16;
  FPI_REQUIRE(psmem <= h->smem_optin, FPI_ECAPACITY, "batched SVD finish: kept rank too large for shared memory");
  if (psmem > 48 * 1024) {
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, h->device, [&] {
      FPI_CUDA(cudaFuncSetAttribute(k_panel_finish, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(h->smem_optin - 1024)));
    });
  }
  k_panel_finish<<<(unsigned)std::min<int64_t>(nf, (int64_t)h->num_sms * 4), 256, psmem, s>>>(dpd, nf, zf);
  FPI_LAUNCH_CHECK();
  note_launch(h);
  std::vector<int> hz(nf);
  FPI_CUDA(cudaMemcpyAsync(hz.data(), zf.get(), sizeof(int) * nf, cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  for (int f = 0; f < nf; ++f)
    if (hz[f]) complete_null_left(h, p[fin[f]], rank[fin[f]], U[fin[f]], rank[fin[f]], sigma[fin[f]], nullptr);
}

// Orthonormal completion of left vectors whose sigma is numerically zero
// (LAPACK returns some orthonormal completion there; any is valid).
void complete_null_left(fpi_context* h, int64_t p, int64_t rank, double* U, int64_t ldu, const double* sigma,
                        fpi_svd_diag* diag) {
  if (rank <= 0) return;
  cudaStream_t s = h->stream;
  std::vector<double> hs(rank);
  FPI_CUDA(cudaMemcpyAsync(hs.data(), sigma, sizeof(double) * rank, cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  const double tol = 2.220446049250313e-16 * (hs[0] > 0 ? hs[0] : 1.0) * (double)(p > rank ? p : rank);
  std::vector<int64_t> nul;
  for (int64_t j = 0; j < rank; ++j)
    if (!(hs[j] > tol)) nul.push_back(j);
  if (nul.empty()) return;
  FPI_REQUIRE((int64_t)nul.size() <= p, FPI_ENUMERIC, "cannot complete the null space");
  const unsigned G = (unsigned)(h->num_sms * 16);
  Scratch<double> v(p, s), t(rank, s);
  std::vector<double> one(1, 1.0);
  int64_t cand = 0;
  for (int64_t j : nul) {
    // zero column j first so it does not project on itself
    cudaMemset2DAsync(U + j, ldu * sizeof(double), 0, sizeof(double), p, s);
    for (; cand < p; ++cand) {
      k_fill<<<grid_for(p, 256, G), 256, 0, s>>>(p, v, 0.0);
      FPI_CUDA(cudaMemcpyAsync(v.get() + cand, one.data(), sizeof(double), cudaMemcpyHostToDevice, s));
      for (int pass = 0; pass < 2; ++pass) {
        gemm(h, true, false, rank, 1, p, 1.0, U, ldu, v, 1, 0.0, t, 1);     // t = U^T v
        gemm(h, false, false, p, 1, rank, -1.0, U, ldu, t, 1, 1.0, v, 1);   // v -= U t
      }
      Scratch<double> nn(1, s);
      col_sumsq(h, p, 1, v, 1, nn);
      double hn = host_read(nn.get(), s);
      if (hn > 0.25) {
        std::vector<double> inv(1, 1.0 / std::sqrt(hn));
        Scratch<double> sc(1, s);
        FPI_CUDA(cudaMemcpyAsync(sc.get(), inv.data(), sizeof(double), cudaMemcpyHostToDevice, s));
        scale_cols(h, p, 1, v, 1, sc, false);
        FPI_CUDA(cudaMemcpy2DAsync(U + j, ldu * sizeof(double), v.get(), sizeof(double), sizeof(double), p,
                                   cudaMemcpyDeviceToDevice, s));
        FPI_CUDA(cudaStreamSynchronize(s));
        ++cand;
        break;
      }
    }
  }
  if (diag) diag->null_completed += (int32_t)nul.size();
}

void dense_svd(fpi_context* h, int64_t p, int64_t q, const double* M, int64_t ldm, int64_t rank, double* U,
               double* sigma, double* Vt, fpi_svd_diag* diag) {
  FPI_REQUIRE(rank >= 1 && rank <= (p < q ? p : q), FPI_EDOMAIN,
              "target rank " + std::to_string(rank) + " out of range [1, " + std::to_string(p < q ? p : q) + "]");
  // (no capacity guard here: the reference guards only the user-facing dense_svd, svd.py:98-102,
  //  not the small SVD inside randomized_svd, svd.py:136; fpi_dense_svd applies it)
  cudaStream_t s = h->stream;
  if (p >= q) {
    dense_svd_tall(h, p, q, M, ldm, rank, U, sigma, Vt, diag);
    return;
  }
  // M = (M^T)^T :  M^T = U' S V'^T  ->  U = V', Vt = U'^T
  Scratch<double> Mt(q * p, s), U2(q * rank, s), Vt2(rank * p, s);
  transpose(h, p, q, M, ldm, Mt, p);
  dense_svd_tall(h, q, p, Mt, p, rank, U2, sigma, Vt2, diag);
  transpose(h, rank, p, Vt2, p, U, rank);
  transpose(h, q, rank, U2, rank, Vt, q);
  canonical_signs(h, rank, p, q, U, rank, Vt, q);
}

// ---------------------------------------------------------------------------
// inner-matrix operator (inner_op.cuh): B (p x k) = inner * X (q x k)
void InnerOp::sparse_apply(fpi_context* h, const double* Xs, int64_t k, double beta, double* B) const {
  const int64_t q2 = q - sd;
  if (!core) {
    spmm(h, p, q2, k, s_ptr, s_idx, s_val, nullptr, 1.0, Xs, k, beta, B, k);
    return;
  }
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  spmm(h, p, q2, k, core->r_ptr, core->r_idx, core->r_val, nullptr, 1.0, Xs, k, beta, B, k);
  // B[rows] += S[rows, cols] Xs[cols]
  Scratch<double> Xc(core->nC * k, s), tmp(core->nR * k, s);
  k_gather_rows32<<<grid_for(core->nC * k, 256, G), 256, 0, s>>>(core->nC, k, Xs, k, core->cols, Xc, k);
  FPI_LAUNCH_CHECK();
  gemm(h, false, false, core->nR, k, core->nC, 1.0, core->dense, core->nC, Xc, k, 0.0, tmp, k);
  k_scatter_add_rows32<<<grid_for(core->nR * k, 256, G), 256, 0, s>>>(core->nR, k, tmp, k, core->rows, B, k);
  FPI_LAUNCH_CHECK();
  note_launch(h, 2);
}
void InnerOp::sparse_applyT(fpi_context* h, const double* B, int64_t k, double* Z2) const {
  const int64_t q2 = q - sd;
  if (!core) {
    spmm(h, q2, p, k, st_ptr, st_idx, st_val, nullptr, 1.0, B, k, 0.0, Z2, k);
    return;
  }
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  spmm(h, q2, p, k, core->rt_ptr, core->rt_idx, core->rt_val, nullptr, 1.0, B, k, 0.0, Z2, k);
  // Z2[cols] += S[rows, cols]^T B[rows]
  Scratch<double> Bg(core->nR * k, s), tmp(core->nC * k, s);
  k_gather_rows32<<<grid_for(core->nR * k, 256, G), 256, 0, s>>>(core->nR, k, B, k, core->rows, Bg, k);
  FPI_LAUNCH_CHECK();
  gemm(h, true, false, core->nC, k, core->nR, 1.0, core->dense, core->nC, Bg, k, 0.0, tmp, k);
  k_scatter_add_rows32<<<grid_for(core->nC * k, 256, G), 256, 0, s>>>(core->nC, k, tmp, k, core->cols, Z2, k);
  FPI_LAUNCH_CHECK();
  note_launch(h, 2);
}
void InnerOp::apply(fpi_context* h, const double* X, int64_t k, double* B) const {
  if (D && sd > 0 && nzr >= 0) {
    cudaStream_t s = h->stream;
    const unsigned G = (unsigned)(h->num_sms * 16);
    if (q > sd)
      sparse_apply(h, X + sd * k, k, 0.0, B);
    else
      FPI_CUDA(cudaMemsetAsync(B, 0, sizeof(double) * p * k, s));
    if (nzr > 0) {
      Scratch<double> Xs(sd * k, s), tmp(nzr * k, s);
      FPI_CUDA(cudaMemcpyAsync(Xs.get(), X, sizeof(double) * sd * k, cudaMemcpyDeviceToDevice, s));
      if (dscale) scale_rows(h, sd, k, Xs, k, dscale);
      gemm(h, false, false, nzr, k, sd, 1.0, Dnz, sd, Xs, k, 0.0, tmp, k);
      k_scatter_add_rows32<<<grid_for(nzr * k, 256, G), 256, 0, s>>>(nzr, k, tmp, k, nz_rows, B, k);
      FPI_LAUNCH_CHECK();
    }
    return;
  }
  if (D && sd > 0) {
    Scratch<double> Xs(sd * k, h->stream);
    FPI_CUDA(cudaMemcpyAsync(Xs.get(), X, sizeof(double) * sd * k, cudaMemcpyDeviceToDevice, h->stream));
    if (dscale) scale_rows(h, sd, k, Xs, k, dscale);
    gemm(h, false, false, p, k, sd, 1.0, D, ldd, Xs, k, 0.0, B, k);
    if (q > sd) sparse_apply(h, X + sd * k, k, 1.0, B);
  } else {
    sparse_apply(h, X, k, 0.0, B);
  }
}
// Z (q x k) = inner^T * B (p x k)
void InnerOp::applyT(fpi_context* h, const double* B, int64_t k, double* Z) const {
  if (D && sd > 0 && nzr >= 0) {
    cudaStream_t s = h->stream;
    const unsigned G = (unsigned)(h->num_sms * 16);
    if (nzr > 0) {
      Scratch<double> Bg(nzr * k, s);
      k_gather_rows32<<<grid_for(nzr * k, 256, G), 256, 0, s>>>(nzr, k, B, k, nz_rows, Bg, k);
      FPI_LAUNCH_CHECK();
      gemm(h, true, false, sd, k, nzr, 1.0, Dnz, sd, Bg, k, 0.0, Z, k);
      if (dscale) scale_rows(h, sd, k, Z, k, dscale);
    } else {
      FPI_CUDA(cudaMemsetAsync(Z, 0, sizeof(double) * sd * k, s));
    }
    if (q > sd) sparse_applyT(h, B, k, Z + sd * k);
    return;
  }
  if (D && sd > 0) {
    gemm(h, true, false, sd, k, p, 1.0, D, ldd, B, k, 0.0, Z, k);
    if (dscale) scale_rows(h, sd, k, Z, k, dscale);
    if (q > sd) sparse_applyT(h, B, k, Z + sd * k);
  } else {
    sparse_applyT(h, B, k, Z);
  }
}
// dense copy (p x q)
void InnerOp::densify(fpi_context* h, double* out) const {
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  k_fill<<<grid_for(p * q, 256, G), 256, 0, s>>>(p * q, out, 0.0);
  if (D && sd > 0) {
    k_copy2d<<<grid_for(p * sd, 256, G), 256, 0, s>>>(p, sd, D, ldd, out, q);
    if (dscale) scale_cols(h, p, sd, out, q, dscale, false);
  }
  if (q > sd) k_csr_to_dense<<<grid_for(p * 32, 256, G), 256, 0, s>>>(p, s_ptr, s_idx, s_val, out, q, sd);
  FPI_LAUNCH_CHECK();
  note_launch(h, 3);
}

void symmetrize(fpi_context* h, int64_t n, double* A, int64_t lda) {
  k_symmetrize<<<grid_for(n * n, 256, (unsigned)(h->num_sms * 16)), 256, 0, h->stream>>>(n, A, lda);
  FPI_LAUNCH_CHECK();
  note_launch(h);
}

// Q = B L^-T orthonormal from the Gram G = B^T B (k x k, preserved): CholeskyQR (svd.py:134's QR
// without forming Q), or, when G is not numerically positive definite, an eigen-based factor.
void orth_factor(fpi_context* h, int64_t k, const double* Gm, double* Linv, fpi_svd_diag* diag) {
  cudaStream_t s = h->stream;
  // (A one-kernel cooperative Cholesky + inverse was measured at 1.6 vs 2.5 ms for k = 1000 but
  // stalled the stream for 0.1-0.6 s on some launches; the launch-per-panel path below is kept.)
  Scratch<double> Gc(k * k, s);
  int info = 0;
  // L and L^-1 in one tile-dataflow kernel (chol_dataflow.cu); the blocked panel path otherwise
  const bool fused = chol_inverse_dataflow(h, k, Gm, k, Gc, k, Linv, k, &info);
  if (!fused) {
    FPI_CUDA(cudaMemcpyAsync(Gc.get(), Gm, sizeof(double) * k * k, cudaMemcpyDeviceToDevice, s));
    cholesky_lower(h, k, Gc, k, &info);
  }
  if (info == 0) {
    if (diag) {
      Scratch<double> ratio(1, s);
      k_diag_ratio<<<1, 256, 0, s>>>(k, Gc, k, ratio);
      diag->cond_estimate = host_read(ratio.get(), s);
      diag->cholqr_passes = 1;
    }
    if (!fused) lower_inverse(h, k, Gc, k, Linv, k);
    return;
  }
  // not numerically PD (B rank deficient): orthonormalise through the eigendecomposition
  Scratch<double> w(k, s), W(k * k, s);
  sym_eig(h, k, Gm, k, w, W, k, 60, 1e-15, true);
  k_eig_orth<<<grid_for(k * k, 256, h->num_sms * 16), 256, 0, s>>>(k, w, W, 1e-26, Linv);
  FPI_LAUNCH_CHECK();
  if (diag) {
    diag->cond_estimate = INFINITY;
    diag->cholqr_passes = 0;
  }
}

// The finish of the randomized SVD from the right side (svd.py:135-137): with W the top eigenvectors
// of Y Y^T = L^-1 (Z^T Z) L^-T, the left vectors are U = Q W = B (L^-T W) and the right ones
// V = Y^T W / sigma = inner^T U / sigma.  For a wide sparse inner (the row update's
// [Sigma Vt11 ; A21], q = n1 >> p) that is one SpMM of inner^T with r columns instead of the
// q x 2r x r product Z (L^-T W) of the left-side finish.  sigma_i = ||inner^T u_i|| as in the
// left-side finish (column norms).  Returns false (nothing written) when the kept spectrum is wide
// enough to need the refined path.
static bool rsvd_finish_right(fpi_context* h, const InnerOp& op, int64_t rank, const double* X, const double* B,
                              const double* Z, const double* Linv, double* U, double* sigma, double* Vt,
                              fpi_svd_diag* diag) {
  cudaStream_t s = h->stream;
  const int64_t p = op.p, q = op.q, k = 2 * rank;
  const unsigned G = (unsigned)(h->num_sms * 16);
  Scratch<double> Gm(k * k, s), T1(k * k, s), W0(k * k, s), w0(k, s);
  gemm(h, true, false, k, k, q, 1.0, Z, k, Z, k, 0.0, Gm, k, /*sym=*/true);
  gemm(h, false, false, k, k, k, 1.0, Linv, k, Gm, k, 0.0, T1, k);   // L^-1 (Z^T Z)
  gemm(h, false, true, k, k, k, 1.0, T1, k, Linv, k, 0.0, Gm, k);    // ... L^-T
  k_symmetrize<<<grid_for(k * k, 256, G), 256, 0, s>>>(k, Gm, k);
  FPI_LAUNCH_CHECK();
  note_launch(h);
  T1.release();
  const int sw0 = sym_eig(h, k, Gm, k, w0, W0, k, 60, 1e-15, true);
  double lam[2];
  FPI_CUDA(cudaMemcpyAsync(&lam[0], w0.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaMemcpyAsync(&lam[1], w0.get() + (rank - 1), sizeof(double), cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  if (!(lam[0] > 0.0) || lam[1] < 1e-6 * lam[0]) return false;  // wide spectrum: refined left-side path
  Gm.release();
  // U0 = Q W[:, :r] = B (L^-T W) or inner (X (L^-T W))
  Scratch<double> Mx(k * rank, s), U0(p * rank, s);
  gemm(h, true, false, k, rank, k, 1.0, Linv, k, W0, k, 0.0, Mx, rank);
  if (!B || op.apply_cost(rank) + 2.0 * (double)q * (double)k * (double)rank < 2.0 * (double)p * (double)k * (double)rank) {
    Scratch<double> XM(q * rank, s);
    gemm(h, false, false, q, rank, k, 1.0, X, k, Mx, rank, 0.0, XM, rank);
    op.apply(h, XM, rank, U0);
  } else {
    gemm(h, false, false, p, rank, k, 1.0, B, k, Mx, rank, 0.0, U0, rank);
  }
  // V sigma = inner^T U0
  Scratch<double> Vs(q * rank, s), ss(rank, s), ss2(rank, s), ones(rank, s), sgn(rank, s);
  op.applyT(h, U0, rank, Vs);
  col_sumsq(h, q, rank, Vs, rank, ss);
  k_sqrt_clamp<<<grid_for(rank, 256, G), 256, 0, s>>>(rank, ss);
  Scratch<int32_t> ord(rank, s), ord2(rank, s);
  k_iota32<<<grid_for(rank, 256, G), 256, 0, s>>>(ord, rank);
  CubTemp tmp(s);
  sort_pairs(tmp, ss.get(), ss2.get(), ord.get(), ord2.get(), rank, true, 0, 64, s);
  FPI_CUDA(cudaMemcpyAsync(sigma, ss2.get(), sizeof(double) * rank, cudaMemcpyDeviceToDevice, s));
  k_gather_vt_div<<<grid_for(rank * q, 256, G), 256, 0, s>>>(q, rank, Vs, rank, ord2, ss2, Vt, q);
  canonical_signs_vt(h, rank, q, Vt, q, sgn);
  k_fill<<<grid_for(rank, 256, G), 256, 0, s>>>(rank, ones, 1.0);
  k_gather_cols_div<<<grid_for(p * rank, 256, G), 256, 0, s>>>(p, rank, U0, rank, ord2, ones, sgn, U, rank);
  FPI_LAUNCH_CHECK();
  note_launch(h, 5);
  if (diag) {
    const int slot = diag->eig_sweeps[0] ? 2 : 0;
    diag->eig_sweeps[slot] = sw0;
    diag->eig_sweeps[slot + 1] = 0;
  }
  return true;
}

// ---------------------------------------------------------------------------
// Robust orthonormalisation of an ill-conditioned or rank-deficient sketch product B (p x k),
// the fallback behind svd.py:134's QR when CholeskyQR's cond(B)^2 is too much for FP64.
// Deflated eigen-orthonormalisation: every pass takes the Gram of the residual R (first B),
// keeps the eigen-directions within 1e-8 of its largest eigenvalue (condition <= 1e4 among
// them, so R W Lambda^-1/2 is orthonormal to ~1e-8), brings them to rounding level by two
// rounds of projection against the columns already found plus CholeskyQR, and removes them from
// R.  Each pass resolves four decades of B's spectrum; the loop ends when k columns are found or
// the residual is at the rounding floor of B, and the remaining columns (a numerically rank-
// deficient B) are an orthonormal completion -- as Householder QR would return.  All GEMM-shaped
// work on DMMA; the k x k eigenproblems on the Jacobi kernel.  On return B holds Q.
__global__ void k_scale_eigvec_cols(int64_t k, int64_t S, const double* __restrict__ W, const double* __restrict__ w,
                                    double* __restrict__ Ws) {
  FPI_GRID_STRIDE(e, k * S) {
    const int64_t i = e / S, j = e - i * S;
    Ws[e] = W[i * k + j] / sqrt(w[j]);
  }
}
__global__ void k_identity_kk(int64_t k, double* __restrict__ A) {
  FPI_GRID_STRIDE(e, k * k) A[e] = (e / k == e % k) ? 1.0 : 0.0;
}
__global__ void k_flags01(int64_t k, int64_t found, double* __restrict__ f) {
  FPI_GRID_STRIDE(i, k) f[i] = i < found ? 1.0 : 0.0;
}

static int64_t orthonormalize_deflated(fpi_context* h, int64_t p, int64_t k, double* B, fpi_svd_diag* diag) {
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  const double eps = 2.220446049250313e-16;
  Scratch<double> Q(p * k, s), Gm(k * k, s), W(k * k, s), w(k, s);
  FPI_CUDA(cudaMemsetAsync(Q.get(), 0, sizeof(double) * p * k, s));
  std::vector<double> hw(k);
  int64_t found = 0;
  double total = 0.0;
  for (int pass = 0; pass < 8 && found < k; ++pass) {
    gemm(h, true, false, k, k, p, 1.0, B, k, B, k, 0.0, Gm, k, /*sym=*/true);
    sym_eig(h, k, Gm, k, w, W, k, 60, 1e-15, true);
    FPI_CUDA(cudaMemcpyAsync(hw.data(), w.get(), sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    FPI_CUDA(cudaStreamSynchronize(s));
    if (pass == 0) total = hw[0];
    // residual at the rounding floor of B (sigma <= 16 eps sqrt(k) ||B||): the rest is a completion
    if (!(hw[0] > 0.0) || hw[0] <= 256.0 * eps * eps * (double)k * total) break;
    int64_t S = 0;
    while (S < k - found && S < k && hw[S] > 1e-8 * hw[0]) ++S;
    if (S == 0) break;
    Scratch<double> Ws(k * S, s), Qn(p * S, s), T(p * S, s);
    k_scale_eigvec_cols<<<grid_for(k * S, 256, G), 256, 0, s>>>(k, S, W, w, Ws);
    FPI_LAUNCH_CHECK();
    gemm(h, false, false, p, S, k, 1.0, B, k, Ws, S, 0.0, Qn, S);
    for (int round = 0; round < 2; ++round) {
      if (found > 0) {  // Qn -= Q (Q^T Qn)
        Scratch<double> C(found * S, s);
        gemm(h, true, false, found, S, p, 1.0, Q, k, Qn, S, 0.0, C, S);
        gemm(h, false, false, p, S, found, -1.0, Q, k, C, S, 1.0, Qn, S);
      }
      Scratch<double> G2(S * S, s), L(S * S, s), Li(S * S, s);
      gemm(h, true, false, S, S, p, 1.0, Qn, S, Qn, S, 0.0, G2, S, /*sym=*/true);
      int info = 0;
      FPI_CUDA(cudaMemcpyAsync(L.get(), G2.get(), sizeof(double) * S * S, cudaMemcpyDeviceToDevice, s));
      cholesky_lower(h, S, L, S, &info);
      FPI_REQUIRE(info == 0, FPI_ENUMERIC, "orthonormalisation of the sketch product failed (re-orthogonalisation)");
      lower_inverse(h, S, L, S, Li, S);
      gemm(h, false, true, p, S, S, 1.0, Qn, S, Li, S, 0.0, T, S);   // Qn L^-T
      FPI_CUDA(cudaMemcpyAsync(Qn.get(), T.get(), sizeof(double) * p * S, cudaMemcpyDeviceToDevice, s));
    }
    FPI_CUDA(cudaMemcpy2DAsync(Q.get() + found, k * sizeof(double), Qn.get(), S * sizeof(double), S * sizeof(double),
                               p, cudaMemcpyDeviceToDevice, s));
    found += S;
    if (found < k) {  // R -= Qn (Qn^T R)
      Scratch<double> C2(S * k, s);
      gemm(h, true, false, S, k, p, 1.0, Qn, S, B, k, 0.0, C2, k);
      gemm(h, false, false, p, k, S, -1.0, Qn, S, C2, k, 1.0, B, k);
    }
  }
  if (found < k) {
    Scratch<double> flags(k, s);
    k_flags01<<<grid_for(k, 256, G), 256, 0, s>>>(k, found, flags);
    FPI_LAUNCH_CHECK();
    complete_null_left(h, p, k, Q, k, flags, diag);
  }
  FPI_CUDA(cudaMemcpyAsync(B, Q.get(), sizeof(double) * p * k, cudaMemcpyDeviceToDevice, s));
  return found;
}

static void randomized_svd(fpi_context* h, const InnerOp& op, int64_t rank, int64_t seed, double* U, double* sigma,
                           double* Vt, fpi_svd_diag* diag) {
  const int64_t p = op.p, q = op.q;
  FPI_REQUIRE(rank >= 1 && rank <= (p < q ? p : q), FPI_EDOMAIN,
              "target rank " + std::to_string(rank) + " out of range [1, " + std::to_string(p < q ? p : q) + "]");
  cudaStream_t s = h->stream;
  const int64_t k = 2 * rank;
  if (diag) diag->engine = 1;
  if (p <= k) {
    // QR of a p x 2r sketch with p <= 2r gives a p x p orthogonal Q: the result is the exact SVD of inner.
    // No capacity guard, as in the reference (svd.py:120-138): p <= 2r rows of q columns fit HBM
    // at every size the rank rule admits.
    Scratch<double> Dn(p * q, s);
    op.densify(h, Dn);
    dense_svd(h, p, q, Dn, q, rank, U, sigma, Vt, diag);
    return;
  }
  trace_point(h, "rsvd:start");
  Scratch<double> X(q * k, s), B, Gm(k * k, s), Linv(k * k, s);
  sketch_normal(h, seed, q, k, X, k);   // svd.py:131-132
  trace_point(h, "rsvd:sketch");
  // Z = inner^T B = inner^T inner X, with B = inner X (svd.py:133) and Y^T = Z L^-T (svd.py:135:
  // Y = Q^T inner).  Two ways: through B (two passes of inner over k columns), or, for a tall
  // inner with few columns, through the q x q Gram H = inner^T inner (gram_route.cu): Z = H X and
  // B never exists.  Both are the same product; the cost model picks the cheaper.
  Scratch<double> Z(q * k, s);
  GramPlan gp;
  SparseGramIn gin;
  if (op.s_ptr && op.st_ptr && q > op.sd && 2 * q < p) {
    gin = op.gram_in();
    gp = plan_inner_gram(h, gin, k);
  }
  bool gram_from_z = gp.use;
  if (gp.use) {
    Scratch<double> H(q * q, s);
    inner_gram(h, gin, gp, H, q);
    trace_point(h, "rsvd:H = M^T M");
    gemm(h, false, false, q, k, q, 1.0, H, q, X, k, 0.0, Z, k);
    trace_point(h, "rsvd:Z = H X");
  } else {
    B.alloc(p * k, s);
    op.apply(h, X, k, B);
    trace_point(h, "rsvd:B = M X");
    // CholeskyQR: B^T B = L L^T, Q = B L^-T  (svd.py:134).  B^T B = X^T (inner^T B) = X^T Z: for a
    // tall inner (q < p / 2) the Gram comes from the q x k Z at 2 q k^2 flops instead of the p x k
    // B at p k^2 -- at c5 that is 0.1 instead of 4 TFLOP.  The product of two different factors
    // is symmetrised; its rounding (eps ||X|| ||Z||) is of the order of the direct Gram's.
    gram_from_z = 2 * q < p && getenv("FPI_RSVD_DIRECT_GRAM") == nullptr;
    if (gram_from_z) {
      op.applyT(h, B, k, Z);
      trace_point(h, "rsvd:Z = M^T B");
    }
  }
  if (gram_from_z) {
    gemm(h, true, false, k, k, q, 1.0, X, k, Z, k, 0.0, Gm, k);
    k_symmetrize<<<grid_for(k * k, 256, (unsigned)(h->num_sms * 16)), 256, 0, s>>>(k, Gm, k);
    FPI_LAUNCH_CHECK();
    note_launch(h);
    trace_point(h, "rsvd:gram X^T Z");
  } else {
    gemm(h, true, false, k, k, p, 1.0, B, k, B, k, 0.0, Gm, k, /*sym=*/true);
    trace_point(h, "rsvd:gram B^T B");
  }
  fpi_svd_diag local_diag{};
  if (!diag) diag = &local_diag;
  orth_factor(h, k, Gm, Linv, diag);
  Gm.release();
  trace_point(h, "rsvd:cholesky/inverse");
  // CholeskyQR loses cond(B)^2: past ~1e4 (or when B^T B is not numerically positive definite) the
  // sketch product is orthonormalised explicitly by the deflated eigen-orthonormalisation and the
  // rest of svd.py:135-137 runs on that Q (L = I).  The BASELINE configs measure cond 1.06 - 4.5.
  const bool robust = getenv("FPI_RSVD_NO_ROBUST") == nullptr &&
                      (diag->cholqr_passes == 0 || !(diag->cond_estimate < 1e4));
  if (robust) {
    if (!B.get()) {
      B.alloc(p * k, s);
      op.apply(h, X, k, B);
    }
    const int64_t found = orthonormalize_deflated(h, p, k, B, diag);
    (void)found;
    k_identity_kk<<<grid_for(k * k, 256, (unsigned)(h->num_sms * 16)), 256, 0, s>>>(k, Linv);
    FPI_LAUNCH_CHECK();
    op.applyT(h, B, k, Z);   // Y^T = inner^T Q
    diag->cholqr_passes = 0;
    trace_point(h, "rsvd:robust orthonormalisation");
  } else if (!gram_from_z) {
    op.applyT(h, B, k, Z);
    trace_point(h, "rsvd:Z = M^T B");
  }
  // SVD of Y (k x q) through its transpose Y^T = Z L^-T = Vy S Uy^T   (svd.py:135-136); for a tall
  // Y^T the product is left implicit (Gram L^-1 (Z^T Z) L^-T)
  // implicit only when L is well conditioned: the Gram of Z carries cond(L)^2 more rounding than
  // the Gram of Y^T (the CholeskyQR sketches here measure cond 1.2 - 2.7)
  const bool implicit_ok = !robust && q >= k && diag->cond_estimate > 0.0 && diag->cond_estimate < 8.0;
  // right-side finish when one pass of inner^T over r columns undercuts the q x 2r x r product
  if (implicit_ok && getenv("FPI_RSVD_LEFT_FINISH") == nullptr &&
      op.apply_cost(rank) < 0.5 * 2.0 * (double)q * (double)k * (double)rank &&
      rsvd_finish_right(h, op, rank, X, B.get(), Z, Linv, U, sigma, Vt, diag)) {
    trace_point(h, "rsvd:right-side finish");
    if (diag) diag->engine = 1;
    return;
  }
  Scratch<double> Vy(q * rank, s), Uyt(rank * k, s);
  if (implicit_ok) {
    dense_svd_tall(h, q, k, Z, k, rank, Vy, sigma, Uyt, diag, Linv);
  } else {
    Scratch<double> Yt(q * k, s);
    gemm(h, false, true, q, k, k, 1.0, Z, k, Linv, k, 0.0, Yt, k);
    dense_svd(h, q, k, Yt, k, rank, Vy, sigma, Uyt, diag);
  }
  Z.release();
  trace_point(h, "rsvd:dense_svd(Yt)");
  transpose(h, q, rank, Vy, rank, Vt, q);                   // Vt = Vy^T
  trace_point(h, "rsvd:transpose Vy");
  // U = Q U~ = B L^-T U~ ,  U~ = Uyt^T   (svd.py:137)
  Scratch<double> Mx(k * rank, s);
  gemm(h, true, true, k, rank, k, 1.0, Linv, k, Uyt, k, 0.0, Mx, rank);
  // canonical signs from Vt; U's columns follow through Mx's (no pass over the p x r U)
  {
    Scratch<double> sgn(rank, s);
    canonical_signs_vt(h, rank, q, Vt, q, sgn);
    scale_cols(h, k, rank, Mx, rank, sgn, false);
  }
  if (!robust && (!B.get() || op.apply_cost(rank) + 2.0 * (double)q * (double)k * (double)rank <
                                  2.0 * (double)p * (double)k * (double)rank)) {
    // = inner (X L^-T U~): the thin q x r factor first, then one pass of the inner operator -- about
    // half the flops of the p x 2r x r product with B when inner is [U Sigma | T] with a tall U
    B.release();
    Scratch<double> XM(q * rank, s);
    gemm(h, false, false, q, rank, k, 1.0, X, k, Mx, rank, 0.0, XM, rank);
    X.release();
    op.apply(h, XM, rank, U);
  } else {
    gemm(h, false, false, p, rank, k, 1.0, B, k, Mx, rank, 0.0, U, rank);
  }
  trace_point(h, "rsvd:U");
  if (diag) diag->engine = 1;
}

static void inner_svd(fpi_context* h, const InnerOp& op, int64_t rank, int64_t n_cols, double thr, int64_t seed,
                      double* U, double* sigma, double* Vt, int* engine, fpi_svd_diag* diag) {
  if ((double)rank < thr * (double)n_cols) {  // pinv.py:122
    *engine = 1;
    randomized_svd(h, op, rank, seed, U, sigma, Vt, diag);
  } else {
    *engine = 2;
    if (diag) diag->engine = 2;
    FPI_REQUIRE(op.p * op.q <= 100000000LL, FPI_ECAPACITY,
                "dense SVD of a " + std::to_string(op.p) + "x" + std::to_string(op.q) +
                    " matrix exceeds the 100000000-entry guard");
    Scratch<double> Dn(op.p * op.q, h->stream);
    op.densify(h, Dn);
    dense_svd(h, op.p, op.q, Dn, op.q, rank, U, sigma, Vt, diag);
  }
}

void row_update(fpi_context* h, int64_t m1, int64_t n1, int64_t rank11, const double* sigma11, const int64_t* u_ptr,
                const int32_t* u_idx, const double* u_val, const int64_t* v_ptr, const int32_t* v_idx,
                const double* v_val, int64_t m2, const int64_t* a_ptr, const int32_t* a_idx, const double* a_val,
                int64_t s_rank, double thr, int64_t seed, double* U, double* sigma, double* Vt, int* engine) {
  cudaStream_t s = h->stream;
  *engine = 0;
  if (s_rank == 0) return;
  const int64_t max_rank = (rank11 + m2 < n1) ? rank11 + m2 : n1;
  FPI_REQUIRE(s_rank >= 1 && s_rank <= max_rank, FPI_EDOMAIN,
              "target rank " + std::to_string(s_rank) + " out of range [1, " + std::to_string(max_rank) + "]");
  const int64_t p = rank11 + m2, q = n1;
  int64_t nnz_v = 0, nnz_a = 0;
  if (rank11) nnz_v = host_read(v_ptr + rank11, s);
  if (m2) nnz_a = host_read(a_ptr + m2, s);
  const int64_t nnz = nnz_v + nnz_a;
  const unsigned G = (unsigned)(h->num_sms * 16);
  // inner = [diag(sigma11) Vt11 ; A21] as one CSR, plus its transpose (pinv.py:161-163)
  Scratch<int64_t> iptr(p + 1, s), itptr(q + 1, s);
  Scratch<int32_t> iidx(nnz, s), itidx(nnz, s);
  Scratch<double> ival(nnz, s), itval(nnz, s);
  Scratch<int64_t> zero_ptr(1, s);
  FPI_CUDA(cudaMemsetAsync(zero_ptr.get(), 0, sizeof(int64_t), s));
  k_inner_rows<<<grid_for(p + 1, 256, G), 256, 0, s>>>(rank11, m2, rank11 ? v_ptr : zero_ptr.get(),
                                                       m2 ? a_ptr : zero_ptr.get(), nnz_v, iptr);
  k_inner_vals<<<grid_for(rank11 * 32 + nnz_a, 256, G), 256, 0, s>>>(rank11, v_ptr, v_idx, v_val, sigma11, nnz_v,
                                                                     nnz_a, a_idx, a_val, iidx, ival);
  FPI_LAUNCH_CHECK();
  note_launch(h, 2);
  csr_transpose(h, p, q, nnz, iptr, iidx, ival, itptr, itidx, itval);
  InnerOp op;
  op.p = p;
  op.q = q;
  op.s_nnz = nnz;
  op.s_ptr = iptr;
  op.s_idx = iidx;
  op.s_val = ival;
  op.st_ptr = itptr;
  op.st_idx = itidx;
  op.st_val = itval;
  Scratch<double> Ui(p * s_rank, s);
  inner_svd(h, op, s_rank, n1, thr, seed, Ui, sigma, Vt, engine, &h->diag);
  // lift: U = [U11 Ui[:rank11] ; Ui[rank11:]]   (pinv.py:168-170)
  if (m1) {
    if (rank11 && (s_rank & 1)) {
      // odd width: the gathered rows go through a copy with an even stride so the SpMM can use
      // its 16-byte gathers (spmm.cu)
      const int64_t ldp = s_rank + 1;
      Scratch<double> Up(rank11 * ldp, s);
      FPI_CUDA(cudaMemcpy2DAsync(Up.get(), ldp * sizeof(double), Ui.get(), s_rank * sizeof(double),
                                 s_rank * sizeof(double), rank11, cudaMemcpyDeviceToDevice, s));
      spmm(h, m1, rank11, s_rank, u_ptr, u_idx, u_val, nullptr, 1.0, Up, ldp, 0.0, U, s_rank);
    } else if (rank11)
      spmm(h, m1, rank11, s_rank, u_ptr, u_idx, u_val, nullptr, 1.0, Ui, s_rank, 0.0, U, s_rank);
    else
      FPI_CUDA(cudaMemsetAsync(U, 0, sizeof(double) * m1 * s_rank, s));
  }
  if (m2)
    FPI_CUDA(cudaMemcpyAsync(U + m1 * s_rank, Ui.get() + rank11 * s_rank, sizeof(double) * m2 * s_rank,
                             cudaMemcpyDeviceToDevice, s));
}

void column_update(fpi_context* h, int64_t m, int64_t s_prev, int64_t n1, const double* U_prev,
                   const double* sigma_prev, const double* Vt_prev, int64_t n2, const int64_t* t_ptr,
                   const int32_t* t_idx, const double* t_val, const int64_t* tt_ptr, const int32_t* tt_idx,
                   const double* tt_val, int64_t r, double thr, int64_t seed, double* U, double* sigma, double* Vt,
                   int* engine) {
  cudaStream_t s = h->stream;
  *engine = 0;
  if (r == 0) return;
  const int64_t max_rank = (s_prev + n2 < m) ? s_prev + n2 : m;
  FPI_REQUIRE(r >= 1 && r <= max_rank, FPI_EDOMAIN,
              "target rank " + std::to_string(r) + " out of range [1, " + std::to_string(max_rank) + "]");
  const int64_t q = s_prev + n2;
  InnerOp op;
  op.p = m;
  op.q = q;
  op.D = U_prev;
  op.ldd = s_prev;
  op.sd = s_prev;
  op.dscale = sigma_prev;
  op.s_ptr = t_ptr;
  op.s_idx = t_idx;
  op.s_val = t_val;
  op.st_ptr = tt_ptr;
  op.st_idx = tt_idx;
  op.st_val = tt_val;
  op.s_nnz = (n2 && m) ? host_read(t_ptr + m, s) : 0;
  // rows of U_prev that are identically zero (spoke rows of column-free blocks): skip them in the
  // dense products of the randomized engine when they are the majority
  Scratch<int32_t> flag, ids, nzl, cntd;
  Scratch<double> Dnz;
  if (s_prev > 0 && (double)r < thr * (double)q) {
    const unsigned G = (unsigned)(h->num_sms * 16);
    flag.alloc(m, s);
    ids.alloc(m, s);
    nzl.alloc(m, s);
    cntd.alloc(1, s);
    k_row_nonzero<<<grid_for(m * 32, 256, G), 256, 0, s>>>(m, s_prev, U_prev, s_prev, flag);
    k_iota_i32<<<grid_for(m, 256, G), 256, 0, s>>>(ids, m);
    CubTemp tmp(s);
    select_if(tmp, ids.get(), nzl.get(), cntd.get(), m, FlagSet{flag.get()}, s);
    const int64_t nzr = host_read(cntd.get(), s);
    if (nzr < (m * 6) / 10) {
      Dnz.alloc(nzr * s_prev + 1, s);
      if (nzr)
        k_gather_rows32<<<grid_for(nzr * s_prev, 256, G), 256, 0, s>>>(nzr, s_prev, U_prev, s_prev, nzl, Dnz,
                                                                       s_prev);
      FPI_LAUNCH_CHECK();
      op.nzr = nzr;
      op.nz_rows = nzl.get();
      op.Dnz = Dnz.get();
    }
  }
  trace_point(h, "col: zero-row scan");
  // the heavy rows x heavy columns rectangle of T on the tensor pipe (sparse_core.cu)
  SparseCore core;
  for (int64_t& v : h->sparse_core) v = 0;
  if (n2 > 0 && (double)r < thr * (double)q && m > 2 * r) {
    build_sparse_core(h, m, n2, op.s_nnz, t_ptr, t_idx, t_val, tt_ptr, tt_idx, tt_val, core);
    if (core.use) {
      op.core = &core;
      h->sparse_core[0] = core.nR;
      h->sparse_core[1] = core.nC;
      h->sparse_core[2] = core.core_nnz;
      h->sparse_core[3] = core.rem_nnz;
    }
    trace_point(h, "col: sparse core");
  }
  Scratch<double> Vti(r * q, s);
  inner_svd(h, op, r, q, thr, seed, U, sigma, Vti, engine, &h->diag);
  trace_point(h, "col: inner svd");
  // lift: Vt = [Vti[:, :s] Vt_prev | Vti[:, s:]]   (pinv.py:205-207)
  const int64_t n = n1 + n2;
  if (n1) {
    if (s_prev)
      gemm(h, false, false, r, n1, s_prev, 1.0, Vti, q, Vt_prev, n1, 0.0, Vt, n);
    else
      FPI_CUDA(cudaMemset2DAsync(Vt, n * sizeof(double), 0, n1 * sizeof(double), r, s));
  }
  if (n2)
    FPI_CUDA(cudaMemcpy2DAsync(Vt + n1, n * sizeof(double), Vti.get() + s_prev, q * sizeof(double),
                               n2 * sizeof(double), r, cudaMemcpyDeviceToDevice, s));
  trace_point(h, "col: lift");
}

void pinv_assemble(fpi_context* h, int64_t r, const double* sigma, int64_t p, int64_t q, double cutoff,
                   double* sdag, double* tol_out, int* all_filtered) {
  cudaStream_t s = h->stream;
  Scratch<double> t(1, s);
  Scratch<int> af(1, s);
  int64_t maxpq = p > q ? p : q;
  if (maxpq < 1) maxpq = 1;
  k_pinv<<<1, 256, 0, s>>>(r, sigma, cutoff, maxpq, sdag, t, af);
  FPI_LAUNCH_CHECK();
  note_launch(h);
  *tol_out = host_read(t.get(), s);
  *all_filtered = host_read(af.get(), s);
}

void unfold_transpose(fpi_context* h, int64_t m, int64_t n, int64_t r, const double* U, const double* Vt,
                      const int64_t* row_fwd, const int64_t* col_fwd, double* V_out, double* Ut_out) {
  cudaStream_t s = h->stream;
  if (Ut_out && m && r) {
    dim3 blk(32, 8);
    int64_t gx = (r + 31) / 32, gy = (m + 31) / 32;
    dim3 grd((unsigned)(gx < 65535 ? gx : 65535), (unsigned)(gy < 65535 ? gy : 65535));
    k_gather_rows_T<<<grd, blk, 0, s>>>(m, r, U, r, row_fwd, Ut_out, m);
  }
  if (V_out && n && r)
    k_gather_cols_T<<<grid_for(n * r, 256, h->num_sms * 16), 256, 0, s>>>(n, r, Vt, n, col_fwd, V_out, r);
  FPI_LAUNCH_CHECK();
  note_launch(h, 2);
}

// Columns of Vt in original order: Vg[:, i] = Vt[:, col_fwd[i]] (the unfold of pinv.py:271-275 for V).
__global__ void k_gather_cols(int64_t r, int64_t n, const double* __restrict__ Vt, const int64_t* __restrict__ col_fwd,
                              double* __restrict__ Vg) {
  FPI_GRID_STRIDE(e, r * n) {
    const int64_t k = e / n, i = e - k * n;
    Vg[e] = Vt[k * n + col_fwd[i]];
  }
}

// Z (n x L) = V diag(sdag) U^T Y  with U, Vt in reordered coordinates and Y (m x L) CSR in original rows
// W (L x r) = Y'^T U_loc for the reordered rows [r0, r0 + m_loc) that U_loc holds (pinv.py:75's U^T Y,
// one row shard of it; the shards' W sum to the full product).  Y is CSR in original row order.
void pinv_project_csr(fpi_context* h, int64_t r0, int64_t m_loc, int64_t r, const double* U_loc,
                      const int64_t* row_fwd, int64_t m, int64_t L, int64_t nnz, const int64_t* y_ptr,
                      const int32_t* y_idx, const double* y_val, double* W) {
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  if (L == 0 || r == 0) return;
  FPI_CUDA(cudaMemsetAsync(W, 0, sizeof(double) * L * r, s));
  if (nnz == 0 || m_loc == 0) return;
  CubTemp tmp(s);
  Scratch<int32_t> rows(nnz, s), rrows(nnz, s);
  expand_rows(h, m, y_ptr, rows);
  k_remap_rows_i32<<<grid_for(nnz, 256, G), 256, 0, s>>>(nnz, rows, row_fwd, rrows);
  const int32_t* major = y_idx;
  const int32_t* minor = rrows.get();
  const double* vals = y_val;
  int64_t cnt = nnz;
  Scratch<int32_t> flag, ids, sel_major, sel_minor;
  Scratch<int> dcnt;
  Scratch<double> sel_val;
  if (r0 > 0 || m_loc < m) {
    flag.alloc(nnz, s);
    ids.alloc(nnz, s);
    sel_major.alloc(nnz, s);
    sel_minor.alloc(nnz, s);
    sel_val.alloc(nnz, s);
    dcnt.alloc(1, s);
    k_rows_in_range<<<grid_for(nnz, 256, G), 256, 0, s>>>(nnz, rrows, r0, m_loc, flag);
    k_iota_i32<<<grid_for(nnz, 256, G), 256, 0, s>>>(ids, nnz);
    Scratch<int32_t> picked(nnz, s);
    select_if(tmp, ids.get(), picked.get(), dcnt.get(), nnz, FlagSet{flag.get()}, s);
    cnt = host_read(dcnt.get(), s);
    if (cnt == 0) return;
    k_gather_triplets<<<grid_for(cnt, 256, G), 256, 0, s>>>(cnt, picked, y_idx, rrows, y_val, r0, sel_major, sel_minor,
                                                             sel_val);
    FPI_LAUNCH_CHECK();
    major = sel_major.get();
    minor = sel_minor.get();
    vals = sel_val.get();
  }
  Scratch<int64_t> yt_ptr(L + 1, s);
  Scratch<int32_t> yt_idx(cnt, s);
  Scratch<double> yt_val(cnt, s);
  build_csr(h, tmp, cnt, major, minor, vals, L, m_loc, yt_ptr, yt_idx, yt_val);
  spmm(h, L, m_loc, r, yt_ptr, yt_idx, yt_val, nullptr, 1.0, U_loc, r, 0.0, W, r);
  note_launch(h, 2);
}

// Z (n x L, original column order) = V diag(sigma+) W^T from the summed W (pinv.py:81); W is scaled in place.
void pinv_lift(fpi_context* h, int64_t n, int64_t r, const double* sdag, const double* Vt, const int64_t* col_fwd,
               int64_t L, double* W, double* Z) {
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  if (n == 0 || L == 0) return;
  if (r == 0) {
    FPI_CUDA(cudaMemsetAsync(Z, 0, sizeof(double) * n * L, s));
    return;
  }
  scale_cols(h, L, r, W, r, sdag, false);
  // Vt's columns in original order first (r x n), so the GEMM writes Z's rows in place
  Scratch<double> Vg(r * n, s);
  k_gather_cols<<<grid_for(r * n, 256, G), 256, 0, s>>>(r, n, Vt, col_fwd, Vg);
  FPI_LAUNCH_CHECK();
  note_launch(h);
  gemm(h, true, true, n, L, r, 1.0, Vg, n, W, r, 0.0, Z, L);
}

void pinv_apply_csr(fpi_context* h, int64_t m, int64_t n, int64_t r, const double* U, const double* sdag,
                    const double* Vt, const int64_t* row_fwd, const int64_t* col_fwd, int64_t L, int64_t nnz,
                    const int64_t* y_ptr, const int32_t* y_idx, const double* y_val, double* Z) {
  cudaStream_t s = h->stream;
  if (n == 0 || L == 0) return;
  if (r == 0) {
    FPI_CUDA(cudaMemsetAsync(Z, 0, sizeof(double) * n * L, s));
    return;
  }
  Scratch<double> W(L * r, s);
  pinv_project_csr(h, 0, m, r, U, row_fwd, m, L, nnz, y_ptr, y_idx, y_val, W);
  pinv_lift(h, n, r, sdag, Vt, col_fwd, L, W, Z);
}

// pinv_apply_csr straight into host memory: the lift Z = V diag(sigma+) W^T runs in row chunks of
// the original order, each chunk's device->host copy (copy stream) overlapping the next chunk's
// GEMM.  h_Z must be page-locked for the copies to be asynchronous.
void pinv_apply_csr_host(fpi_context* h, int64_t m, int64_t n, int64_t r, const double* U, const double* sdag,
                         const double* Vt, const int64_t* row_fwd, const int64_t* col_fwd, int64_t L, int64_t nnz,
                         const int64_t* y_ptr, const int32_t* y_idx, const double* y_val, double* h_Z) {
  cudaStream_t s = h->stream;
  if (n == 0 || L == 0) return;
  if (r == 0) {
    memset(h_Z, 0, sizeof(double) * n * L);
    return;
  }
  if (!h->copy_stream) FPI_CUDA(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  for (auto& e : h->copy_ev)
    if (!e) FPI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  Scratch<double> W(L * r, s), Vg(r * n, s);
  pinv_project_csr(h, 0, m, r, U, row_fwd, m, L, nnz, y_ptr, y_idx, y_val, W);
  scale_cols(h, L, r, W, r, sdag, false);
  k_gather_cols<<<grid_for(r * n, 256, (int64_t)h->num_sms * 16), 256, 0, s>>>(r, n, Vt, col_fwd, Vg);
  FPI_LAUNCH_CHECK();
  note_launch(h);
  // ~64 MB chunks, at least 256 rows, double-buffered on the device
  int64_t rows = (int64_t)((64ll << 20) / (8 * L));
  if (rows < 256) rows = 256;
  rows &= ~(int64_t)1;  // even chunk offsets keep Vg + a 16-byte aligned (the GEMM's 16-byte / TMA tiles)
  if (rows > n) rows = n;
  Scratch<double> buf(2 * rows * L, s);
  cudaStream_t cs = h->copy_stream;
  cudaEvent_t* ready = h->copy_ev;      // [0], [1]: chunk computed
  cudaEvent_t* drained = h->copy_ev + 2;  // [2], [3]: buffer copied out
  int64_t c = 0;
  // the copies are the longer pole (PCIe), so the first one should start early: the chunks grow
  // 1/8, 1/4, 1/2, 1, 1, ... of the buffer size
  int64_t step = rows / 8 >= 256 ? (rows / 8) & ~(int64_t)1 : rows;
  for (int64_t a = 0; a < n; a += step, step = (2 * step < rows ? 2 * step : rows), ++c) {
    const int64_t nr = (n - a < step) ? n - a : step;
    const int sl = (int)(c & 1);
    double* d = buf.get() + sl * rows * L;
    if (c >= 2) FPI_CUDA(cudaStreamWaitEvent(s, drained[sl], 0));
    gemm(h, true, true, nr, L, r, 1.0, Vg.get() + a, n, W, r, 0.0, d, L);
    FPI_CUDA(cudaEventRecord(ready[sl], s));
    FPI_CUDA(cudaStreamWaitEvent(cs, ready[sl], 0));
    FPI_CUDA(cudaMemcpyAsync(h_Z + a * L, d, sizeof(double) * nr * L, cudaMemcpyDeviceToHost, cs));
    FPI_CUDA(cudaEventRecord(drained[sl], cs));
  }
  // the compute stream owns the scratch: it must not be freed before the last copy
  FPI_CUDA(cudaStreamWaitEvent(s, drained[0], 0));
  FPI_CUDA(cudaStreamWaitEvent(s, drained[1], 0));
  FPI_CUDA(cudaStreamSynchronize(s));
}

void pinv_apply_dense(fpi_context* h, int64_t m, int64_t n, int64_t r, const double* U, const double* sdag,
                      const double* Vt, const int64_t* row_fwd, const int64_t* col_fwd, int64_t L, const double* Y,
                      int64_t ldy, double* Z) {
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  if (n == 0 || L == 0) return;
  if (r == 0) {
    FPI_CUDA(cudaMemsetAsync(Z, 0, sizeof(double) * n * L, s));
    return;
  }
  Scratch<double> Yr(m * L, s), W(r * L, s), Vg(r * n, s);
  k_scatter_rows<<<grid_for(m * L, 256, G), 256, 0, s>>>(m, L, Y, ldy, row_fwd, Yr, L);
  gemm(h, true, false, r, L, m, 1.0, U, r, Yr, L, 0.0, W, L);
  scale_rows(h, r, L, W, L, sdag);
  k_gather_cols<<<grid_for(r * n, 256, G), 256, 0, s>>>(r, n, Vt, col_fwd, Vg);
  gemm(h, true, false, n, L, r, 1.0, Vg, n, W, L, 0.0, Z, L);
  FPI_LAUNCH_CHECK();
  note_launch(h, 2);
}

}  // namespace fpi

// ---- C ABI -----------------------------------------------------------------
extern "C" int fpi_dense_svd(fpi_handle h, int64_t p, int64_t q, const double* d_M, int64_t ldm, int64_t rank,
                             double* d_U, double* d_sigma, double* d_Vt) {
  FPI_API_BEGIN(h)
  h->diag = fpi_svd_diag{};
  h->diag.engine = 2;
  FPI_REQUIRE(p * q <= 100000000LL, FPI_ECAPACITY,
              "dense SVD of a " + std::to_string(p) + "x" + std::to_string(q) +
                  " matrix exceeds the 100000000-entry guard");
  fpi::dense_svd(h, p, q, d_M, ldm, rank, d_U, d_sigma, d_Vt, &h->diag);
  FPI_API_END(h)
}

// ---- building blocks of the row-sharded randomized SVD (sharded.py) ----
extern "C" int fpi_gram(fpi_handle h, int trans_a, int64_t n, int64_t k, const double* d_A, int64_t lda, double* d_C,
                        int64_t ldc) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(n >= 0 && k >= 0, FPI_EDOMAIN, "negative Gram dimension");
  // C = op(A) op(A)^T, op(A) n x k: the symmetric (SYRK-style) product of svd.py:134's CholeskyQR
  fpi::gemm(h, trans_a != 0, trans_a == 0, n, n, k, 1.0, d_A, lda, d_A, lda, 0.0, d_C, ldc, /*sym=*/true);
  FPI_API_END(h)
}

extern "C" int fpi_orth_factor(fpi_handle h, int64_t k, const double* d_G, double* d_Linv, double* h_cond) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(k >= 1, FPI_EDOMAIN, "orth_factor needs k >= 1");
  fpi_svd_diag dg{};
  fpi::orth_factor(h, k, d_G, d_Linv, &dg);
  h->diag.cond_estimate = dg.cond_estimate;
  h->diag.cholqr_passes = dg.cholqr_passes;
  if (h_cond) *h_cond = dg.cond_estimate;
  FPI_API_END(h)
}

extern "C" int fpi_scale_rows(fpi_handle h, int64_t rows, int64_t cols, double* d_A, int64_t lda,
                              const double* d_scale) {
  FPI_API_BEGIN(h)
  if (rows > 0 && cols > 0) fpi::scale_rows(h, rows, cols, d_A, lda, d_scale);
  FPI_API_END(h)
}

extern "C" int fpi_canonical_signs(fpi_handle h, int64_t r, int64_t p, int64_t q, double* d_U, int64_t ldu,
                                   double* d_Vt, int64_t ldv) {
  FPI_API_BEGIN(h)
  if (r > 0) fpi::canonical_signs(h, r, p, q, d_U, ldu, d_Vt, ldv);
  FPI_API_END(h)
}

extern "C" int fpi_transpose(fpi_handle h, int64_t rows, int64_t cols, const double* d_A, int64_t lda, double* d_At,
                             int64_t ldat) {
  FPI_API_BEGIN(h)
  if (rows > 0 && cols > 0) fpi::transpose(h, rows, cols, d_A, lda, d_At, ldat);
  FPI_API_END(h)
}

extern "C" int fpi_randomized_svd(fpi_handle h, int64_t p, int64_t q, const int64_t* a_ptr, const int32_t* a_idx,
                                  const double* a_val, const int64_t* at_ptr, const int32_t* at_idx,
                                  const double* at_val, int64_t rank, int64_t seed, double* d_U, double* d_sigma,
                                  double* d_Vt) {
  FPI_API_BEGIN(h)
  h->diag = fpi_svd_diag{};
  fpi::InnerOp op;
  op.p = p;
  op.q = q;
  op.s_ptr = a_ptr;
  op.s_idx = a_idx;
  op.s_val = a_val;
  op.st_ptr = at_ptr;
  op.st_idx = at_idx;
  op.st_val = at_val;
  op.s_nnz = p ? fpi::host_read(a_ptr + p, h->stream) : 0;
  fpi::randomized_svd(h, op, rank, seed, d_U, d_sigma, d_Vt, &h->diag);
  FPI_API_END(h)
}

extern "C" int fpi_row_update(fpi_handle h, int64_t m1, int64_t n1, int64_t rank11, const double* sigma11,
                              const int64_t* u_ptr, const int32_t* u_idx, const double* u_val, const int64_t* v_ptr,
                              const int32_t* v_idx, const double* v_val, int64_t m2, const int64_t* a_ptr,
                              const int32_t* a_idx, const double* a_val, int64_t s, double thr, int64_t seed,
                              double* d_U, double* d_sigma, double* d_Vt, int32_t* h_engine) {
  FPI_API_BEGIN(h)
  h->diag = fpi_svd_diag{};
  int eng = 0;
  fpi::row_update(h, m1, n1, rank11, sigma11, u_ptr, u_idx, u_val, v_ptr, v_idx, v_val, m2, a_ptr, a_idx, a_val, s,
                  thr, seed, d_U, d_sigma, d_Vt, &eng);
  if (h_engine) *h_engine = eng;
  FPI_API_END(h)
}

extern "C" int fpi_column_update(fpi_handle h, int64_t m, int64_t s_prev, int64_t n1, const double* U_prev,
                                 const double* sigma_prev, const double* Vt_prev, int64_t n2, const int64_t* t_ptr,
                                 const int32_t* t_idx, const double* t_val, const int64_t* tt_ptr,
                                 const int32_t* tt_idx, const double* tt_val, int64_t r, double thr, int64_t seed,
                                 double* d_U, double* d_sigma, double* d_Vt, int32_t* h_engine) {
  FPI_API_BEGIN(h)
  h->diag = fpi_svd_diag{};
  int eng = 0;
  fpi::column_update(h, m, s_prev, n1, U_prev, sigma_prev, Vt_prev, n2, t_ptr, t_idx, t_val, tt_ptr, tt_idx, tt_val,
                     r, thr, seed, d_U, d_sigma, d_Vt, &eng);
  if (h_engine) *h_engine = eng;
  FPI_API_END(h)
}

extern "C" int fpi_pinv_assemble(fpi_handle h, int64_t r, const double* d_sigma, int64_t p, int64_t q,
                                 double cutoff, double* d_sigma_dagger, double* h_tol, int32_t* h_all_filtered) {
  FPI_API_BEGIN(h)
  int af = 0;
  double tol = 0;
  fpi::pinv_assemble(h, r, d_sigma, p, q, cutoff, d_sigma_dagger, &tol, &af);
  if (h_tol) *h_tol = tol;
  if (h_all_filtered) *h_all_filtered = af;
  FPI_API_END(h)
}

extern "C" int fpi_unfold(fpi_handle h, int64_t m, int64_t n, int64_t r, const double* d_U, const double* d_Vt,
                          const int64_t* d_row_fwd, const int64_t* d_col_fwd, double* d_V_out, double* d_Ut_out) {
  FPI_API_BEGIN(h)
  fpi::unfold_transpose(h, m, n, r, d_U, d_Vt, d_row_fwd, d_col_fwd, d_V_out, d_Ut_out);
  FPI_API_END(h)
}

extern "C" int fpi_pinv_apply_csr(fpi_handle h, int64_t m, int64_t n, int64_t r, const double* d_U,
                                  const double* d_sigma_dagger, const double* d_Vt, const int64_t* d_row_fwd,
                                  const int64_t* d_col_fwd, int64_t L, int64_t nnz, const int64_t* y_ptr,
                                  const int32_t* y_idx, const double* y_val, double* d_Z) {
  FPI_API_BEGIN(h)
  fpi::pinv_apply_csr(h, m, n, r, d_U, d_sigma_dagger, d_Vt, d_row_fwd, d_col_fwd, L, nnz, y_ptr, y_idx, y_val, d_Z);
  FPI_API_END(h)
}

extern "C" int fpi_pinv_apply_csr_host(fpi_handle h, int64_t m, int64_t n, int64_t r, const double* d_U,
                                       const double* d_sigma_dagger, const double* d_Vt, const int64_t* d_row_fwd,
                                       const int64_t* d_col_fwd, int64_t L, int64_t nnz, const int64_t* y_ptr,
                                       const int32_t* y_idx, const double* y_val, double* h_Z) {
  FPI_API_BEGIN(h)
  fpi::pinv_apply_csr_host(h, m, n, r, d_U, d_sigma_dagger, d_Vt, d_row_fwd, d_col_fwd, L, nnz, y_ptr, y_idx, y_val,
                           h_Z);
  FPI_API_END(h)
}

extern "C" int fpi_pinv_project_csr(fpi_handle h, int64_t r0, int64_t m_loc, int64_t r, const double* d_U_loc,
                                    const int64_t* d_row_fwd, int64_t m, int64_t L, int64_t nnz, const int64_t* y_ptr,
                                    const int32_t* y_idx, const double* y_val, double* d_W) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(r0 >= 0 && m_loc >= 0 && r0 + m_loc <= m, FPI_EDOMAIN, "row shard out of range");
  fpi::pinv_project_csr(h, r0, m_loc, r, d_U_loc, d_row_fwd, m, L, nnz, y_ptr, y_idx, y_val, d_W);
  FPI_API_END(h)
}

extern "C" int fpi_pinv_lift(fpi_handle h, int64_t n, int64_t r, const double* d_sigma_dagger, const double* d_Vt,
                             const int64_t* d_col_fwd, int64_t L, double* d_W, double* d_Z) {
  FPI_API_BEGIN(h)
  fpi::pinv_lift(h, n, r, d_sigma_dagger, d_Vt, d_col_fwd, L, d_W, d_Z);
  FPI_API_END(h)
}

extern "C" int fpi_pinv_apply_dense(fpi_handle h, int64_t m, int64_t n, int64_t r, const double* d_U,
                                    const double* d_sigma_dagger, const double* d_Vt, const int64_t* d_row_fwd,
                                    const int64_t* d_col_fwd, int64_t L, const double* d_Y, int64_t ldy,
                                    double* d_Z) {
  FPI_API_BEGIN(h)
  fpi::pinv_apply_dense(h, m, n, r, d_U, d_sigma_dagger, d_Vt, d_row_fwd, d_col_fwd, L, d_Y, ldy, d_Z);
  FPI_API_END(h)
}
