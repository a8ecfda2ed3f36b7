// Dense FP64 building blocks for the SVD engines:
//   * Cholesky (blocked, right-looking; trailing updates on the DMMA GEMM) and
//     lower-triangular solves with many right-hand sides -- CholeskyQR of the
//     sketch (replaces LAPACK dgeqrf+dorgqr, svd.py:134),
//   * (the symmetric eigensolver lives in jacobi.cu),
//   * small helpers: transpose, column norms, scaling, canonical signs.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "capi_guard.cuh"
#include "cub_util.cuh"
#include "gemm.cuh"
#include "linalg.cuh"
#include "instrument.cuh"

namespace cg = cooperative_groups;

namespace fpi {
namespace {

constexpr int NB = 32;  // Cholesky / TRSM panel width

// ---- Cholesky ------------------------------------------------------------
__global__ void k_potrf_diag(double* A, int64_t lda, int jb, int* info, int64_t j0) {
  __shared__ double S[NB][NB + 1];
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) S[e / jb][e % jb] = A[(e / jb) * lda + (e % jb)];
  __syncthreads();
  for (int k = 0; k < jb; ++k) {
    if (threadIdx.x == 0) {
      double d = S[k][k];
      if (!(d > 0.0)) {
        atomicCAS(info, 0, (int)(j0 + k + 1));
        d = 1e-300;
      }
      S[k][k] = sqrt(d);
    }
    __syncthreads();
    for (int i = k + 1 + threadIdx.x; i < jb; i += blockDim.x) S[i][k] /= S[k][k];
    __syncthreads();
    for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
      int i = e / jb, j = e % jb;
      if (j > k && i >= j) S[i][j] -= S[i][k] * S[j][k];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    int i = e / jb, j = e % jb;
    A[i * lda + j] = (i >= j) ? S[i][j] : 0.0;
  }
}

// rows below the diagonal block: x L11^T = a  (forward substitution), one thread per row
__global__ void k_trsm_panel(double* A, int64_t lda, int64_t j0, int jb, int64_t n) {
  __shared__ double L[NB][NB + 1];
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) L[e / jb][e % jb] = A[(j0 + e / jb) * lda + j0 + e % jb];
  __syncthreads();
  for (int64_t r = j0 + jb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double x[NB];
    double* a = A + r * lda + j0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      if (k < jb) {
        double v = a[k];
        for (int i = 0; i < k; ++i) v -= x[i] * L[k][i];
        x[k] = v / L[k][k];
      }
    }
#pragma unroll
    for (int k = 0; k < NB; ++k)
      if (k < jb) a[k] = x[k];
  }
}

// X[j0:j0+jb, :] = L_jj^{-1} X[j0:j0+jb, :]   one thread per right-hand-side column
__global__ void k_trsm_diag(const double* L, int64_t ldl, int64_t j0, int jb, double* X, int64_t ldx, int64_t nrhs) {
  __shared__ double S[NB][NB + 1];
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) S[e / jb][e % jb] = L[(j0 + e / jb) * ldl + j0 + e % jb];
  __syncthreads();
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nrhs; c += (int64_t)gridDim.x * blockDim.x) {
    double x[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      if (k < jb) {
        double v = X[(j0 + k) * ldx + c];
        for (int i = 0; i < k; ++i) v -= S[k][i] * x[i];
        x[k] = v / S[k][k];
      }
    }
#pragma unroll
    for (int k = 0; k < NB; ++k)
      if (k < jb) X[(j0 + k) * ldx + c] = x[k];
  }
}

__global__ void k_set_identity(int64_t n, double* A, int64_t lda) {
  FPI_GRID_STRIDE(e, n * n) {
    int64_t i = e / n, j = e - i * n;
    A[i * lda + j] = i == j ? 1.0 : 0.0;
  }
}

// ---- helpers ------------------------------------------------------------
__global__ void k_transpose(int64_t M, int64_t N, const double* __restrict__ A, int64_t lda, double* __restrict__ B,
                            int64_t ldb) {
  __shared__ double t[32][33];
  for (int64_t by = blockIdx.y; by * 32 < M; by += gridDim.y)
    for (int64_t bx = blockIdx.x; bx * 32 < N; bx += gridDim.x) {
      for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        int64_t r = by * 32 + i, c = bx * 32 + threadIdx.x;
        t[i][threadIdx.x] = (r < M && c < N) ? A[r * lda + c] : 0.0;
      }
      __syncthreads();
      for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        int64_t r = bx * 32 + i, c = by * 32 + threadIdx.x;
        if (r < N && c < M) B[r * ldb + c] = t[threadIdx.x][i];
      }
      __syncthreads();
    }
}

// column sums of squares, deterministic: one CTA per column group, fixed-order tree
__global__ void k_col_sumsq(int64_t M, int64_t N, const double* __restrict__ A, int64_t lda, double* __restrict__ out) {
  // blockDim (32, 8): x = column within group, y = row stripe
  __shared__ double part[8][33];
  int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  double s = 0.0;
  if (c < N)
    for (int64_t r = threadIdx.y; r < M; r += 8) {
      double v = A[r * lda + c];
      s = fma(v, v, s);
    }
  part[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && c < N) {
    double t = 0.0;
    for (int y = 0; y < 8; ++y) t += part[y][threadIdx.x];
    out[c] = t;
  }
}

// rows [chunk * M / chunks, (chunk + 1) * M / chunks) of 32 columns -> part[chunk][col]
__global__ void k_col_sumsq_part(int64_t M, int64_t N, const double* __restrict__ A, int64_t lda, int64_t chunks,
                                 double* __restrict__ part) {
  __shared__ double ps[8][33];
  const int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int64_t r0 = M * blockIdx.y / chunks, r1 = M * (blockIdx.y + 1) / chunks;
  double sacc = 0.0;
  if (c < N)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      const double v = A[r * lda + c];
      sacc = fma(v, v, sacc);
    }
  ps[threadIdx.y][threadIdx.x] = sacc;
  __syncthreads();
  if (threadIdx.y == 0 && c < N) {
    double t = 0.0;
    for (int y = 0; y < 8; ++y) t += ps[y][threadIdx.x];
    part[blockIdx.y * N + c] = t;
  }
}

__global__ void k_sum_parts(int64_t N, int64_t chunks, const double* __restrict__ part, double* __restrict__ out) {
  FPI_GRID_STRIDE(c, N) {
    double t = 0.0;
    for (int64_t k = 0; k < chunks; ++k) t += part[k * N + c];
    out[c] = t;
  }
}

__global__ void k_scale_cols(int64_t M, int64_t N, double* A, int64_t lda, const double* s, int mode) {
  // mode 0: multiply by s[j]; 1: divide by s[j] (0 where s == 0)
  FPI_GRID_STRIDE(e, M * N) {
    int64_t i = e / N, j = e - i * N;
    double f = s[j];
    A[i * lda + j] = mode == 0 ? A[i * lda + j] * f : (f != 0.0 ? A[i * lda + j] / f : 0.0);
  }
}

__global__ void k_scale_rows(int64_t M, int64_t N, double* A, int64_t lda, const double* s) {
  FPI_GRID_STRIDE(e, M * N) {
    int64_t i = e / N, j = e - i * N;
    A[i * lda + j] *= s[i];
  }
}

// Canonical sign per singular triplet: the largest-|.| entry of the right
// vector (row j of Vt, length q) is made positive (ties -> lowest index);
// the matching left vector (column j of U) flips with it.
__global__ void k_canon_sign(int64_t r, int64_t q, double* Vt, int64_t ldvt, double* sign) {
  __shared__ double best[32];
  __shared__ int64_t bidx[32];
  for (int64_t j = blockIdx.x; j < r; j += gridDim.x) {
    double bv = -1.0;
    int64_t bi = 0;
    for (int64_t c = threadIdx.x; c < q; c += blockDim.x) {
      double a = fabs(Vt[j * ldvt + c]);
      if (a > bv) { bv = a; bi = c; }
    }
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { best[w] = bv; bidx[w] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
        if (best[k] > best[0] || (best[k] == best[0] && bidx[k] < bidx[0])) { best[0] = best[k]; bidx[0] = bidx[k]; }
    }
    __syncthreads();
    const bool flip = q > 0 && Vt[j * ldvt + bidx[0]] < 0.0;
    __syncthreads();
    if (flip)
      for (int64_t c = threadIdx.x; c < q; c += blockDim.x) Vt[j * ldvt + c] = -Vt[j * ldvt + c];
    if (threadIdx.x == 0) sign[j] = flip ? -1.0 : 1.0;
  }
}

// U[:, j] *= sign[j], row-major and coalesced (the left vectors follow their right vectors)
__global__ void k_apply_col_signs(int64_t p, int64_t r, double* U, int64_t ldu, const double* sign) {
  FPI_GRID_STRIDE(e, p * r) {
    const int64_t i = e / r, j = e - i * r;
    const double sg = sign[j];
    if (sg < 0.0) U[i * ldu + j] = -U[i * ldu + j];
  }
}

}  // namespace

void cholesky_lower(fpi_context* h, int64_t n, double* A, int64_t lda, int* h_info) {
  cudaStream_t s = h->stream;
  Scratch<int> info(1, s);
  FPI_CUDA(cudaMemsetAsync(info.get(), 0, sizeof(int), s));
  for (int64_t j = 0; j < n; j += NB) {
    int jb = (int)(n - j < NB ? n - j : NB);
    k_potrf_diag<<<1, 256, 0, s>>>(A + j * lda + j, lda, jb, info, j);
    if (j + jb < n) {
      int64_t rows = n - j - jb;
      k_trsm_panel<<<grid_for(rows, 128, h->num_sms * 4), 128, 0, s>>>(A, lda, j, jb, n);
      gemm(h, false, true, rows, rows, jb, -1.0, A + (j + jb) * lda + j, lda, A + (j + jb) * lda + j, lda, 1.0,
           A + (j + jb) * lda + j + jb, lda, /*sym=*/true);
    }
    note_launch(h, 2);
  }
  FPI_LAUNCH_CHECK();
  *h_info = host_read(info.get(), s);
}

void trsm_lower_left(fpi_context* h, int64_t n, const double* L, int64_t ldl, double* X, int64_t ldx, int64_t nrhs) {
  cudaStream_t s = h->stream;
  for (int64_t j = 0; j < n; j += NB) {
    int jb = (int)(n - j < NB ? n - j : NB);
    k_trsm_diag<<<grid_for(nrhs, 128, h->num_sms * 4), 128, 0, s>>>(L, ldl, j, jb, X, ldx, nrhs);
    if (j + jb < n)
      gemm(h, false, false, n - j - jb, nrhs, jb, -1.0, L + (j + jb) * ldl + j, ldl, X + j * ldx, ldx, 1.0,
           X + (j + jb) * ldx, ldx);
    note_launch(h);
  }
  FPI_LAUNCH_CHECK();
}

void lower_inverse(fpi_context* h, int64_t n, const double* L, int64_t ldl, double* Linv, int64_t ldi) {
  k_set_identity<<<grid_for(n * n, 256, h->num_sms * 16), 256, 0, h->stream>>>(n, Linv, ldi);
  note_launch(h);
  trsm_lower_left(h, n, L, ldl, Linv, ldi, n);
}

void transpose(fpi_context* h, int64_t M, int64_t N, const double* A, int64_t lda, double* B, int64_t ldb) {
  if (M <= 0 || N <= 0) return;
  dim3 blk(32, 8);
  int64_t gx = (N + 31) / 32, gy = (M + 31) / 32;
  dim3 grd((unsigned)(gx < 65535 ? gx : 65535), (unsigned)(gy < 65535 ? gy : 65535));
  k_transpose<<<grd, blk, 0, h->stream>>>(M, N, A, lda, B, ldb);
  FPI_LAUNCH_CHECK();
  note_launch(h);
}

void col_sumsq(fpi_context* h, int64_t M, int64_t N, const double* A, int64_t lda, double* out) {
  if (N <= 0) return;
  const int64_t groups = (N + 31) / 32;
  // enough row chunks to fill the GPU (one CTA per (column group, chunk)); partial sums are
  // reduced in chunk order, so the result does not depend on scheduling
  int64_t chunks = ((int64_t)h->num_sms * 4 + groups - 1) / groups;
  const int64_t max_chunks = (M + 255) / 256;
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks <= 1) {
    k_col_sumsq<<<(unsigned)groups, dim3(32, 8), 0, h->stream>>>(M, N, A, lda, out);
  } else {
    Scratch<double> part(chunks * N, h->stream);
    k_col_sumsq_part<<<dim3((unsigned)groups, (unsigned)chunks), dim3(32, 8), 0, h->stream>>>(M, N, A, lda, chunks,
                                                                                              part);
    k_sum_parts<<<grid_for(N, 256, (int64_t)h->num_sms * 4), 256, 0, h->stream>>>(N, chunks, part, out);
    note_launch(h);
  }
  FPI_LAUNCH_CHECK();
  note_launch(h);
}

void scale_cols(fpi_context* h, int64_t M, int64_t N, double* A, int64_t lda, const double* s, bool divide) {
  if (M <= 0 || N <= 0) return;
  k_scale_cols<<<grid_for(M * N, 256, h->num_sms * 16), 256, 0, h->stream>>>(M, N, A, lda, s, divide ? 1 : 0);
  FPI_LAUNCH_CHECK();
  note_launch(h);
}

void scale_rows(fpi_context* h, int64_t M, int64_t N, double* A, int64_t lda, const double* s) {
  if (M <= 0 || N <= 0) return;
  k_scale_rows<<<grid_for(M * N, 256, h->num_sms * 16), 256, 0, h->stream>>>(M, N, A, lda, s);
  FPI_LAUNCH_CHECK();
  note_launch(h);
}

// The sign rule on the right vectors alone: Vt's rows flipped, the signs left in sign_out (r) for the
// caller to fold into whatever produces the left vectors.
void canonical_signs_vt(fpi_context* h, int64_t r, int64_t q, double* Vt, int64_t ldvt, double* sign_out) {
  if (r <= 0) return;
  k_canon_sign<<<(unsigned)(r < 4096 ? r : 4096), 256, 0, h->stream>>>(r, q, Vt, ldvt, sign_out);
  FPI_LAUNCH_CHECK();
  note_launch(h);
}

void canonical_signs(fpi_context* h, int64_t r, int64_t p, int64_t q, double* U, int64_t ldu, double* Vt,
                     int64_t ldvt) {
  if (r <= 0) return;
  Scratch<double> sign(r, h->stream);
  k_canon_sign<<<(unsigned)(r < 4096 ? r : 4096), 256, 0, h->stream>>>(r, q, Vt, ldvt, sign);
  if (p > 0)
    k_apply_col_signs<<<grid_for(p * r, 256, (int64_t)h->num_sms * 16), 256, 0, h->stream>>>(p, r, U, ldu, sign);
  FPI_LAUNCH_CHECK();
  note_launch(h, 2);
}

}  // namespace fpi

extern "C" int fpi_cholesky(fpi_handle h, int64_t n, double* d_A, int64_t lda) {
  FPI_API_BEGIN(h)
  int info = 0;
  fpi::cholesky_lower(h, n, d_A, lda, &info);
  FPI_REQUIRE(info == 0, FPI_ENUMERIC, "matrix is not positive definite (pivot " + std::to_string(info) + ")");
  FPI_API_END(h)
}

