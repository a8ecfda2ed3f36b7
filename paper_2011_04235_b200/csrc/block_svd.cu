// Block-diagonal SVD of the spoke region A11 (svd.py:141-193).
//
// Every non-degenerate span (h x w) gets keep = ceil(alpha * min(h, w))
// leading singular triplets; degenerate spans (h == 0 or w == 0) only advance
// the offsets.  Output is the reference's block-sparse layout as CSR:
//   U11  (m1 x rank11): row i of block b holds keep_b entries at columns
//        rank_off_b .. rank_off_b + keep_b - 1,
//   Vt11 (rank11 x n1): row rank_off_b + t holds w_b entries at columns
//        col_start_b .. col_start_b + w_b - 1,
//   sigma in block order (unsorted across blocks, sorted within a block).
//
// Tiers:
//   * small  -- the block (oriented so it has c = min(h, w) columns) plus its
//     c x c rotation fit in shared memory: one CTA per block runs a one-sided
//     (Hestenes) Jacobi SVD with round-robin column pairs, one warp per pair,
//     warp-shuffle reductions for the 2x2 Gram entries.  Blocks with c == 1
//     (most of them) reduce to a normalisation.
//   * large  -- everything else goes through the dense Gram-refined SVD
//     (svd_engine.cu), one block at a time.
// Each triplet gets the canonical sign (largest |.| entry of the right vector
// positive) and zero singular values get an orthonormal completion.
#include <algorithm>

#include "common.cuh"
#include "capi_guard.cuh"
#include "cub_util.cuh"
#include "svd_engine.cuh"
#include "instrument.cuh"

namespace fpi {
namespace {

constexpr int BT = 256;  // threads per block-SVD CTA
constexpr int64_t TINY_DOUBLES = 3000;  // blocks needing <= 24 KB smem run many CTAs per SM
#ifndef FPI_GRAM_MIN_DIM
#define FPI_GRAM_MIN_DIM 48
#endif
constexpr int64_t GRAM_MIN_DIM = FPI_GRAM_MIN_DIM;

struct BlockMeta {
  int64_t* keep;      // per span
  int64_t* rank_off;  // exclusive scan of keep
  int64_t* u_off;     // exclusive scan of h * keep
  int64_t* v_off;     // exclusive scan of keep * w
};

__global__ void k_plan(int64_t nspans, const int64_t* __restrict__ spans, double alpha, int64_t* keep,
                       int64_t* uk, int64_t* vk, int64_t* large_flag, int64_t smem_doubles) {
  FPI_GRID_STRIDE(b, nspans) {
    int64_t h = spans[4 * b + 1], w = spans[4 * b + 3];
    int64_t kp = 0;
    int64_t lg = 0;
    if (h > 0 && w > 0) {
      int64_t c = h < w ? h : w, r = h < w ? w : h;
      kp = (int64_t)ceil(alpha * (double)c);  // int(np.ceil(alpha * min(h, w))), svd.py:167
      int64_t cpad = c + (c & 1);
      const int64_t need = r * cpad + cpad * cpad + 4 * cpad;
      // blocks whose one-sided Jacobi chain would be long (min dimension >= GRAM_MIN_DIM: the chain
      // grows with c^2 sweeps-rounds and the kernel ends with its slowest CTA) join the batched Gram
      // path with the blocks that do not fit in shared memory
      lg = (need > smem_doubles || c >= GRAM_MIN_DIM) ? 1 : (need > TINY_DOUBLES ? 2 : 0);
    }
    keep[b] = kp;
    uk[b] = h * kp;
    vk[b] = kp * w;
    large_flag[b] = lg;
  }
}

// U11 / Vt11 CSR structure (values written by the SVD kernels)
__global__ void k_u_rows(int64_t nspans, const int64_t* __restrict__ spans, const int64_t* __restrict__ keep,
                         int64_t* __restrict__ row_cnt) {
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < nspans; b += nw) {
    int64_t rs = spans[4 * b], h = spans[4 * b + 1];
    for (int64_t i = lane; i < h; i += 32) row_cnt[rs + i] = keep[b];
  }
}

__global__ void k_structure(int64_t nspans, const int64_t* __restrict__ spans, const int64_t* __restrict__ keep,
                            const int64_t* __restrict__ rank_off, const int64_t* __restrict__ u_off,
                            const int64_t* __restrict__ v_off, int32_t* __restrict__ u_idx,
                            int64_t* __restrict__ vt_ptr, int32_t* __restrict__ vt_idx) {
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < nspans; b += nw) {
    int64_t h = spans[4 * b + 1], cs = spans[4 * b + 2], w = spans[4 * b + 3], kp = keep[b];
    if (kp == 0) continue;
    for (int64_t e = lane; e < h * kp; e += 32) u_idx[u_off[b] + e] = (int32_t)(rank_off[b] + e % kp);
    for (int64_t t = lane; t < kp; t += 32) vt_ptr[rank_off[b] + t] = v_off[b] + t * w;
    for (int64_t e = lane; e < kp * w; e += 32) vt_idx[v_off[b] + e] = (int32_t)(cs + e % w);
  }
}

// circle-method round robin: position pos of n (even) players in round `step`
__device__ __forceinline__ int rr_index(int pos, int step, int n) {
  return pos == 0 ? 0 : 1 + ((pos - 1 + step) % (n - 1));
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One CTA per small non-degenerate block.  smem: M (r x cpad, column-major: column j at M + j*r),
// V (cpad x cpad, column-major), norms / order scratch.
__global__ void __launch_bounds__(BT)
    k_block_svd_small(const int64_t* __restrict__ blist, int64_t nb, const int64_t* __restrict__ spans,
                      const int64_t* __restrict__ keep, const int64_t* __restrict__ rank_off,
                      const int64_t* __restrict__ u_off, const int64_t* __restrict__ v_off,
                      const int64_t* __restrict__ a_ptr, const int32_t* __restrict__ a_idx,
                      const double* __restrict__ a_val, double* __restrict__ sigma, double* __restrict__ u_val,
                      double* __restrict__ vt_val, int max_sweeps) {
  extern __shared__ double sm[];
  __shared__ int rotated;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = BT / 32;
  for (int64_t bi = blockIdx.x; bi < nb; bi += gridDim.x) {
    const int64_t b = blist[bi];
    const int64_t rs = spans[4 * b], h = spans[4 * b + 1], cs = spans[4 * b + 2], w = spans[4 * b + 3];
    const bool tr = h < w;                      // work on A^T so that rows >= cols
    const int r = (int)(tr ? w : h), c = (int)(tr ? h : w);
    const int cp = c + (c & 1);
    double* M = sm;                             // r x cp, column-major
    double* V = sm + (int64_t)r * cp;           // cp x cp, column-major
    double* nrm = V + cp * cp;                  // cp
    int* ord = (int*)(nrm + cp);                // cp
    for (int e = threadIdx.x; e < r * cp + cp * cp; e += BT) sm[e] = 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < cp; i += BT) V[i * cp + i] = 1.0;
    // scatter block entries: A row rs+i, col cs+j  ->  M[i][j] (or M[j][i] if transposed)
    for (int64_t i = warp; i < h; i += nwarps) {
      const int64_t pb = a_ptr[rs + i], pe = a_ptr[rs + i + 1];
      for (int64_t p = pb + lane; p < pe; p += 32) {
        const int64_t j = a_idx[p] - cs;
        if (!tr)
          M[j * r + i] = a_val[p];
        else
          M[i * r + j] = a_val[p];
      }
    }
    __syncthreads();
    // one-sided Jacobi sweeps over column pairs (round-robin over cp columns)
    if (c > 1) {
      for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        if (threadIdx.x == 0) rotated = 0;
        __syncthreads();
        for (int step = 0; step < cp - 1; ++step) {
          for (int k = warp; k < cp / 2; k += nwarps) {
            const int p = rr_index(k, step, cp), q = rr_index(cp - 1 - k, step, cp);
            double* mp = M + (int64_t)p * r;
            double* mq = M + (int64_t)q * r;
            double al = 0.0, be = 0.0, ga = 0.0;
            for (int i = lane; i < r; i += 32) {
              const double x = mp[i], y = mq[i];
              al = fma(x, x, al);
              be = fma(y, y, be);
              ga = fma(x, y, ga);
            }
            al = warp_sum(al);
            be = warp_sum(be);
            ga = warp_sum(ga);
            if (ga != 0.0 && fabs(ga) > 1e-15 * sqrt(al * be)) {
              const double zeta = (be - al) / (2.0 * ga);
              const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
              const double cc = 1.0 / sqrt(1.0 + t * t), ss = cc * t;
              for (int i = lane; i < r; i += 32) {
                const double x = mp[i], y = mq[i];
                mp[i] = cc * x - ss * y;
                mq[i] = ss * x + cc * y;
              }
              double* vp = V + (int64_t)p * cp;
              double* vq = V + (int64_t)q * cp;
              for (int i = lane; i < cp; i += 32) {
                const double x = vp[i], y = vq[i];
                vp[i] = cc * x - ss * y;
                vq[i] = ss * x + cc * y;
              }
              if (lane == 0) rotated = 1;
            }
          }
          __syncthreads();
        }
        if (!rotated) break;
        __syncthreads();
      }
    }
    // singular values = column norms; order descending (ties by index)
    for (int j = warp; j < cp; j += nwarps) {
      double s = 0.0;
      for (int i = lane; i < r; i += 32) s = fma(M[(int64_t)j * r + i], M[(int64_t)j * r + i], s);
      s = warp_sum(s);
      if (lane == 0) nrm[j] = j < c ? sqrt(s) : -1.0;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cp; j += BT) {
      int rk = 0;
      for (int k2 = 0; k2 < cp; ++k2) rk += (nrm[k2] > nrm[j]) || (nrm[k2] == nrm[j] && k2 < j);
      ord[rk] = j;
    }
    __syncthreads();
    const int64_t kp = keep[b];
    const double smax = nrm[ord[0]];
    const double null_tol = 2.220446049250313e-16 * (smax > 0 ? smax : 1.0) * (double)(r > c ? r : c);
    // emit the top kp triplets (one warp per triplet)
    for (int t = warp; t < kp; t += nwarps) {
      const int j = ord[t];
      const double s = nrm[j];
      const bool null_col = !(s > null_tol);
      const double* mj = M + (int64_t)j * r;
      const double* vj = V + (int64_t)j * cp;
      // left (length r) = mj / s ; right (length c) = vj   [oriented problem]
      // canonical sign from the block's RIGHT vector: vj if !tr, normalised mj if tr
      const double* rv = tr ? mj : vj;
      const int rn = tr ? r : c;
      double bv = -1.0;
      int bi2 = 0;
      for (int i = lane; i < rn; i += 32) {
        const double a = fabs(rv[i]);
        if (a > bv) { bv = a; bi2 = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi2, o);
        if (ov > bv || (ov == bv && oi < bi2)) { bv = ov; bi2 = oi; }
      }
      const double sgn = (rv[bi2] < 0.0) ? -1.0 : 1.0;
      if (lane == 0) sigma[rank_off[b] + t] = s;
      const double inv = null_col ? 0.0 : 1.0 / s;
      // U11 rows of this block: entry (i, t) at u_off + i*kp + t ;  Vt11 row t: v_off + t*w + j
      if (!tr) {
        for (int i = lane; i < h; i += 32) u_val[u_off[b] + (int64_t)i * kp + t] = sgn * mj[i] * inv;
        for (int i = lane; i < w; i += 32) vt_val[v_off[b] + (int64_t)t * w + i] = sgn * vj[i];
      } else {
        for (int i = lane; i < h; i += 32) u_val[u_off[b] + (int64_t)i * kp + t] = sgn * vj[i];
        for (int i = lane; i < w; i += 32) vt_val[v_off[b] + (int64_t)t * w + i] = sgn * mj[i] * inv;
      }
    }
    __syncthreads();
  }
}

// Orthonormal completion of null left/right vectors inside small blocks
// (sigma == 0): Gram-Schmidt of unit vectors against the block's other vectors.
__global__ void k_complete_null(const int64_t* __restrict__ blist, int64_t nb, const int64_t* __restrict__ spans,
                                const int64_t* __restrict__ keep, const int64_t* __restrict__ rank_off,
                                const int64_t* __restrict__ u_off, const int64_t* __restrict__ v_off,
                                const double* __restrict__ sigma, double* __restrict__ u_val,
                                double* __restrict__ vt_val) {
  // one thread per block (rare path, tiny blocks); the vector on the long side is completed
  for (int64_t bi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; bi < nb; bi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = blist[bi];
    const int64_t h = spans[4 * b + 1], w = spans[4 * b + 3], kp = keep[b];
    const double* sg = sigma + rank_off[b];
    double smax = kp ? sg[0] : 0.0;
    const double tol = 2.220446049250313e-16 * (smax > 0 ? smax : 1.0) * (double)(h > w ? h : w);
    for (int64_t t = 0; t < kp; ++t) {
      if (sg[t] > tol) continue;
      // complete U column t (length h, stride kp) if !transposed, else Vt row t (length w)
      const bool tr = h < w;
      const int64_t len = tr ? w : h;
      double* base = tr ? vt_val + v_off[b] : u_val + u_off[b];
      const int64_t stride = tr ? 1 : kp;    // element i of vector t
      const int64_t vstep = tr ? w : 1;      // start offset of vector t
      for (int64_t e = 0; e < len; ++e) {
        // candidate e_e minus projections on the other vectors
        for (int64_t i = 0; i < len; ++i) base[t * vstep + i * stride] = (i == e) ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass)
          for (int64_t o = 0; o < kp; ++o) {
            if (o == t || (o > t && sg[o] <= tol)) continue;
            double d = 0.0;
            for (int64_t i = 0; i < len; ++i) d += base[o * vstep + i * stride] * base[t * vstep + i * stride];
            for (int64_t i = 0; i < len; ++i) base[t * vstep + i * stride] -= d * base[o * vstep + i * stride];
          }
        double nn = 0.0;
        for (int64_t i = 0; i < len; ++i) nn += base[t * vstep + i * stride] * base[t * vstep + i * stride];
        if (nn > 0.25) {
          const double inv = 1.0 / sqrt(nn);
          for (int64_t i = 0; i < len; ++i) base[t * vstep + i * stride] *= inv;
          break;
        }
      }
    }
  }
}

struct IsFlag {
  const int64_t* flag;
  int64_t want;
  __device__ bool operator()(int64_t b) const { return flag[b] == want; }
};
// non-degenerate block of size class cls inside the owned block range [lo, hi) (a sharded solve's
// rank owns a contiguous range of blocks, sharded.cu; one rank owns them all)
struct IsNonDeg {
  const int64_t* keep;
  const int64_t* large;
  int64_t cls;
  int64_t lo, hi;
  __device__ bool operator()(int64_t b) const { return keep[b] > 0 && large[b] == cls && b >= lo && b < hi; }
};

__global__ void k_iota64(int64_t* a, int64_t n) {
  FPI_GRID_STRIDE(i, n) a[i] = i;
}

// scatter one block (rows rs.., cols cs..) into a zeroed row-major h x w buffer
__global__ void k_scatter_block(int64_t rs, int64_t h, int64_t cs, int64_t w, const int64_t* __restrict__ a_ptr,
                                const int32_t* __restrict__ a_idx, const double* __restrict__ a_val,
                                double* __restrict__ D, int transposed) {
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < h; i += nw)
    for (int64_t p = a_ptr[rs + i] + lane; p < a_ptr[rs + i + 1]; p += 32) {
      const int64_t j = a_idx[p] - cs;
      if (transposed) D[j * h + i] = a_val[p]; else D[i * w + j] = a_val[p];
    }
}

// copy the oriented factors of one block into the CSR value arrays: U11 part (h x kp), Vt11 part (kp x w).
// not transposed: Uo (h x kp), Vto (kp x w).  transposed (oriented panel = A^T): Uo (w x kp), Vto (kp x h).
__global__ void k_store_large(int64_t h, int64_t w, int64_t kp, const double* __restrict__ Uo,
                              const double* __restrict__ Vto, int transposed, double* __restrict__ u_val,
                              double* __restrict__ vt_val) {
  FPI_GRID_STRIDE(e, h * kp) {
    const int64_t i = e / kp, t = e - i * kp;
    u_val[e] = transposed ? Vto[t * h + i] : Uo[e];
  }
  FPI_GRID_STRIDE(e2, kp * w) {
    const int64_t t = e2 / w, j = e2 - t * w;
    vt_val[e2] = transposed ? Uo[j * kp + t] : Vto[e2];
  }
}

}  // namespace

struct BlockSvdState {
  int64_t nspans = 0;
  Scratch<int64_t> keep, rank_off, u_off, v_off, uk, vk, large;
  int64_t rank11 = 0, nnz_u = 0, nnz_v = 0, n_small = 0, n_large = 0;
};

__global__ void k_large_meta(int64_t nl, const int64_t* __restrict__ large, const int64_t* __restrict__ spans,
                             const int64_t* __restrict__ keep, const int64_t* __restrict__ roff,
                             const int64_t* __restrict__ uoff, const int64_t* __restrict__ voff,
                             int64_t* __restrict__ meta) {
  FPI_GRID_STRIDE(i, nl) {
    const int64_t b = large[i];
    int64_t* m = meta + 8 * i;
    m[0] = spans[4 * b];
    m[1] = spans[4 * b + 1];
    m[2] = spans[4 * b + 2];
    m[3] = spans[4 * b + 3];
    m[4] = keep[b];
    m[5] = roff[b];
    m[6] = uoff[b];
    m[7] = voff[b];
  }
}

static int64_t smem_limit_doubles(fpi_context* h) { return (int64_t)(h->smem_optin - 1024) / 8; }

__global__ void k_plan_tails(int64_t n, const int64_t* __restrict__ a0, const int64_t* __restrict__ a1,
                             const int64_t* __restrict__ a2, const int64_t* __restrict__ a3,
                             const int64_t* __restrict__ a4, const int64_t* __restrict__ a5, int64_t* __restrict__ out) {
  if (threadIdx.x == 0) {
    out[0] = a0[n - 1];
    out[1] = a1[n - 1];
    out[2] = a2[n - 1];
    out[3] = a3[n - 1];
    out[4] = a4[n - 1];
    out[5] = a5[n - 1];
  }
}

static void plan(fpi_context* h, int64_t nspans, const int64_t* spans, double alpha, BlockSvdState& st) {
  cudaStream_t s = h->stream;
  st.nspans = nspans;
  int64_t n = nspans > 0 ? nspans : 1;
  st.keep.alloc(n + 1, s); st.rank_off.alloc(n + 1, s); st.u_off.alloc(n + 1, s); st.v_off.alloc(n + 1, s);
  st.uk.alloc(n + 1, s); st.vk.alloc(n + 1, s); st.large.alloc(n + 1, s);
  if (nspans == 0) return;
  const int T = 256;
  k_plan<<<grid_for(nspans, T, h->num_sms * 16), T, 0, s>>>(nspans, spans, alpha, st.keep, st.uk, st.vk, st.large,
                                                            smem_limit_doubles(h));
  CubTemp tmp(s);
  exclusive_sum(tmp, st.keep.get(), st.rank_off.get(), nspans + 0, s);
  exclusive_sum(tmp, st.uk.get(), st.u_off.get(), nspans, s);
  exclusive_sum(tmp, st.vk.get(), st.v_off.get(), nspans, s);
  FPI_LAUNCH_CHECK();
  note_launch(h, 4);
  // the six scan tails in one pinned read (one synchronisation instead of six pageable copies)
  Scratch<int64_t> tails(6, s);
  k_plan_tails<<<1, 32, 0, s>>>(nspans, st.rank_off, st.keep, st.u_off, st.uk, st.v_off, st.vk, tails);
  FPI_LAUNCH_CHECK();
  int64_t last[6];
  host_read_n(tails.get(), last, 6, s);
  st.rank11 = last[0] + last[1];
  st.nnz_u = last[2] + last[3];
  st.nnz_v = last[4] + last[5];
}

void block_svd(fpi_context* h, int64_t m1, int64_t n1, const int64_t* a_ptr, const int32_t* a_idx,
               const double* a_val, int64_t nspans, const int64_t* spans, double alpha, double* sigma,
               int64_t* u_ptr, int32_t* u_idx, double* u_val, int64_t* vt_ptr, int32_t* vt_idx, double* vt_val,
               fpi_block_plan* out_plan, int64_t b_lo, int64_t b_hi, int64_t* keep_range) {
  FPI_REQUIRE(alpha > 0.0 && alpha <= 1.0, FPI_EDOMAIN, "target rank ratio alpha must be in (0, 1]");
  cudaStream_t s = h->stream;
  BlockSvdState st;
  plan(h, nspans, spans, alpha, st);
  const int T = 256;
  const unsigned G = (unsigned)(h->num_sms * 16);
  // structure of U11 (m1 x rank11) and Vt11 (rank11 x n1)
  CubTemp tmp(s);
  if (u_ptr) {
    Scratch<int64_t> row_cnt(m1 + 1, s);
    FPI_CUDA(cudaMemsetAsync(row_cnt.get(), 0, sizeof(int64_t) * (m1 + 1), s));
    if (nspans) k_u_rows<<<grid_for(nspans * 32, T, G), T, 0, s>>>(nspans, spans, st.keep, row_cnt);
    FPI_CUDA(cudaMemsetAsync(u_ptr, 0, sizeof(int64_t), s));
    if (m1) inclusive_sum(tmp, row_cnt.get(), u_ptr + 1, m1, s);
  }
  if (nspans && u_idx && vt_ptr && vt_idx)
    k_structure<<<grid_for(nspans * 32, T, G), T, 0, s>>>(nspans, spans, st.keep, st.rank_off, st.u_off, st.v_off,
                                                          u_idx, vt_ptr, vt_idx);
  if (vt_ptr) FPI_CUDA(cudaMemcpyAsync(vt_ptr + st.rank11, &st.nnz_v, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  FPI_LAUNCH_CHECK();
  note_launch(h, 3);
  if (nspans == 0) {
    if (out_plan) *out_plan = fpi_block_plan{0, 0, 0, 0, 0};
    FPI_CUDA(cudaStreamSynchronize(s));
    return;
  }
  // small tier: class 0 (tiny, many CTAs per SM) and class 2 (up to the full opt-in smem)
  Scratch<int64_t> ids(nspans, s), small(nspans, s), mid(nspans, s), large(nspans, s);
  Scratch<int> cnt(3, s);
  k_iota64<<<grid_for(nspans, T, G), T, 0, s>>>(ids, nspans);
  select_if(tmp, ids.get(), small.get(), cnt.get(), nspans,
            IsNonDeg{st.keep.get(), st.large.get(), 0, b_lo, b_hi}, s);
  select_if(tmp, ids.get(), mid.get(), cnt.get() + 1, nspans,
            IsNonDeg{st.keep.get(), st.large.get(), 2, b_lo, b_hi}, s);
  select_if(tmp, ids.get(), large.get(), cnt.get() + 2, nspans, IsFlag{st.large.get(), 1}, s);
  const bool partial = b_lo > 0 || b_hi < nspans;
  if (keep_range) {
    // keep offsets [k_lo, k_hi) of the owned block range (rank_off is the exclusive keep prefix)
    keep_range[0] = b_lo >= nspans ? st.rank11 : (b_lo <= 0 ? 0 : host_read(st.rank_off.get() + b_lo, s));
    keep_range[1] = b_hi >= nspans ? st.rank11 : (b_hi <= 0 ? 0 : host_read(st.rank_off.get() + b_hi, s));
  }
  if (partial) {
    // only this rank's blocks are written: the others' values stay zero, so a sum over the ranks
    // (the all-reduce of the sharded solve) assembles the full factors
    if (st.rank11) FPI_CUDA(cudaMemsetAsync(sigma, 0, sizeof(double) * st.rank11, s));
    if (u_val && st.nnz_u) FPI_CUDA(cudaMemsetAsync(u_val, 0, sizeof(double) * st.nnz_u, s));
    if (vt_val && st.nnz_v) FPI_CUDA(cudaMemsetAsync(vt_val, 0, sizeof(double) * st.nnz_v, s));
  }
  int hc[3];
  FPI_CUDA(cudaMemcpyAsync(hc, cnt.get(), sizeof(hc), cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  st.n_small = hc[0] + hc[1];
  st.n_large = hc[2];
  // metadata of the (few) large blocks only, fetched before the small-block kernels are queued so
  // the host builds the large batch while the device works
  std::vector<int64_t> meta(8 * (size_t)st.n_large);
  if (st.n_large) {
    Scratch<int64_t> dmeta(8 * st.n_large, s);
    k_large_meta<<<grid_for(st.n_large, T, G), T, 0, s>>>(st.n_large, large, spans, st.keep, st.rank_off, st.u_off,
                                                            st.v_off, dmeta);
    FPI_LAUNCH_CHECK();
    note_launch(h);
    FPI_CUDA(cudaMemcpyAsync(meta.data(), dmeta.get(), sizeof(int64_t) * meta.size(), cudaMemcpyDeviceToHost, s));
    FPI_CUDA(cudaStreamSynchronize(s));
  }
  {
    static std::atomic<uint64_t> attr{0};
    const size_t full = h->smem_optin - 1024;
    once_per_device(attr, h->device, [&] {
      FPI_CUDA(cudaFuncSetAttribute(k_block_svd_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)full));
    });
    const int64_t counts[2] = {hc[0], hc[1]};
    const int64_t* lists[2] = {small.get(), mid.get()};
    const size_t smem[2] = {(size_t)TINY_DOUBLES * 8, full};
    for (int c = 0; c < 2; ++c) {
      const int64_t nsm = counts[c];
      if (!nsm) continue;
      KTimer kt(h, c == 0 ? "block_svd_jacobi_tiny" : "block_svd_jacobi_smem", 0.0, 0.0);
      k_block_svd_small<<<(unsigned)(nsm < 65535 ? nsm : 65535), BT, smem[c], s>>>(
          lists[c], nsm, spans, st.keep, st.rank_off, st.u_off, st.v_off, a_ptr, a_idx, a_val, sigma, u_val, vt_val,
          60);
      k_complete_null<<<grid_for(nsm, 128, G), 128, 0, s>>>(lists[c], nsm, spans, st.keep, st.rank_off, st.u_off,
                                                            st.v_off, sigma, u_val, vt_val);
      FPI_LAUNCH_CHECK();
      note_launch(h, 2);
    }
  }
  if (st.n_large && (b_lo > 0 || b_hi < nspans)) {
    // block-range ownership: the large blocks inside [b_lo, b_hi)
    std::vector<int64_t> ids(st.n_large), kept;
    FPI_CUDA(cudaMemcpyAsync(ids.data(), large.get(), sizeof(int64_t) * st.n_large, cudaMemcpyDeviceToHost, s));
    FPI_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < st.n_large; ++i)
      if (ids[i] >= b_lo && ids[i] < b_hi)
        for (int f = 0; f < 8; ++f) kept.push_back(meta[8 * i + f]);
    meta.swap(kept);
    st.n_large = (int64_t)(meta.size() / 8);
  }
  if (st.n_large) {
    // meta row i: rs, hh, cs, ww, keep, rank_off, u_off, v_off of the i-th large block
    // dense, oriented (rows >= cols) copies of every large block, one batched SVD for all of them
    const int nl = (int)st.n_large;
    std::vector<int64_t> pp(nl), qq(nl), kk(nl), ldm(nl);
    std::vector<int> tr(nl);
    int64_t tot = 0;
    for (int i = 0; i < nl; ++i) {
      const int64_t* mt = meta.data() + 8 * i;
      const int64_t hh = mt[1], ww = mt[3];
      FPI_REQUIRE(hh * ww <= 4000000, FPI_ECAPACITY,
                  "diagonal block of " + std::to_string(hh) + "x" + std::to_string(ww) +
                      " entries exceeds the 4000000-entry guard; reordering produced a pathological block");
      tr[i] = hh < ww;
      pp[i] = tr[i] ? ww : hh;
      qq[i] = tr[i] ? hh : ww;
      kk[i] = mt[4];
      ldm[i] = qq[i];
      tot += hh * ww;
    }
    Scratch<double> Dall(tot, s);
    FPI_CUDA(cudaMemsetAsync(Dall.get(), 0, sizeof(double) * tot, s));
    std::vector<const double*> Mp(nl);
    std::vector<double*> Up(nl), Sp(nl), Vp(nl);
    int64_t tu = 0, tv = 0;
    for (int i = 0; i < nl; ++i) {
      tu += pp[i] * kk[i];
      tv += kk[i] * qq[i];
    }
    Scratch<double> Uall(tu, s), Vall(tv, s);
    int64_t od = 0, ou = 0, ov = 0;
    for (int i = 0; i < nl; ++i) {
      const int64_t* mt = meta.data() + 8 * i;
      const int64_t rs = mt[0], hh = mt[1], cs = mt[2], ww = mt[3];
      double* D = Dall.get() + od;
      k_scatter_block<<<grid_for(hh * 32, T, G), T, 0, s>>>(rs, hh, cs, ww, a_ptr, a_idx, a_val, D, tr[i]);
      Mp[i] = D;
      Up[i] = Uall.get() + ou;
      Vp[i] = Vall.get() + ov;
      Sp[i] = sigma + mt[5];
      od += hh * ww;
      ou += pp[i] * kk[i];
      ov += kk[i] * qq[i];
    }
    FPI_LAUNCH_CHECK();
    dense_svd_batched(h, nl, pp.data(), qq.data(), Mp.data(), ldm.data(), kk.data(), Up.data(), Sp.data(),
                      Vp.data());
    for (int i = 0; i < nl; ++i) {
      const int64_t* mt = meta.data() + 8 * i;
      const int64_t hh = mt[1], ww = mt[3];
      // oriented M = U' S V'^T; for a transposed block A = V' S U'^T
      k_store_large<<<grid_for(hh * kk[i] + kk[i] * ww, T, G), T, 0, s>>>(hh, ww, kk[i], Up[i], Vp[i], tr[i],
                                                                           u_val + mt[6], vt_val + mt[7]);
      note_launch(h, 2);
    }
    FPI_LAUNCH_CHECK();
  }
  if (out_plan) *out_plan = fpi_block_plan{st.rank11, st.nnz_u, st.nnz_v, st.n_small + st.n_large, st.n_large};
}

void block_plan_only(fpi_context* h, int64_t nspans, const int64_t* spans, double alpha, fpi_block_plan* out) {
  FPI_REQUIRE(alpha > 0.0 && alpha <= 1.0, FPI_EDOMAIN, "target rank ratio alpha must be in (0, 1]");
  BlockSvdState st;
  plan(h, nspans, spans, alpha, st);
  out->rank11 = st.rank11;
  out->nnz_u11 = st.nnz_u;
  out->nnz_vt11 = st.nnz_v;
  out->n_blocks_svd = 0;
  out->n_blocks_large = 0;
}

}  // namespace fpi

extern "C" int fpi_block_svd_plan(fpi_handle h, int64_t n_spans, const int64_t* d_spans, double alpha,
                                  fpi_block_plan* h_plan) {
  FPI_API_BEGIN(h)
  fpi::block_plan_only(h, n_spans, d_spans, alpha, h_plan);
  FPI_API_END(h)
}

extern "C" int fpi_block_svd(fpi_handle h, int64_t m1, int64_t n1, const int64_t* a11_ptr, const int32_t* a11_idx,
                             const double* a11_val, int64_t n_spans, const int64_t* d_spans, double alpha,
                             double* d_sigma, int64_t* u_ptr, int32_t* u_idx, double* u_val, int64_t* vt_ptr,
                             int32_t* vt_idx, double* vt_val, fpi_block_plan* h_plan) {
  FPI_API_BEGIN(h)
  fpi::block_svd(h, m1, n1, a11_ptr, a11_idx, a11_val, n_spans, d_spans, alpha, d_sigma, u_ptr, u_idx, u_val,
                 vt_ptr, vt_idx, vt_val, h_plan, 0, n_spans, nullptr);
  FPI_API_END(h)
}

extern "C" int fpi_block_svd_range(fpi_handle h, int64_t m1, int64_t n1, const int64_t* a11_ptr,
                                   const int32_t* a11_idx, const double* a11_val, int64_t n_spans,
                                   const int64_t* d_spans, double alpha, int64_t b_lo, int64_t b_hi, double* d_sigma,
                                   int64_t* u_ptr, int32_t* u_idx, double* u_val, int64_t* vt_ptr, int32_t* vt_idx,
                                   double* vt_val, fpi_block_plan* h_plan, int64_t* h_keep_range) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(0 <= b_lo && b_lo <= b_hi && b_hi <= n_spans, FPI_EDOMAIN, "bad block range");
  fpi::block_svd(h, m1, n1, a11_ptr, a11_idx, a11_val, n_spans, d_spans, alpha, d_sigma, u_ptr, u_idx, u_val,
                 vt_ptr, vt_idx, vt_val, h_plan, b_lo, b_hi, h_keep_range);
  FPI_API_END(h)
}
