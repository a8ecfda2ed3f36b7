// Cholesky factor and its inverse in ONE tile-dataflow kernel (the CholeskyQR factor of the
// randomized SVD: B^T B = L L^T, Q = B L^-T -- svd.py:134's QR without forming Q).
//
// The (padded) n x n matrix is cut into 32 x 32 tiles.  Every lower tile is one task of each
// phase, handed out in a dependency-respecting (column-major) order from an atomic counter:
//   phase 1 (left-looking Cholesky)  A_ij -= sum_{k<j} L_ik L_jk^T, then
//            i == j: L_jj = chol(A_jj) and D_j = L_jj^-1 (one warp, shared memory)
//            i >  j: L_ij = A_ij D_j^T
//   phase 2 (inverse, X = L^-1)      X_jj = D_j,  X_ij = -D_i sum_{k=j}^{i-1} L_ik X_kj
// A task waits (acquire spin on a per-tile flag) only for tiles earlier in the order, which are
// held by running CTAs, so the schedule cannot deadlock and needs no grid barrier.  The 32^3
// tile products run on the FP64 tensor path (mma.sync m8n8k4 -> DMMA); every tile sums its
// terms in a fixed order, so the result is deterministic.  The critical path is ~nt diagonal
// steps instead of the ~5 nt kernel launches of the blocked panel algorithm.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "instrument.cuh"
#include "linalg.cuh"

namespace fpi {
namespace {

constexpr int TS = 32;
constexpr int LD = 36;  // smem tile stride (doubles)
constexpr int CT = 256;  // threads per CTA (8 warps, two 8 x 8 output tiles each)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void wait_flag(const int* f) {
  if (threadIdx.x == 0)
    while (ld_acquire(f) == 0) __nanosleep(32);
  __syncthreads();
}

// publish a tile written by this CTA
__device__ __forceinline__ void set_flag(int* f) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release(f, 1);
}

// this thread's output elements: warp w owns 8 x 8 tiles (w >> 1, 2 (w & 1)) and (w >> 1, 2 (w & 1) + 1)
struct Frag {
  int r, c0, c1;  // row and the first column of the two pairs
  __device__ Frag() {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    r = 8 * (w >> 1) + (lane >> 2);
    c0 = 16 * (w & 1) + 2 * (lane & 3);
    c1 = c0 + 8;
  }
};

// acc (+)= sign * X Y^T  (both row-major tiles in smem)
__device__ __forceinline__ void mma_xyt(double acc[4], const double (*X)[LD], const double (*Y)[LD], double sign) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = 8 * (w >> 1), c0 = 16 * (w & 1);
  const int ar = r0 + (lane >> 2), ak = lane & 3, bn = lane >> 2;
#pragma unroll
  for (int k0 = 0; k0 < TS; k0 += 4) {
    const double a = sign * X[ar][k0 + ak];
    dmma(acc[0], acc[1], a, Y[c0 + bn][k0 + ak]);
    dmma(acc[2], acc[3], a, Y[c0 + 8 + bn][k0 + ak]);
  }
}

// acc (+)= sign * X Y  (Y row-major (k, n))
__device__ __forceinline__ void mma_xy(double acc[4], const double (*X)[LD], const double (*Y)[LD], double sign) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = 8 * (w >> 1), c0 = 16 * (w & 1);
  const int ar = r0 + (lane >> 2), ak = lane & 3, bn = lane >> 2;
#pragma unroll
  for (int k0 = 0; k0 < TS; k0 += 4) {
    const double a = sign * X[ar][k0 + ak];
    dmma(acc[0], acc[1], a, Y[k0 + ak][c0 + bn]);
    dmma(acc[2], acc[3], a, Y[k0 + ak][c0 + 8 + bn]);
  }
}

__device__ __forceinline__ void load_tile(double (*S)[LD], const double* T, int64_t ld) {
  for (int e = threadIdx.x; e < TS * TS / 2; e += CT) {
    const int r = e >> 4, c = (e & 15) * 2;
    const double2 v = __ldcg(reinterpret_cast<const double2*>(T + r * ld + c));
    S[r][c] = v.x;
    S[r][c + 1] = v.y;
  }
}

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// asynchronous tile copy (one commit group per call)
__device__ __forceinline__ void load_tiles_async(double (*S0)[LD], const double* T0, int64_t ld0, double (*S1)[LD],
                                                 const double* T1, int64_t ld1) {
  for (int e = threadIdx.x; e < TS * TS / 2; e += CT) {
    const int r = e >> 4, c = (e & 15) * 2;
    cp_async16(&S0[r][c], T0 + r * ld0 + c);
    cp_async16(&S1[r][c], T1 + r * ld1 + c);
  }
  cp_commit();
}

__device__ __forceinline__ void acc_to_smem(double (*S)[LD], const double acc[4]) {
  const Frag f;
  S[f.r][f.c0] = acc[0];
  S[f.r][f.c0 + 1] = acc[1];
  S[f.r][f.c1] = acc[2];
  S[f.r][f.c1 + 1] = acc[3];
}

__device__ __forceinline__ void acc_to_global(double* T, int64_t ld, const double acc[4]) {
  const Frag f;
  *reinterpret_cast<double2*>(T + f.r * ld + f.c0) = make_double2(acc[0], acc[1]);
  *reinterpret_cast<double2*>(T + f.r * ld + f.c1) = make_double2(acc[2], acc[3]);
}

// Step K of the register Cholesky (template recursion keeps every register index static).
template <int K>
__device__ __forceinline__ void chol_step(double (&a)[TS], int lane, double& myinv, int& badk) {
  if constexpr (K < TS) {
    double d = __shfl_sync(0xffffffffu, a[K], K);
    badk = (badk < 0 && !(d > 0.0)) ? K : badk;  // branch-free: the step chain stays one basic block
    d = (d > 0.0) ? d : 1e-300;
    // 1/sqrt(d) from the MUFU estimate plus one Newton step (a few ulp; the factor only has to
    // reproduce B^T B to rounding), sqrt(d) = d / sqrt(d)
    double inv;
    asm("rsqrt.approx.f64 %0, %1;" : "=d"(inv) : "d"(d));
    inv = inv * fma(-0.5 * d * inv, inv, 1.5);
    const double lkk = d * inv;
    const double scaled = a[K] * inv;
    a[K] = (lane == K) ? lkk : ((lane > K) ? scaled : a[K]);
    myinv = (lane == K) ? inv : myinv;
#pragma unroll
    for (int jj = K + 1; jj < TS; ++jj) {
      const double ljk = __shfl_sync(0xffffffffu, a[K], jj);
      const double upd = fma(-a[K], ljk, a[jj]);
      a[jj] = (jj <= lane) ? upd : a[jj];
    }
    chol_step<K + 1>(a, lane, myinv, badk);
  }
}

// Row R of the forward substitution x = L^-1 e_lane (template recursion: static register indices).
template <int R>
__device__ __forceinline__ void inv_step(double (&x)[TS], const double (*SC)[LD], const double* sdinv, int lane) {
  if constexpr (R < TS) {
    double s = (R == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) s = fma(-SC[R][q], x[q], s);
    x[R] = s * sdinv[R];
    inv_step<R + 1>(x, SC, sdinv, lane);
  }
}

// Warp 0: Cholesky of the 32 x 32 tile in SC (lower part valid) in registers (lane = row, the
// column-k multipliers broadcast by shuffles), L written back to SC with the upper part zeroed;
// then D = L^-1 by forward substitution (lane = column), written to SD.
__device__ __forceinline__ void chol_inv_warp(double (*SC)[LD], double (*SD)[LD], double* sdinv, int* info,
                                           int64_t base, unsigned long long* dbg) {
  const int lane = threadIdx.x & 31;
  double a[TS];
#pragma unroll
  for (int c = 0; c < TS; ++c) a[c] = SC[lane][c];
  if (dbg && lane == 0) dbg[0] = gtimer_ns();
  double myinv = 0.0;
  int badk = -1;
  chol_step<0>(a, lane, myinv, badk);
  sdinv[lane] = myinv;
  if (badk >= 0 && lane == 0) atomicCAS(info, 0, (int)(base + badk + 1));
  if (dbg && lane == 0) dbg[1] = gtimer_ns();
#pragma unroll
  for (int c = 0; c < TS; ++c) SC[lane][c] = c <= lane ? a[c] : 0.0;
  __syncwarp();
  // forward substitution, lane = column of D (x in registers; rows above the diagonal come out 0)
  double x[TS];
  inv_step<0>(x, SC, sdinv, lane);
  if (dbg && lane == 0) dbg[2] = gtimer_ns();
#pragma unroll
  for (int r = 0; r < TS; ++r) SD[r][lane] = x[r];
}

__global__ void __launch_bounds__(CT, 1)
    k_chol_inv_dataflow(int64_t n, int nt, const double* __restrict__ G, int64_t ldg, double* Lp, double* Xp,
                        double* Dv, int* flagL, int* flagX, int* counter, int* info,
                        unsigned long long* prof) {
  __shared__ __align__(16) double SAB[2][2][TS][LD];  // double-buffered operand tiles
  __shared__ __align__(16) double SC[TS][LD];
  double(*SA)[LD] = SAB[0][0];
  double(*SB)[LD] = SAB[0][1];
  __shared__ int s_task;
  __shared__ double sdinv[TS];
  const int64_t N = (int64_t)nt * TS;
  const int ntri = nt * (nt + 1) / 2;
  const Frag f;
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(counter, 1);
    __syncthreads();
    const int t = s_task;
    __syncthreads();
    if (t >= 2 * ntri) break;
    const bool ph2 = t >= ntri;
    int tt = ph2 ? t - ntri : t, j = 0;
    while (tt >= nt - j) {
      tt -= nt - j;
      ++j;
    }
    const int i = j + tt;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (prof && threadIdx.x == 0) prof[3 * t] = gtimer_ns();
    if (!ph2) {
      // A_ij with the identity padding beyond n
      {
        const int64_t R = (int64_t)i * TS + f.r;
        const int64_t C4[4] = {(int64_t)j * TS + f.c0, (int64_t)j * TS + f.c0 + 1, (int64_t)j * TS + f.c1,
                               (int64_t)j * TS + f.c1 + 1};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          acc[e] = (R < n && C4[e] < n) ? G[R * ldg + C4[e]] : (R == C4[e] ? 1.0 : 0.0);
      }
      // sum_{k<j} L_ik L_jk^T, the next pair of tiles in flight while this one multiplies
      auto issue1 = [&](int k) {
        wait_flag(flagL + i * nt + k);
        wait_flag(flagL + j * nt + k);
        load_tiles_async(SAB[k & 1][0], Lp + (int64_t)i * TS * N + (int64_t)k * TS, N, SAB[k & 1][1],
                         Lp + (int64_t)j * TS * N + (int64_t)k * TS, N);
      };
      if (j > 0) issue1(0);
      for (int k = 0; k < j; ++k) {
        if (k + 1 < j) {
          issue1(k + 1);
          cp_wait<1>();
        } else {
          cp_wait<0>();
        }
        __syncthreads();
        mma_xyt(acc, SAB[k & 1][0], SAB[k & 1][1], -1.0);
        __syncthreads();
      }
      if (prof && threadIdx.x == 0) prof[3 * t + 1] = gtimer_ns();
      if (i == j) {
        acc_to_smem(SC, acc);
        __syncthreads();
        unsigned long long* dbg = prof ? prof + 3 * 2 * ntri + 4 * j : nullptr;
        if (threadIdx.x < 32) chol_inv_warp(SC, SA, sdinv, info, (int64_t)j * TS, dbg);
        __syncthreads();
        double* Lt = Lp + (int64_t)j * TS * N + (int64_t)j * TS;
        double* Dt = Dv + (int64_t)j * TS * TS;
        for (int e = threadIdx.x; e < TS * TS; e += CT) {
          const int r = e >> 5, c = e & 31;
          Lt[r * N + c] = SC[r][c];
          Dt[e] = SA[r][c];
        }
        if (dbg && threadIdx.x == 0) dbg[3] = gtimer_ns();
        set_flag(flagL + j * nt + j);
        if (prof && threadIdx.x == 0) prof[3 * t + 2] = gtimer_ns();
      } else {
        wait_flag(flagL + j * nt + j);
        load_tile(SB, Dv + (int64_t)j * TS * TS, TS);
        acc_to_smem(SC, acc);
        __syncthreads();
        double out[4] = {0.0, 0.0, 0.0, 0.0};
        mma_xyt(out, SC, SB, 1.0);  // L_ij = A_ij D_j^T
        acc_to_global(Lp + (int64_t)i * TS * N + (int64_t)j * TS, N, out);
        set_flag(flagL + i * nt + j);
        if (prof && threadIdx.x == 0) prof[3 * t + 2] = gtimer_ns();
      }
    } else {
      double* Xt = Xp + (int64_t)i * TS * N + (int64_t)j * TS;
      if (i == j) {
        wait_flag(flagL + j * nt + j);
        const double* Dt = Dv + (int64_t)j * TS * TS;
        for (int e = threadIdx.x; e < TS * TS; e += CT) Xt[(e >> 5) * N + (e & 31)] = __ldcg(Dt + e);
        set_flag(flagX + j * nt + j);
      } else {
        auto issue2 = [&](int k) {
          wait_flag(flagL + i * nt + k);
          wait_flag(flagX + k * nt + j);
          load_tiles_async(SAB[k & 1][0], Lp + (int64_t)i * TS * N + (int64_t)k * TS, N, SAB[k & 1][1],
                           Xp + (int64_t)k * TS * N + (int64_t)j * TS, N);
        };
        issue2(j);
        for (int k = j; k < i; ++k) {
          if (k + 1 < i) {
            issue2(k + 1);
            cp_wait<1>();
          } else {
            cp_wait<0>();
          }
          __syncthreads();
          mma_xy(acc, SAB[k & 1][0], SAB[k & 1][1], 1.0);
          __syncthreads();
        }
        wait_flag(flagL + i * nt + i);
        load_tile(SA, Dv + (int64_t)i * TS * TS, TS);
        acc_to_smem(SC, acc);
        __syncthreads();
        double out[4] = {0.0, 0.0, 0.0, 0.0};
        mma_xy(out, SA, SC, -1.0);  // X_ij = -D_i sum_k L_ik X_kj
        acc_to_global(Xt, N, out);
        set_flag(flagX + i * nt + j);
      }
      if (prof && threadIdx.x == 0) prof[3 * t + 2] = gtimer_ns();
    }
  }
}

__global__ void k_copy_lower(int64_t n, const double* __restrict__ S, int64_t lds, double* __restrict__ D,
                             int64_t ldd, int zero_upper) {
  FPI_GRID_STRIDE(e, n * n) {
    const int64_t r = e / n, c = e - r * n;
    if (c <= r)
      D[r * ldd + c] = S[r * lds + c];
    else if (zero_upper)
      D[r * ldd + c] = 0.0;
  }
}

}  // namespace

bool chol_inverse_dataflow(fpi_context* h, int64_t n, const double* G, int64_t ldg, double* L, int64_t ldl,
                           double* Linv, int64_t ldi, int* h_info) {
  if (getenv("FPI_CHOL_BLOCKED") != nullptr || n <= 0) return false;
  cudaStream_t s = h->stream;
  const int nt = (int)((n + TS - 1) / TS);
  const int64_t N = (int64_t)nt * TS;
  const int ntri = nt * (nt + 1) / 2;
  Scratch<double> Lp(N * N, s), Xp(N * N, s), Dv((int64_t)nt * TS * TS, s);
  Scratch<int> flags(2 * nt * nt + 2, s);
  FPI_CUDA(cudaMemsetAsync(flags.get(), 0, sizeof(int) * (2 * nt * nt + 2), s));
  int* counter = flags.get() + 2 * nt * nt;
  int* info = counter + 1;
  KTimer kt(h, "cholesky_inverse_dataflow", (double)n * n * n, 0.0);
  int grid = h->num_sms;
  if (grid > 2 * ntri) grid = 2 * ntri;
  const bool prof_on = getenv("FPI_CHOL_PROFILE") != nullptr;
  Scratch<unsigned long long> prof(prof_on ? 3 * 2 * ntri + 4 * nt : 1, s);
  if (prof_on) FPI_CUDA(cudaMemsetAsync(prof.get(), 0, sizeof(unsigned long long) * (3 * 2 * ntri + 4 * nt), s));
  k_chol_inv_dataflow<<<grid, CT, 0, s>>>(n, nt, G, ldg, Lp, Xp, Dv, flags.get(), flags.get() + nt * nt, counter,
                                          info, prof_on ? prof.get() : nullptr);
  if (prof_on) {
    std::vector<unsigned long long> hp(3 * 2 * ntri + 4 * nt);
    FPI_CUDA(cudaMemcpyAsync(hp.data(), prof.get(), sizeof(unsigned long long) * hp.size(), cudaMemcpyDeviceToHost, s));
    FPI_CUDA(cudaStreamSynchronize(s));
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int t = 0; t < 2 * ntri; ++t) {
      if (hp[3 * t] && hp[3 * t] < t0) t0 = hp[3 * t];
      if (hp[3 * t + 2] > t1) t1 = hp[3 * t + 2];
    }
    fprintf(stderr, "[chol n=%lld nt=%d] total %.1f us; diagonal tasks (grab / deps ready / done, us):\n", (long long)n,
            nt, (t1 - t0) * 1e-3);
    int t = 0;
    for (int j = 0; j < nt; ++j) {
      fprintf(stderr, "  d%02d %7.1f %7.1f %7.1f |", j, (hp[3 * t] - t0) * 1e-3, (hp[3 * t + 1] - t0) * 1e-3,
              (hp[3 * t + 2] - t0) * 1e-3);
      if (j + 1 < nt)
        fprintf(stderr, " L%02d,%02d done %7.1f", j + 1, j, (hp[3 * (t + 1) + 2] - t0) * 1e-3);
      const unsigned long long* dg = hp.data() + 3 * 2 * ntri + 4 * j;
      fprintf(stderr, " [chol %.1f inv %.1f store %.1f]", (dg[1] - dg[0]) * 1e-3, (dg[2] - dg[1]) * 1e-3,
              (dg[3] - dg[2]) * 1e-3);
      const int tx = ntri + t;  // X_jj
      fprintf(stderr, " | X%02d,%02d done %7.1f\n", j, j, (hp[3 * tx + 2] - t0) * 1e-3);
      t += nt - j;
    }
    // last X of column 0
    fprintf(stderr, "  X%02d,00 done %7.1f\n", nt - 1, (hp[3 * (ntri + nt - 1) + 2] - t0) * 1e-3);
  }
  const unsigned g2 = grid_for(n * n, 256, (int64_t)h->num_sms * 16);
  k_copy_lower<<<g2, 256, 0, s>>>(n, Lp, N, L, ldl, 1);
  k_copy_lower<<<g2, 256, 0, s>>>(n, Xp, N, Linv, ldi, 1);
  FPI_LAUNCH_CHECK();
  note_launch(h, 3);
  *h_info = host_read(info, s);
  return true;
}

}  // namespace fpi
