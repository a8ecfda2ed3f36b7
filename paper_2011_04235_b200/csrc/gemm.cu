// FP64 GEMM on the sm_100a double-precision tensor path (mma.sync m8n8k4 f64
// -> SASS DMMA).  tcgen05 has no f64 kind, so DMMA is the FP64 tensor-core
// instruction on B200.
//
//   C = alpha * op(A) * op(B) + beta * C,   all row-major, op = identity / transpose
//
// CTA tile 64 x 64 x 16, 4 warps (2 x 2), warp tile 32 x 32 = 4 x 4 DMMA tiles
// (32 accumulator doubles per thread), three CTAs per SM: while one CTA sits at
// its k-tile barrier the others keep the DMMA pipe issuing.  Operands stream global -> smem with a
// 3-stage cp.async ring (16-byte copies when the operands are 16-byte aligned
// along their contiguous dimension, 8-byte otherwise); the smem layouts are
// padded so every fragment load is bank-conflict free for all four transpose
// combinations.  Split-K (deterministic: partial tiles + ordered reduction)
// covers the tall-skinny Gram / projection shapes where M x N alone cannot fill
// 148 SMs; the split count minimises a wave-quantisation + reduction model.
// Used for: U.Sigma x X1 and Q^T inner (svd.py:133,135 dense parts), the
// Gram matrices of CholeskyQR and of the small SVD, the lifts
// (pinv.py:169,206) and V (Sigma+ U^T Y) (pinv.py:81).
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "capi_guard.cuh"
#include "gemm.cuh"
#include "instrument.cuh"

namespace fpi {
namespace {

// Tile configuration (tools/gemm_variants.sh measures the alternatives on the solve's shapes:
// 128x64 / 2 CTAs, 64x32 / 4-5 CTAs, 64x64 / 4 stages, 128x128 / 64x32 warps all land at 28-31
// TFLOP/s; 64x64 with 4 warps and 3 CTAs per SM is the best overall at 31-32).
#ifndef FPI_GEMM_CFG_BM
#define FPI_GEMM_CFG_BM 64
#define FPI_GEMM_CFG_BN 64
#define FPI_GEMM_CFG_WM 32
#define FPI_GEMM_CFG_WN 32
#define FPI_GEMM_CFG_STAGES 3
#define FPI_GEMM_CFG_CTAS 3
#endif
#ifndef FPI_GEMM_CFG_BK
#define FPI_GEMM_CFG_BK 16
#endif
constexpr int BM = FPI_GEMM_CFG_BM, BN = FPI_GEMM_CFG_BN, BK = FPI_GEMM_CFG_BK, STAGES = FPI_GEMM_CFG_STAGES;
constexpr int WM = FPI_GEMM_CFG_WM, WN = FPI_GEMM_CFG_WN;  // warp tile
constexpr int MI = WM / 8, NJ = WN / 8;                    // DMMA tiles per warp
constexpr int WARPS_N = BN / WN;                            // warp grid (BM / WM) x (BN / WN)
constexpr int NT = (BM / WM) * (BN / WN) * 32;
constexpr int PAD = 4;
// smem strides (doubles)
constexpr int LDA_MK = BK + PAD;   // As[m][k]
constexpr int LDA_KM = BM + PAD;   // As[k][m]
constexpr int LDB_KN = BN + PAD;   // Bs[k][n]
constexpr int LDB_NK = BK + PAD;   // Bs[n][k]
constexpr int A_STAGE = (BM * LDA_MK > BK * LDA_KM) ? BM * LDA_MK : BK * LDA_KM;
constexpr int B_STAGE = (BN * LDB_NK > BK * LDB_KN) ? BN * LDB_NK : BK * LDB_KN;
constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
static_assert((BM * BK) % NT == 0 && (BN * BK) % NT == 0, "tile loads divide evenly over the threads");

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
// 16-byte copy of up to two doubles (nvalid in 0..2; the rest zero-filled)
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int nvalid) {
  unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  int sz = nvalid * 8;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Load one BM x BK tile of op(A) and one BK x BN tile of op(B) into stage buffers.  V16: pairs of
// doubles along each operand's contiguous dimension (16-byte aligned by the caller's check).
template <bool TA, bool TB, bool V16>
__device__ __forceinline__ void load_tiles(double* As, double* Bs, const double* A, int64_t lda, const double* B,
                                           int64_t ldb, int64_t M, int64_t N, int64_t K, int64_t m0, int64_t n0,
                                           int64_t k0) {
  const int tid = threadIdx.x;
  constexpr int W = V16 ? 2 : 1;
#pragma unroll
  for (int i = 0; i < (BM * BK) / (NT * W); ++i) {
    const int e = (tid + i * NT) * W;
    int m, k;
    if (!TA) { m = e / BK; k = e % BK; } else { k = e / BM; m = e % BM; }
    const int64_t gm = m0 + m, gk = k0 + k;
    double* dst = TA ? As + k * LDA_KM + m : As + m * LDA_MK + k;
    if (V16) {
      // contiguous dimension: k (A[m][k]) or m (A^T stored K x M)
      const int64_t lim = TA ? M - gm : K - gk;
      const bool row_ok = TA ? gk < K : gm < M;
      const int nv = !row_ok || lim <= 0 ? 0 : (lim >= 2 ? 2 : 1);
      cp_async16(dst, nv ? (TA ? A + gk * lda + gm : A + gm * lda + gk) : A, nv);
    } else {
      const bool p = gm < M && gk < K;
      cp_async8(dst, p ? (TA ? A + gk * lda + gm : A + gm * lda + gk) : A, p);
    }
  }
#pragma unroll
  for (int i = 0; i < (BN * BK) / (NT * W); ++i) {
    const int e = (tid + i * NT) * W;
    int n, k;
    if (!TB) { k = e / BN; n = e % BN; } else { n = e / BK; k = e % BK; }
    const int64_t gn = n0 + n, gk = k0 + k;
    double* dst = TB ? Bs + n * LDB_NK + k : Bs + k * LDB_KN + n;
    if (V16) {
      const int64_t lim = TB ? K - gk : N - gn;
      const bool row_ok = TB ? gn < N : gk < K;
      const int nv = !row_ok || lim <= 0 ? 0 : (lim >= 2 ? 2 : 1);
      cp_async16(dst, nv ? (TB ? B + gn * ldb + gk : B + gk * ldb + gn) : B, nv);
    } else {
      const bool p = gn < N && gk < K;
      cp_async8(dst, p ? (TB ? B + gn * ldb + gk : B + gk * ldb + gn) : B, p);
    }
  }
}

// sym: C is symmetric (A == B, op(A) = op(B)^T).  Tiles entirely above the diagonal are skipped;
// every computed element (r, c) with c <= r is stored, and mirrored to (c, r) when c < r, so each
// upper element has exactly one (deterministic) writer.
__host__ __device__ __forceinline__ bool tile_above_diag(int64_t bx, int64_t by) {
  return bx * BN >= (by + 1) * BM;
}

template <bool TA, bool TB, bool V16>
__global__ void __launch_bounds__(NT, FPI_GEMM_CFG_CTAS)
    k_gemm(int64_t M, int64_t N, int64_t K, double alpha, const double* __restrict__ A, int64_t lda,
           const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C, int64_t ldc,
           int64_t k_per_split, double* __restrict__ partial, int sym) {
  if (sym && tile_above_diag(blockIdx.x, blockIdx.y)) return;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kb = (int64_t)blockIdx.z * k_per_split;
  const int64_t ke = kb + k_per_split < K ? kb + k_per_split : K;
  const int64_t ntiles = ke > kb ? (ke - kb + BK - 1) / BK : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp / WARPS_N) * WM, wn = (warp % WARPS_N) * WN;
  const int g = lane >> 2, t = lane & 3;

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // prologue
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntiles)
      load_tiles<TA, TB, V16>(As + s * A_STAGE, Bs + s * B_STAGE, A, lda, B, ldb, M, N, ke, m0, n0, kb + s * BK);
    cp_async_commit();
  }
  for (int64_t kt = 0; kt < ntiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    // prefetch tile kt + STAGES - 1 into the slot freed last iteration
    {
      int64_t nk = kt + STAGES - 1;
      int slot = (int)(nk % STAGES);
      if (nk < ntiles)
        load_tiles<TA, TB, V16>(As + slot * A_STAGE, Bs + slot * B_STAGE, A, lda, B, ldb, M, N, ke, m0, n0,
                                kb + nk * BK);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * A_STAGE;
    const double* bs = Bs + (kt % STAGES) * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        int m = wm + i * 8 + g;
        af[i] = TA ? as[(kk + t) * LDA_KM + m] : as[m * LDA_MK + kk + t];
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        int n = wn + j * 8 + g;
        bf[j] = TB ? bs[n * LDB_NK + kk + t] : bs[(kk + t) * LDB_KN + n];
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: accumulator (i, j) holds rows wm+8i+g, cols wn+8j+2t, +1
  if (partial) {
    double* P = partial + (int64_t)blockIdx.z * M * N;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      int64_t r = m0 + wm + i * 8 + g;
      if (r >= M) continue;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        int64_t c = n0 + wn + j * 8 + 2 * t;
        if (c < N && (!sym || c <= r)) P[r * N + c] = acc[i][j][0];
        if (c + 1 < N && (!sym || c + 1 <= r)) P[r * N + c + 1] = acc[i][j][1];
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    int64_t r = m0 + wm + i * 8 + g;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      int64_t c = n0 + wn + j * 8 + 2 * t;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t cq = c + q;
        if (cq < N && (!sym || cq <= r)) {
          double v = alpha * acc[i][j][q];
          double* dst = C + r * ldc + cq;
          *dst = beta == 0.0 ? v : v + beta * *dst;
          if (sym && cq < r) {
            double* mir = C + cq * ldc + r;
            *mir = beta == 0.0 ? v : v + beta * *mir;
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// TMA-fed variant (operands 16-byte aligned along their contiguous dimension, even leading
// dimensions): the same 64 x 64 x 16 CTA tile and DMMA warp tiles, but every stage's A and B tiles
// arrive by cp.async.bulk.tensor (one elected thread issues them, an mbarrier counts the bytes)
// into 128-byte-swizzled shared memory, so the fragment loads stay conflict-free without padding.
// Tiles reaching past M / N / K are zero-filled by the TMA unit (no predicated copies).
// Sub-tiles are 16 doubles (128 B, the swizzle span) wide: a K-contiguous operand is one
// 16 x 64 box per stage, an M- or N-contiguous one four 16 x 16 boxes.
constexpr int TSTAGES = 4;
constexpr int T_STAGE = BM * BK + BN * BK;  // doubles per stage (A then B)
constexpr size_t TMA_SMEM_BYTES = (size_t)TSTAGES * T_STAGE * sizeof(double) + 1024 + 16 * TSTAGES;
static_assert(BM == 64 && BN == 64 && BK == 16, "the TMA box layout assumes 64 x 64 x 16 tiles");

// element (r, c) of a [rows][16] sub-tile written by TMA with CU_TENSOR_MAP_SWIZZLE_128B: the
// 16-byte chunk index is XORed with the row index mod 8
__device__ __forceinline__ int swz(int r, int c) { return r * 16 + ((((c >> 1) ^ (r & 7)) << 1) | (c & 1)); }

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(double* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT + 32, FPI_GEMM_CFG_CTAS)
    k_gemm_tma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t M,
               int64_t N, int64_t K, double alpha, double beta, double* __restrict__ C, int64_t ldc,
               int64_t k_per_split, double* __restrict__ partial, int sym) {
  static_assert(TA != TB, "the TMA kernel serves the conflict-free NT / TN layouts");
  constexpr bool NT_MODE = !TA && TB;
  constexpr int CONSUMERS = NT / 32;  // compute warps; warp CONSUMERS is the TMA producer
  if (sym && tile_above_diag(blockIdx.x, blockIdx.y)) return;
  extern __shared__ unsigned char smem_raw[];
  double* st = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(st + TSTAGES * T_STAGE);
  uint64_t* empty = full + TSTAGES;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kb = (int64_t)blockIdx.z * k_per_split;
  const int64_t ke = kb + k_per_split < K ? kb + k_per_split : K;
  const int64_t ntiles = ke > kb ? (ke - kb + BK - 1) / BK : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == CONSUMERS) {
    // producer warp: one elected lane refills a slot as soon as every compute warp released it
    if (lane == 0) {
      for (int64_t kt = 0; kt < ntiles; ++kt) {
        const int slot = (int)(kt % TSTAGES);
        if (kt >= TSTAGES) mbar_wait(&empty[slot], (unsigned)(((kt / TSTAGES) - 1) & 1));
        double* As = st + slot * T_STAGE;
        double* Bs = As + BM * BK;
        mbar_expect_tx(&full[slot], (unsigned)(T_STAGE * sizeof(double)));
        const int k0 = (int)(kb + kt * BK);
        if (!TA) {
          tma_load_2d(As, &tmA, k0, (int)m0, &full[slot]);  // A[m][k]: one 16 (k) x 64 (m) box
        } else {
#pragma unroll
          for (int j = 0; j < BM / 16; ++j) tma_load_2d(As + j * 256, &tmA, (int)m0 + 16 * j, k0, &full[slot]);
        }
        if (TB) {
          tma_load_2d(Bs, &tmB, k0, (int)n0, &full[slot]);  // B stored N x K: one 16 (k) x 64 (n) box
        } else {
#pragma unroll
          for (int j = 0; j < BN / 16; ++j) tma_load_2d(Bs + j * 256, &tmB, (int)n0 + 16 * j, k0, &full[slot]);
        }
      }
    }
    return;
  }
  const int wm = (warp / WARPS_N) * WM, wn = (warp % WARPS_N) * WN;
  const int g = lane >> 2, t = lane & 3;

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Fragment placement that keeps the swizzled loads conflict-free (one 256-byte warp load = two
  // wavefronts): the 128-byte swizzle XORs the chunk index with (row mod 8), so
  //  * NT (both operands K-contiguous rows): fragment row g takes tile row pi(g) = 2(g mod 4) + g/4,
  //    putting the two 16-byte chunks of consecutive k for half a warp's 4 rows on 8 distinct chunks;
  //    C rows and columns follow pi;
  //  * TN (both M- / N-contiguous): the four k of one DMMA step are k0 + 2t (k0 in 0, 1, 8, 9), whose
  //    rows' XOR patterns spread a half warp's 8 chunk slots over all 8 chunks.
  const int pg = NT_MODE ? (((g & 3) << 1) | (g >> 2)) : g;
  for (int64_t kt = 0; kt < ntiles; ++kt) {
    const int slot = (int)(kt % TSTAGES);
    mbar_wait(&full[slot], (unsigned)((kt / TSTAGES) & 1));
    const double* as = st + slot * T_STAGE;
    const double* bs = as + BM * BK;
#pragma unroll
    for (int step = 0; step < BK / 4; ++step) {
      double af[MI], bf[NJ];
      if (NT_MODE) {
        const int k = step * 4 + t;
#pragma unroll
        for (int i = 0; i < MI; ++i) af[i] = as[swz(wm + i * 8 + pg, k)];
#pragma unroll
        for (int j = 0; j < NJ; ++j) bf[j] = bs[swz(wn + j * 8 + pg, k)];
      } else {
        const int k = ((step & 1) | ((step >> 1) << 3)) + 2 * t;
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int m = wm + i * 8 + g;
          af[i] = as[(m >> 4) * 256 + swz(k, m & 15)];
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int n = wn + j * 8 + g;
          bf[j] = bs[(n >> 4) * 256 + swz(k, n & 15)];
        }
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[slot])) : "memory");
  }

  // accumulator (i, j, q) holds C[m0 + wm + 8i + pi(g)][n0 + wn + 8j + pi(2t + q)]  (pi = id for TN)
  auto colmap = [](int c) { return NT_MODE ? (((c & 3) << 1) | (c >> 2)) : c; };
  if (partial) {
    double* P = partial + (int64_t)blockIdx.z * M * N;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int64_t r = m0 + wm + i * 8 + pg;
      if (r >= M) continue;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int64_t c = n0 + wn + j * 8 + colmap(2 * t + q);
          if (c < N && (!sym || c <= r)) P[r * N + c] = acc[i][j][q];
        }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t r = m0 + wm + i * 8 + pg;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t cq = n0 + wn + j * 8 + colmap(2 * t + q);
        if (cq < N && (!sym || cq <= r)) {
          double v = alpha * acc[i][j][q];
          double* dst = C + r * ldc + cq;
          *dst = beta == 0.0 ? v : v + beta * *dst;
          if (sym && cq < r) {
            double* mir = C + cq * ldc + r;
            *mir = beta == 0.0 ? v : v + beta * *mir;
          }
        }
      }
    }
  }
}

__global__ void k_reduce_split(int64_t M, int64_t N, int splits, const double* __restrict__ P, double alpha,
                               double beta, double* __restrict__ C, int64_t ldc, int sym) {
  FPI_GRID_STRIDE(e, M * N) {
    int64_t r = e / N, c = e - r * N;
    // upper elements of a symmetric product were not computed: read the mirrored partials
    const int64_t src = (sym && c > r) ? c * N + r : e;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += P[(int64_t)z * M * N + src];
    double* dst = C + r * ldc + c;
    double v = alpha * s;
    *dst = beta == 0.0 ? v : v + beta * *dst;
  }
}

__global__ void k_scale(int64_t M, int64_t N, double beta, double* __restrict__ C, int64_t ldc) {
  FPI_GRID_STRIDE(e, M * N) {
    int64_t r = e / N, c = e - r * N;
    double* dst = C + r * ldc + c;
    *dst = beta == 0.0 ? 0.0 : beta * *dst;
  }
}

// Split count: minimise (waves of CTAs) x (K per CTA) + the partial-tile reduction traffic.
int choose_splits(int64_t tiles, int64_t M, int64_t N, int64_t K, int num_sms) {
  const int64_t slots = (int64_t)FPI_GEMM_CFG_CTAS * num_sms;  // resident CTAs
  const double cta_flops = 36.0e12 / (double)slots, red_bw = 4.0e12;
  int best = 1;
  double best_t = 1e300;
  const int64_t max_splits = K / (BK * 8) < 64 ? K / (BK * 8) : 64;
  for (int sp = 1; sp <= (max_splits > 1 ? max_splits : 1); ++sp) {
    const int64_t kps = ((K + sp - 1) / sp + BK - 1) / BK * BK;
    const int64_t real = (K + kps - 1) / kps;
    if (real != sp) continue;
    const int64_t waves = (tiles * sp + slots - 1) / slots;
    double t = (double)waves * 2.0 * BM * BN * (double)kps / cta_flops;
    if (sp > 1) t += (double)M * N * (sp + 1) * 8.0 / red_bw;
    if (t < best_t * 0.98) {
      best_t = t;
      best = sp;
    }
  }
  return best;
}

template <bool TA, bool TB, bool V16>
void launch(fpi_context* h, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
            const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int sym) {
  static std::atomic<uint64_t> attr_set{0};
  once_per_device(attr_set, h->device, [] {
    FPI_CUDA(cudaFuncSetAttribute(k_gemm<TA, TB, V16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
  });
  cudaStream_t s = h->stream;
  const int64_t tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  int64_t tiles = tm * tn;
  if (sym) {
    tiles = 0;
    for (int64_t by = 0; by < tm; ++by) {
      const int64_t lim = ((by + 1) * BM + BN - 1) / BN;  // bx < lim are not entirely above the diagonal
      tiles += lim < tn ? lim : tn;
    }
  }
  int splits = choose_splits(tiles, M, N, K, h->num_sms);
  if (const char* e = getenv("FPI_GEMM_SPLITS")) splits = atoi(e) > 0 ? atoi(e) : splits;
  FPI_REQUIRE(tm < 65536 && tn < (1LL << 31), FPI_ECAPACITY, "gemm grid too large");
  if (splits == 1) {
    dim3 grid((unsigned)tn, (unsigned)tm, 1);
    k_gemm<TA, TB, V16><<<grid, NT, SMEM_BYTES, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, K, nullptr, sym);
    FPI_LAUNCH_CHECK();
    note_launch(h);
    return;
  }
  int64_t kps = (K + splits - 1) / splits;
  kps = (kps + BK - 1) / BK * BK;
  splits = (int)((K + kps - 1) / kps);
  Scratch<double> part((size_t)splits * M * N, s);
  dim3 grid((unsigned)tn, (unsigned)tm, (unsigned)splits);
  k_gemm<TA, TB, V16><<<grid, NT, SMEM_BYTES, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kps, part, sym);
  k_reduce_split<<<grid_for(M * N, 256, (int64_t)h->num_sms * 16), 256, 0, s>>>(M, N, splits, part, alpha, beta, C,
                                                                                 ldc, sym);
  FPI_LAUNCH_CHECK();
  note_launch(h, 2);
}

// ---- TMA descriptors (driver entry point fetched through the runtime: no -lcuda at link time)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// row-major rows x cols (leading dimension ld) operand, boxes of 16 (contiguous) x box_rows
bool encode_operand(CUtensorMap* tm, const double* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool TA, bool TB>
bool launch_tma(fpi_context* h, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int sym) {
  if (M >= (1LL << 31) || N >= (1LL << 31) || K >= (1LL << 31)) return false;
  alignas(64) CUtensorMap tmA, tmB;
  // op(A) = A (M x K, K contiguous: 16 x 64 boxes) or A^T (A stored K x M: 16 x 16 boxes)
  if (!(TA ? encode_operand(&tmA, A, K, M, lda, 16) : encode_operand(&tmA, A, M, K, lda, 64))) return false;
  // op(B) = B (K x N stored, N contiguous: 16 x 16 boxes) or B^T (B stored N x K: 16 x 64 boxes)
  if (!(TB ? encode_operand(&tmB, B, N, K, ldb, 64) : encode_operand(&tmB, B, K, N, ldb, 16))) return false;
  static std::atomic<uint64_t> attr_set{0};
  once_per_device(attr_set, h->device, [] {
    FPI_CUDA(cudaFuncSetAttribute(k_gemm_tma<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)TMA_SMEM_BYTES));
  });
  cudaStream_t s = h->stream;
  const int64_t tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  int64_t tiles = tm * tn;
  if (sym) {
    tiles = 0;
    for (int64_t by = 0; by < tm; ++by) {
      const int64_t lim = ((by + 1) * BM + BN - 1) / BN;
      tiles += lim < tn ? lim : tn;
    }
  }
  int splits = choose_splits(tiles, M, N, K, h->num_sms);
  if (const char* e = getenv("FPI_GEMM_SPLITS")) splits = atoi(e) > 0 ? atoi(e) : splits;
  FPI_REQUIRE(tm < 65536 && tn < (1LL << 31), FPI_ECAPACITY, "gemm grid too large");
  if (splits == 1) {
    dim3 grid((unsigned)tn, (unsigned)tm, 1);
    k_gemm_tma<TA, TB><<<grid, NT + 32, TMA_SMEM_BYTES, s>>>(tmA, tmB, M, N, K, alpha, beta, C, ldc, K, nullptr, sym);
    FPI_LAUNCH_CHECK();
    note_launch(h);
    return true;
  }
  int64_t kps = (K + splits - 1) / splits;
  kps = (kps + BK - 1) / BK * BK;  // a k-tile never straddles two splits
  splits = (int)((K + kps - 1) / kps);
  Scratch<double> part((size_t)splits * M * N, s);
  dim3 grid((unsigned)tn, (unsigned)tm, (unsigned)splits);
  k_gemm_tma<TA, TB><<<grid, NT + 32, TMA_SMEM_BYTES, s>>>(tmA, tmB, M, N, K, alpha, beta, C, ldc, kps, part, sym);
  k_reduce_split<<<grid_for(M * N, 256, (int64_t)h->num_sms * 16), 256, 0, s>>>(M, N, splits, part, alpha, beta, C,
                                                                                 ldc, sym);
  FPI_LAUNCH_CHECK();
  note_launch(h, 2);
  return true;
}

// An operand with an odd leading dimension (or an 8-byte aligned base) would put the whole product on
// the 8-byte copies (18-24 instead of 26-30 TFLOP/s); the row update's rank s is such a dimension
// (399 at c4, 939 at c5).  When the product is large enough to pay for one pass over the operand,
// it is repacked into an even-stride scratch buffer first and the 16-byte / TMA tiles take it.
__global__ void k_repack(int64_t rows, int64_t cols, const double* __restrict__ src, int64_t lds,
                         double* __restrict__ dst, int64_t ldd) {
  FPI_GRID_STRIDE(e, rows * cols) {
    const int64_t r = e / cols, c = e - r * cols;
    dst[r * ldd + c] = src[r * lds + c];
  }
}

template <bool TA, bool TB>
void launch_any(fpi_context* h, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int sym) {
  static const bool no_repack = getenv("FPI_GEMM_NO_REPACK") != nullptr;
  const bool a_ok = (uintptr_t)A % 16 == 0 && lda % 2 == 0, b_ok = (uintptr_t)B % 16 == 0 && ldb % 2 == 0;
  Scratch<double> Ar, Br;
  if (!(a_ok && b_ok) && !no_repack && (double)M * (double)N * (double)K >= 2.5e8 && (a_ok || N >= 256) &&
      (b_ok || M >= 256)) {
    cudaStream_t s = h->stream;
    const bool same = A == B && lda == ldb && TA != TB && M == N;  // the Gram products pass one operand twice
    auto repack = [&](const double* src, int64_t rows, int64_t cols, int64_t ld, Scratch<double>& dst) {
      const int64_t ldd = cols + (cols & 1);
      dst.alloc(rows * ldd, s);
      k_repack<<<grid_for(rows * cols, 256, (int64_t)h->num_sms * 16), 256, 0, s>>>(rows, cols, src, ld, dst.get(), ldd);
      FPI_LAUNCH_CHECK();
      note_launch(h);
      return ldd;
    };
    if (!a_ok) {
      lda = repack(A, TA ? K : M, TA ? M : K, lda, Ar);
      if (same) {
        B = Ar;
        ldb = lda;
      }
      A = Ar;
    }
    if (!b_ok && B != A) {
      ldb = repack(B, TB ? N : K, TB ? K : N, ldb, Br);
      B = Br;
    }
  }
  const bool v16 = ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0) && lda % 2 == 0 && ldb % 2 == 0 &&
                   !getenv("FPI_GEMM_NO_V16");
  // TMA needs 16-byte aligned bases and row strides (the v16 condition)
  const bool no_tma = getenv("FPI_GEMM_NO_TMA") != nullptr;
  // TMA for the NT / TN layouts (both operands contiguous along the same dimension: the fixed
  // 128-byte swizzle then admits conflict-free fragment loads); NN / TT keep the padded cp.async
  // tiles (with TMA one operand's loads would be 2-way bank-conflicted: measured 7% slower)
  // (symmetric Gram products stay on cp.async: with TMA their lower-tile / long split-K grids measured
  // 3-35% slower -- tools/gram_bench.py: 256^2 x 2M 18.4 vs 24.8, 940^2 x 349k 25.4 vs 29.1 TFLOP/s)
  if constexpr (TA != TB) {
    if (v16 && !no_tma && !sym && launch_tma<TA, TB>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sym)) return;
  }
  if (v16) launch<TA, TB, true>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sym);
  else launch<TA, TB, false>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sym);
}

}  // namespace

void gemm(fpi_context* h, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
          int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, bool sym) {
  if (M <= 0 || N <= 0) return;
  const int sy = (sym && M == N && A == B && ta != tb) ? 1 : 0;
  if (K <= 0) {
    k_scale<<<grid_for(M * N, 256, (int64_t)h->num_sms * 16), 256, 0, h->stream>>>(M, N, beta, C, ldc);
    FPI_LAUNCH_CHECK();
    return;
  }
  KTimer kt(h, "gemm_f64_dmma", (sy ? 1.0 : 2.0) * (double)M * (double)N * (double)K,
            8.0 * ((double)M * K + (double)K * N + (beta == 0.0 ? 1.0 : 2.0) * (double)M * N));
  // FPI_GEMM_LOG=1: shape and device time of every product on stderr (serialising; diagnostics only)
  static const bool log = getenv("FPI_GEMM_LOG") != nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (log) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, h->stream);
  }
  if (!ta && !tb) launch_any<false, false>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, 0);
  else if (!ta && tb) launch_any<false, true>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sy);
  else if (ta && !tb) launch_any<true, false>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sy);
  else launch_any<true, true>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, 0);
  if (log) {
    cudaEventRecord(e1, h->stream);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    fprintf(stderr, "[gemm] %c%c sym=%d M=%lld N=%lld K=%lld %.3f ms %.1f TFLOP/s\n", ta ? 'T' : 'N', tb ? 'T' : 'N',
            sy, (long long)M, (long long)N, (long long)K, ms,
            (sy ? 1.0 : 2.0) * (double)M * (double)N * (double)K / (ms * 1e9));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
}

}  // namespace fpi

extern "C" int fpi_gemm(fpi_handle h, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, double alpha,
                        const double* d_A, int64_t lda, const double* d_B, int64_t ldb, double beta, double* d_C,
                        int64_t ldc) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(M >= 0 && N >= 0 && K >= 0, FPI_EDOMAIN, "negative GEMM dimension");
  fpi::gemm(h, trans_a != 0, trans_b != 0, M, N, K, alpha, d_A, lda, d_B, ldb, beta, d_C, ldc);
  FPI_API_END(h)
}
