// Symmetric eigensolver: parallel two-sided block Jacobi, one cooperative
// kernel (replaces LAPACK's dsyevd / the eigen part of dgesdd, svd.py:105,136).
//
// The n x n matrix (padded to nb * 16) is split into 16-wide index blocks.
// A sweep is nb - 1 rounds of the round-robin pairing of blocks; in a round
// every block pair (I, J) owns the 32 x 32 sub-problem G[I u J, I u J]:
//   phase A  one CTA per pair, the sub-problem in shared memory: 16 threads
//            compute the 16 disjoint rotations of a step, all 256 threads apply
//            them as independent 2 x 2 block updates.  Round 0 of a sweep
//            rotates the within-block pairs (15 steps), every round the cross
//            pairs (16 steps), so each index pair is visited once per sweep (a
//            cyclic Jacobi ordering).
//   phase B  every upper 32 x 32 block of G gets G'[P, P'] = R_P^T G[P, P'] R_P'
//            (written to both triangles), as 32^3 products on the FP64 tensor
//            path (mma.sync m8n8k4 -> DMMA); each CTA streams a contiguous run
//            of blocks through a two-stage cp.async pipeline.
//   V        the eigenvector update V[:, P'] <- V[:, P'] R_P' of round r does
//            not feed the iteration, so it runs during phase A of round r + 1
//            on the CTAs phase A leaves idle (R is double-buffered by round).
// Grid-wide barriers separate the phases.  A sweep ends by checking the
// largest off-diagonal measure seen (relative |a_pq| / sqrt(a_pp a_qq), or
// absolute |a_pq| / max|a_ii| for Gram matrices) against the tolerance, or
// its stagnation at the rounding floor.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "capi_guard.cuh"
#include "cub_util.cuh"
#include "instrument.cuh"
#include "linalg.cuh"

namespace cg = cooperative_groups;

namespace fpi {
namespace {

constexpr int JB = 16;      // index block
constexpr int JS = 32;      // sub-problem (two blocks)
constexpr int JT = 256;     // threads per CTA
constexpr int LDS_ = 36;    // smem stride (doubles): conflict-free DMMA fragment loads

__device__ __forceinline__ int rr_block(int pos, int round, int nb) {
  // (pos - 1 + round) mod (nb - 1) without the integer division: both terms are below nb - 1
  const int m = nb - 1;
  int x = pos - 1 + round;
  while (x >= m) x -= m;  // at most once for round < nb - 1
  return pos == 0 ? 0 : 1 + x;
}
__device__ __forceinline__ int sub_to_global(int l, int bi, int bj) { return l < JB ? bi * JB + l : bj * JB + (l - JB); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---- phase A: cyclic Jacobi on one 32 x 32 sub-problem in shared memory ---
// Step descriptors: within-block step t (circle method on 16, both halves:
// pairs k < 8 in the first half, k >= 8 in the second) and cross step t
// (k <-> 16 + (k + t) % 16).  Each step rotates 16 disjoint index pairs.
__device__ __forceinline__ int pos16(int i, int t) { return i == 0 ? 0 : 1 + ((i - 1 + t) % 15); }
__device__ __forceinline__ void step_pair(int mode, int t, int k, int& p, int& q) {
  if (mode == 0) {
    const int h = k < 8 ? 0 : 16, kk = k & 7;
    p = h + pos16(kk, t);
    q = h + pos16(15 - kk, t);
  } else {
    p = k;
    q = 16 + ((k + t) & 15);
  }
}

// Per-step pairing tables (steps 0..14 within-block, 15..30 cross).
struct StepTables {
  signed char P[31][16], Q[31][16];
  signed char pair_of[31][32];  // pair index of each local index
  signed char is_p[31][32];     // 1 if the index is the pair's p
};

__device__ void build_tables(StepTables& tb) {
  for (int e = threadIdx.x; e < 31 * 16; e += blockDim.x) {
    const int st = e / 16, k = e % 16;
    int p, q;
    step_pair(st < 15 ? 0 : 1, st < 15 ? st : st - 15, k, p, q);
    tb.P[st][k] = (signed char)p;
    tb.Q[st][k] = (signed char)q;
    tb.pair_of[st][p] = (signed char)k;
    tb.pair_of[st][q] = (signed char)k;
    tb.is_p[st][p] = 1;
    tb.is_p[st][q] = 0;
  }
}

#ifndef JACOBI_CS32
#define JACOBI_CS32 1
#endif
#ifndef JACOBI_ROT32
#define JACOBI_ROT32 1
#endif

// MUFU approximations for the rotation (measured on B200: rsqrt.approx.f64 ~2^-52.4 -- ptxas
// refines MUFU.RSQ64H -- and rcp.approx.ftz.f64 ~2^-20).
__device__ __forceinline__ __attribute__((unused)) double rcp_apx(double x) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ double rsqrt_apx(double x) { double r; asm("rsqrt.approx.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }

// Rotation of one pair from (app, aqq, apq), without the z = (aqq - app) / (2 apq) division:
//   t = tan(theta) = sign(d) 2 apq / (|d| + sqrt(d^2 + 4 apq^2)),  d = aqq - app,
// with sqrt through rsqrt.approx.f64 (MUFU + refinement, ~2^-52) and the reciprocal through the
// raw MUFU (2^-20: only the angle needs it), then c = 1/sqrt(1 + t^2) to full precision and
// s = c t, so the rotation is orthogonal to rounding whatever the angle error.  Operands outside
// [1e-150, 1e150] are rescaled first (the ratio d : apq is all the angle depends on).
__device__ __forceinline__ void rotation(double app, double aqq, double apq, double tol, double ascale, bool absolute,
                                         double& c, double& sn) {
  const double den2 = absolute ? ascale * ascale : fabs(app) * fabs(aqq);
  const bool rot = apq != 0.0 && apq * apq > tol * tol * den2;
  double d = aqq - app, f2 = 2.0 * apq;
  const double mx = fmax(fabs(d), fabs(f2));
#if !JACOBI_ROT32
  if (mx > 1e150 || mx < 1e-150) {
    const double sc = mx > 0.0 ? rcp_apx(mx) : 1.0;
    d *= sc;
    f2 *= sc;
  }
  const double v = fma(d, d, f2 * f2);
  const double hyp = v * rsqrt_apx(v);
  const double t0 = f2 * rcp_apx(fabs(d) + hyp);
  const double tt = d < 0.0 ? -t0 : t0;
#else
  // The angle in FP32 (MUFU.RSQ / MUFU.RCP, ~2^-22 relative -- better than the 2^-20 the FP64
  // path's raw reciprocal gives), after scaling d and f2 by 2^-e (e = exponent of their larger
  // magnitude) into FP32's range; orthogonality comes from c and s below, computed in FP64.
  const int ex = (int)((__double_as_longlong(mx) >> 52) & 0x7ff) - 1023;
  const int ef = 1023 - ex < 1 ? 1 : (1023 - ex > 2046 ? 2046 : 1023 - ex);
  const double sc2 = __longlong_as_double((long long)ef << 52);
  const float df = (float)(d * sc2), ff = (float)(f2 * sc2);
  const float vf = fmaf(df, df, ff * ff);
  float rs;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(vf));
#if JACOBI_CS32
  // c, s straight from h = sqrt(d^2 + f^2) and w = |d| + h: 1 + t^2 = 2 h / w, so
  // c = w / sqrt(2 h w) and s = sign(d) f / sqrt(2 h w) -- two MUFU.RSQ, no reciprocal (~2^-22);
  // then made orthogonal in FP64 by the series 1 / sqrt(1 + e) = 1 - e / 2 + 3 e^2 / 8
  // (e = c0^2 + s0^2 - 1 ~ 1e-7: the next term is below FP64 rounding) -- four dependent FMAs
  // instead of a refined MUFU.RSQ64H
  float uf;
  const float hf = vf * rs, wf = fmaf(vf, rs, fabsf(df));
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(uf) : "f"(2.0f * hf * wf));
  const float c0f = wf * uf, s0f = (df < 0.0f ? -ff : ff) * uf;
  const double c0 = (double)c0f, s0 = (double)s0f;
  const double e = fma(c0, c0, fma(s0, s0, -1.0));
  const double rn = fma(e, fma(e, 0.375, -0.5), 1.0);
  c = rot ? c0 * rn : 1.0;
  sn = rot ? s0 * rn : 0.0;
  return;
#endif
  float rc;
  const float hypf = vf * rs;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(fabsf(df) + hypf));
  const float tf = ff * rc;
  const float tsf = df < 0.0f ? -tf : tf;
  const double tt = (double)tsf;
#endif
  const double cy = rsqrt_apx(fma(tt, tt, 1.0));
  c = rot ? cy : 1.0;
  sn = rot ? cy * tt : 0.0;
}

struct PairBuf {
  double c[2][16], s[2][16], app[2][16], aqq[2][16], apq[2][16];
};

// New diagonal entry of index x after its pair's rotation (2x2 congruence).
__device__ __forceinline__ double new_diag(bool isp, double c, double sn, double app, double aqq, double apq) {
  return isp ? c * c * app - 2.0 * c * sn * apq + sn * sn * aqq : sn * sn * app + 2.0 * c * sn * apq + c * c * aqq;
}

// One round's sub-problem: S (JS x JS, stride LDS_) <- J^T S J, R = J.  One barrier per step.
// Within-block steps (round 0 of a sweep only): thread (k, l) = (tid / 16, tid % 16) updates the
// 2 x 2 block of pairs k, l, and whichever thread produces a next-step pair's off-diagonal entry
// also derives that pair's new diagonals and computes its next rotation.  Cross steps (every
// round, the hot loop): thread tid = 16 d + k owns block (k, k + 1 + d); the producers of the
// next rotations are exactly d = 0, i.e. lanes 0..15 of warp 0, so the rotation chain (the
// critical path) runs on one warp while warps 1..7 apply the previous rotations to R.
// With Jout, the final rotation is written there as row-major J (straight from the registers of the
// cross steps) and *rot says whether this thread saw a non-identity entry; R is then left stale.
__device__ double subsolve(double* S, double* R, const StepTables& tb, PairBuf& pb, bool round0, double tol,
                           double ascale, bool absolute, double* Jout = nullptr, int* rot = nullptr) {
  const int st0 = round0 ? 0 : 15, st_end = 31;
  const int tid = threadIdx.x;
  // convergence measure of this sub-problem before rotating -- on warps 1..7, so warp 0 starts the
  // prologue rotations (the critical path) at once
  double om = 0.0;
  for (int e = tid - 32; e >= 0 && e < JS * JS; e += JT - 32) {
    const int x = e >> 5, y = e & 31;
    if (x == y) continue;
    const double sxy = S[x * LDS_ + y];
    const double den2 = absolute ? ascale * ascale : fabs(S[x * LDS_ + x]) * fabs(S[y * LDS_ + y]);
    if (sxy != 0.0) om = fmax(om, den2 > 0.0 ? fabs(sxy) * rsqrt_apx(den2) : 1.0);
  }
  // block maximum: warp partials now, thread 0 combines them after the steps' barriers
  __shared__ double s_om[JT / 32];
  for (int o = 16; o; o >>= 1) om = fmax(om, __shfl_xor_sync(0xffffffffu, om, o));
  if ((tid & 31) == 0) s_om[tid >> 5] = om;
  // prologue: rotations of the first step
  if (tid < 16) {
    const int k = tid, p = tb.P[st0][k], q = tb.Q[st0][k];
    const double app = S[p * LDS_ + p], aqq = S[q * LDS_ + q], apq = S[p * LDS_ + q];
    double c, sn;
    rotation(app, aqq, apq, tol, ascale, absolute, c, sn);
    const int b = st0 & 1;
    pb.c[b][k] = c; pb.s[b][k] = sn; pb.app[b][k] = app; pb.aqq[b][k] = aqq; pb.apq[b][k] = apq;
  }
  __syncthreads();
  if (round0) {
    const int k = tid >> 4, l = tid & 15;
    for (int st = 0; st < 15; ++st) {
      const int b = st & 1, nbuf = b ^ 1;
      const int pk = tb.P[st][k], qk = tb.Q[st][k], pl = tb.P[st][l], ql = tb.Q[st][l];
      const double ck = pb.c[b][k], sk = pb.s[b][k], cl = pb.c[b][l], sl = pb.s[b][l];
      if (sk != 0.0 || sl != 0.0) {
        const double a = S[pk * LDS_ + pl], bb = S[pk * LDS_ + ql], c2 = S[qk * LDS_ + pl], d = S[qk * LDS_ + ql];
        const double ra = ck * a - sk * c2, rb = ck * bb - sk * d;
        const double rc = sk * a + ck * c2, rd = sk * bb + ck * d;
        S[pk * LDS_ + pl] = ra * cl - rb * sl;
        S[pk * LDS_ + ql] = ra * sl + rb * cl;
        S[qk * LDS_ + pl] = rc * cl - rd * sl;
        S[qk * LDS_ + ql] = rc * sl + rd * cl;
      }
      if (sk != 0.0) {  // R is stored transposed (Rt[col][row]): conflict-free column updates
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int row = l + 16 * h2;
          const double rp = R[pk * LDS_ + row], rq = R[qk * LDS_ + row];
          R[pk * LDS_ + row] = ck * rp - sk * rq;
          R[qk * LDS_ + row] = sk * rp + ck * rq;
        }
      }
      if (k != l) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int x = (e < 2) ? pk : qk, y = (e & 1) ? ql : pl;
          const int kn = tb.pair_of[st + 1][x];
          if (tb.is_p[st + 1][x] && tb.Q[st + 1][kn] == y) {
            const double axy = S[x * LDS_ + y];
            const double dx = new_diag(e < 2, ck, sk, pb.app[b][k], pb.aqq[b][k], pb.apq[b][k]);
            const double dy = new_diag(!(e & 1), cl, sl, pb.app[b][l], pb.aqq[b][l], pb.apq[b][l]);
            double c, sn;
            rotation(dx, dy, axy, tol, ascale, absolute, c, sn);
            pb.c[nbuf][kn] = c; pb.s[nbuf][kn] = sn; pb.app[nbuf][kn] = dx; pb.aqq[nbuf][kn] = dy;
            pb.apq[nbuf][kn] = axy;
          }
        }
      }
      __syncthreads();
    }
  }
  // cross steps: pair k = (k, 16 + (k + t) % 16).  Identity rotations (c = 1, s = 0) are applied
  // as arithmetic (exact), so every load of a step is issued up front without branches.
  const int k = tid & 15, l = (k + 1 + (tid >> 4)) & 15;
  // R (stored transposed, Rt[col][row]) lives in registers during the cross steps: thread
  // (g, k) of warps 1..7 (g = (tid - 32) / 16) holds rows g, g + 14, g + 28 of column k and of the
  // column currently paired with k.  Step t pairs k with 16 + (k + t) % 16, and step t + 1 pairs k
  // with the column lane k + 1 held at step t, so the updated q values move one lane down (a
  // shuffle inside each 16-lane group) instead of round-tripping through shared memory.
  const int u = tid - 32, g = u >> 4, lane = tid & 31;
  const int src = (lane & 16) | ((lane + 1) & 15);
  double rp_[3] = {0.0, 0.0, 0.0}, rq_[3] = {0.0, 0.0, 0.0};
  if (u >= 0) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int row = g + 14 * r;
      if (row < JS) {  // R = I unless round 0's within-block steps ran
        rp_[r] = round0 ? R[k * LDS_ + row] : (row == k ? 1.0 : 0.0);
        rq_[r] = round0 ? R[(16 + k) * LDS_ + row] : (row == 16 + k ? 1.0 : 0.0);
      }
    }
  }
  for (int st = 15; st < st_end; ++st) {
    const int t = st - 15, b = st & 1, nbuf = b ^ 1;
    const int pk = k, qk = 16 + ((k + t) & 15), pl = l, ql = 16 + ((l + t) & 15);
    const double ck = pb.c[b][k], sk = pb.s[b][k], cl = pb.c[b][l], sl = pb.s[b][l];
    const double a = S[pk * LDS_ + pl], bb = S[pk * LDS_ + ql], c2 = S[qk * LDS_ + pl], d = S[qk * LDS_ + ql];
    // the producer's inputs for the new diagonals, loaded before any store of the step
    double appk = 0.0, aqqk = 0.0, apqk = 0.0, appl = 0.0, aqql = 0.0, apql = 0.0;
    if (tid < 16) {
      appk = pb.app[b][k]; aqqk = pb.aqq[b][k]; apqk = pb.apq[b][k];
      appl = pb.app[b][l]; aqql = pb.aqq[b][l]; apql = pb.apq[b][l];
    }
    const double ra = ck * a - sk * c2, rb = ck * bb - sk * d;
    const double rc = sk * a + ck * c2, rd = sk * bb + ck * d;
    const double o1 = ra * sl + rb * cl;
    S[pk * LDS_ + pl] = ra * cl - rb * sl;
    S[pk * LDS_ + ql] = o1;
    S[qk * LDS_ + pl] = rc * cl - rd * sl;
    S[qk * LDS_ + ql] = rc * sl + rd * cl;
    if (tid < 16) {
      // next cross pair k is (k, 16 + (k + t + 1) % 16) = (pk, ql) with l = k + 1: entry o1
      if (st + 1 < st_end) {
        const double dx = new_diag(true, ck, sk, appk, aqqk, apqk);
        const double dy = new_diag(false, cl, sl, appl, aqql, apql);
        double c, sn;
        rotation(dx, dy, o1, tol, ascale, absolute, c, sn);
        pb.c[nbuf][k] = c; pb.s[nbuf][k] = sn; pb.app[nbuf][k] = dx; pb.aqq[nbuf][k] = dy; pb.apq[nbuf][k] = o1;
      }
    } else if (u >= 0) {
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        if (g + 14 * r < JS) {  // warp-uniform
          const double p0 = rp_[r], q0 = rq_[r];
          rp_[r] = ck * p0 - sk * q0;
          rq_[r] = __shfl_sync(0xffffffffu, sk * p0 + ck * q0, src);
        }
      }
    }
    __syncthreads();
  }
  // after the 16th shift thread k holds column 16 + k again
  if (Jout) {
    int nz = 0;
    if (u >= 0) {
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int row = g + 14 * r;
        if (row < JS) {
          Jout[row * JS + k] = rp_[r];
          Jout[row * JS + 16 + k] = rq_[r];
          nz |= (rp_[r] != (row == k ? 1.0 : 0.0)) | (rq_[r] != (row == 16 + k ? 1.0 : 0.0));
        }
      }
    }
    *rot = nz;
    if (tid == 0)
      for (int w = 1; w < JT / 32; ++w) om = fmax(om, s_om[w]);
    return om;  // the sub-problem's measure in thread 0
  }
  if (u >= 0) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int row = g + 14 * r;
      if (row < JS) {
        R[k * LDS_ + row] = rp_[r];
        R[(16 + k) * LDS_ + row] = rq_[r];
      }
    }
  }
  __syncthreads();
  if (tid == 0)
    for (int w = 1; w < JT / 32; ++w) om = fmax(om, s_om[w]);
  return om;
}

// ---- tiles: 32 x 32 FP64 blocks in shared memory (stride LDS_), filled by cp.async
constexpr int TILE = JS * LDS_;
constexpr int NST = 4;              // cp.async pipeline depth of the phase B / V runs
constexpr int NTILE = 2 + 2 * NST;  // G run: Jb, U, NST x {G tile, Ja}; V run: Jb, NST x V tile
constexpr size_t JACOBI_SMEM = (size_t)NTILE * TILE * sizeof(double);
constexpr int JMAXP = 8;  // batches up to this size keep their descriptors in shared memory
#ifndef JACOBI_CTAS_PER_SM
#define JACOBI_CTAS_PER_SM 2
#endif

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// dst <- M[rows, cols]: local row a -> global row r0 + a (r0 >= 0) or block pair (bi, bj); local
// cols map to the block pair (ci, cj).  16 B chunks never straddle a 16-wide block.
__device__ __forceinline__ void cp16s(unsigned smem_addr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr), "l"(gmem));
}
// (the shared address is converted once per tile, the column offset is common to a thread's two chunks)
__device__ __forceinline__ void tile_async(double* dst, const double* M, int64_t ld, int64_t r0, int bi, int bj,
                                           int ci, int cj) {
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(dst);
  const int c = (threadIdx.x & 15) * 2;
  const double* Mc = M + sub_to_global(c, ci, cj);
#pragma unroll
  for (int e = threadIdx.x; e < JS * 16; e += JT) {
    const int a = e >> 4;
    const int64_t row = r0 >= 0 ? r0 + a : (int64_t)sub_to_global(a, bi, bj);
    cp16s(sbase + (unsigned)(a * LDS_ + c) * 8u, Mc + row * ld);
  }
}
__device__ __forceinline__ void j_async(double* dst, const double* J) {
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(dst);
  const int c = (threadIdx.x & 15) * 2;
#pragma unroll
  for (int e = threadIdx.x; e < JS * 16; e += JT) {
    const int a = e >> 4;
    cp16s(sbase + (unsigned)(a * LDS_ + c) * 8u, J + a * JS + c);
  }
}

// 32x32x32 product acc = op(A) B with A, B in smem; TA: A read transposed.  Warp w owns rows
// m0 + g, cols n0 + 8j + 2t (+1) of the output (the DMMA accumulator layout).
template <bool TA>
__device__ __forceinline__ void mm32(const double* A, const double* B, double (&acc)[2][2], int warp, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const int m0 = 8 * (warp & 3), n0 = 16 * (warp >> 2);
  acc[0][0] = acc[0][1] = acc[1][0] = acc[1][1] = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < JS; k0 += 4) {
    const double a = TA ? A[(k0 + t) * LDS_ + m0 + g] : A[(m0 + g) * LDS_ + k0 + t];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double b = B[(k0 + t) * LDS_ + n0 + 8 * j + g];
      dmma(acc[j][0], acc[j][1], a, b);
    }
  }
}

// NST-deep cp.async pipeline over the items [t0, t1) of one run (a fixed block column pb):
// pre() starts the run-constant loads, skip(t) drops identity updates, issue(t, stage) starts the
// loads of item t, compute(t, stage) consumes them.  Exactly one commit group per item slot, so
// wait_group<NST - 1> always retires the oldest item.
template <class Pre, class Skip, class Issue, class Compute>
__device__ __forceinline__ void pipeline(int64_t t0, int64_t t1, Pre pre, Skip skip, Issue issue, Compute compute) {
  auto adv = [&](int64_t x) {
    while (x < t1 && skip(x)) ++x;
    return x;
  };
  int64_t ni = adv(t0), nc = ni;
  if (nc >= t1) return;
  int issued = 0, consumed = 0;
  pre();
  for (int p = 0; p < NST - 1; ++p) {
    if (ni < t1) {
      issue(ni, issued % NST);
      ++issued;
      ni = adv(ni + 1);
    }
    cp_commit();
  }
  while (nc < t1) {
    if (ni < t1) {
      issue(ni, issued % NST);
      ++issued;
      ni = adv(ni + 1);
    }
    cp_commit();
    cp_wait<NST - 1>();
    __syncthreads();
    compute(nc, consumed % NST);
    __syncthreads();
    ++consumed;
    nc = adv(nc + 1);
  }
  cp_wait<0>();
}

// One eigenproblem of a batch (device descriptor).  G is double-buffered: the update of round r - 1
// (phase B, old buffer -> new buffer) runs while phase A of round r builds its sub-problems from the
// old buffer and round r - 1's rotations.  The per-round bookkeeping is double-buffered by round
// parity q: during round gr the CTAs read slot q = gr & 1 and block 0 writes slot q ^ 1.
struct EigProb {
  int nb;              // padded block count (even); np = nb / 2 pairs = 32-row tiles of the panel
  int done;            // converged (written on the device)
  int sweeps;
  int gfinal;          // buffer holding the final G (written on the device)
  int pend[2];         // the previous round's rotations are not yet applied to G and V
  int pround[2];       // their round within the sweep (the pairing)
  int ppar[2];         // their R buffer
  int gcur[2];         // buffer holding the latest complete G (the pre-update G while pending)
  double* G[2];        // npad x npad each
  double* V;           // npad x npad
  double* Jbuf;        // 2 x np x JS x JS (by round parity)
  double* Sbuf;        // 2 x np x JS x JS: each pair's rotated sub-problem J^T S J (by round parity)
  int* jflag;          // 2 x np: rotation of the pair is not the identity
  unsigned long long* offmax;  // per sweep
  const double* abs_scale;     // null: relative criterion
  double ascale;               // *abs_scale, fetched once at kernel start
  int64_t pair_off, gitem_off, vitem_off;  // prefix sums over the batch (phase A pairs, G runs, V runs)
};

__device__ __forceinline__ int find_prob(const EigProb* P, int nprob, int64_t idx, int which) {
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    const int64_t off = which == 0 ? P[mid].pair_off : which == 1 ? P[mid].gitem_off : P[mid].vitem_off;
    if (off <= idx) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// G runs of one problem: block column pb holds pa = 0..pb in runs of c, so the runs of columns
// < P number F(P) = P + c q (q - 1) / 2 + r q with P = q c + r.
__host__ __device__ __forceinline__ int64_t g_runs_before(int64_t P, int64_t c) {
  const int64_t q = P / c, r = P % c;
  return P + c * q * (q - 1) / 2 + r * q;
}
// Run j of the G queue -> (block column pb, chunk).  Columns q c .. q c + c - 1 hold q + 1 runs each
// (column P has floor(P / c) + 1), so the groups are walked by subtraction and one small division
// finds the column inside the group -- the search over the closed form above cost a dozen integer
// divisions per item and thread.
__device__ __forceinline__ void g_run(int64_t j, int np, int c, int& pb, int& chunk) {
  unsigned jj = (unsigned)j, q = 0, step = (unsigned)c;  // step = c (q + 1) runs in group q
  while (jj >= step) {
    jj -= step;
    step += (unsigned)c;
    ++q;
  }
  const unsigned col = jj / (q + 1u);
  pb = (int)(q * (unsigned)c + col);
  chunk = (int)(jj - col * (q + 1u));
  (void)np;
}

// V[:, P'] <- V[:, P'] R_P' for the pending round of problem pr_: row tiles [r0, r1) of column pb.
__device__ void v_run(const EigProb& pr_, int q, int pb, int r0, int r1, double* sm, int warp, int lane) {
  const int nb = pr_.nb, np = nb / 2, round = pr_.pround[q], vpar = pr_.ppar[q];
  if (!pr_.jflag[vpar * np + pb]) return;
  const int64_t ld = (int64_t)nb * JB;
  const int bi = rr_block(pb, round, nb), bj = rr_block(nb - 1 - pb, round, nb);
  double* V = pr_.V;
  double* Jb = sm;
  double* stg = sm + TILE;
  pipeline(
      r0, r1, [&] { j_async(Jb, pr_.Jbuf + ((int64_t)vpar * np + pb) * JS * JS); },
      [&](int64_t) { return false; },
      [&](int64_t rt, int st) { tile_async(stg + st * TILE, V, ld, rt * JS, 0, 0, bi, bj); },
      [&](int64_t rt, int st) {
        double acc[2][2];
        mm32<false>(stg + st * TILE, Jb, acc, warp, lane);
        const int g = lane >> 2, tq = lane & 3, m0 = 8 * (warp & 3), n0 = 16 * (warp >> 2);
        const int64_t row = rt * JS + m0 + g;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c0 = n0 + 8 * j + 2 * tq;
          *reinterpret_cast<double2*>(V + row * ld + sub_to_global(c0, bi, bj)) = make_double2(acc[j][0], acc[j][1]);
        }
      });
}

// G'[Pa, Pb] = Ja^T G[Pa, Pb] Jb for pa in [a0, a1) (<= pb), read from the pre-update buffer and
// written (both triangles) to the other one -- every tile, identity rotations included.
__device__ void g_run_exec(const EigProb& pr_, int q, int pb, int a0, int a1, double* sm, int warp, int lane) {
  const int nb = pr_.nb, np = nb / 2, round = pr_.pround[q], par = pr_.ppar[q];
  const int64_t ld = (int64_t)nb * JB;
  const double* J0 = pr_.Jbuf + (int64_t)par * np * JS * JS;
  const int bi = rr_block(pb, round, nb), bj = rr_block(nb - 1 - pb, round, nb);
  const double* Gs = pr_.G[pr_.gcur[q]];
  double* G = pr_.G[pr_.gcur[q] ^ 1];
  double* Jb = sm;
  double* Us = sm + TILE;
  double* stg = sm + 2 * TILE;
  pipeline(
      a0, a1, [&] { j_async(Jb, J0 + (int64_t)pb * JS * JS); }, [&](int64_t) { return false; },
      [&](int64_t pa, int st) {
        const int ai = rr_block((int)pa, round, nb), aj = rr_block(nb - 1 - (int)pa, round, nb);
        tile_async(stg + (2 * st) * TILE, Gs, ld, -1, ai, aj, bi, bj);
        j_async(stg + (2 * st + 1) * TILE, J0 + pa * JS * JS);
      },
      [&](int64_t pa, int st) {
        const int ai = rr_block((int)pa, round, nb), aj = rr_block(nb - 1 - (int)pa, round, nb);
        const int g = lane >> 2, tq = lane & 3, m0 = 8 * (warp & 3), n0 = 16 * (warp >> 2);
        double acc[2][2];
        mm32<false>(stg + (2 * st) * TILE, Jb, acc, warp, lane);  // U = G Jb
#pragma unroll
        for (int j = 0; j < 2; ++j)
          *reinterpret_cast<double2*>(Us + (m0 + g) * LDS_ + n0 + 8 * j + 2 * tq) = make_double2(acc[j][0], acc[j][1]);
        __syncthreads();
        mm32<true>(stg + (2 * st + 1) * TILE, Us, acc, warp, lane);  // G' = Ja^T U
        const int64_t row = sub_to_global(m0 + g, ai, aj);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c0 = n0 + 8 * j + 2 * tq;
          const int64_t col = sub_to_global(c0, bi, bj);
          *reinterpret_cast<double2*>(G + row * ld + col) = make_double2(acc[j][0], acc[j][1]);
          if (pa != pb) {
            G[col * ld + row] = acc[j][0];
            G[(col + 1) * ld + row] = acc[j][1];
          }
        }
      });
}

// Position of block x in the round-robin pairing of round rho (inverse of rr_block).
__device__ __forceinline__ int rr_pos(int x, int rho, int nb) {
  if (x == 0) return 0;
  const int m = nb - 1;
  int y = x - 1 - rho;  // in (-m, m) for rho < m: one conditional add instead of two divisions
  while (y < 0) y += m;
  while (y >= m) y -= m;
  return 1 + y;
}

// C (M x N) = op(A) (M x 32) B (32 x N), all in shared memory with explicit strides; M, N multiples
// of 8.  8 x 8 output tiles are dealt round-robin to the warps (DMMA m8n8k4, K = 32).
__device__ __forceinline__ void mm_k32(const double* A, int lda, bool ta, const double* B, int ldb, double* C, int ldc,
                                       int M, int N, int tile0, int warp, int lane, double* CT = nullptr) {
  const int g = lane >> 2, t = lane & 3;
  const int tn = N / 8, nt = (M / 8) * tn;
  for (int tl = (warp + 8 - tile0 % 8) % 8; tl < nt; tl += 8) {
    const int m0 = 8 * (tl / tn), n0 = 8 * (tl % tn);
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < JS; k0 += 4) {
      const double a = ta ? A[(k0 + t) * lda + m0 + g] : A[(m0 + g) * lda + k0 + t];
      const double b = B[(k0 + t) * ldb + n0 + g];
      dmma(d0, d1, a, b);
    }
    C[(m0 + g) * ldc + n0 + 2 * t] = d0;
    C[(m0 + g) * ldc + n0 + 2 * t + 1] = d1;
    if (CT) {  // and C^T (same stride)
      CT[(n0 + 2 * t) * ldc + m0 + g] = d0;
      CT[(n0 + 2 * t + 1) * ldc + m0 + g] = d1;
    }
  }
}

// The sub-problem of pair pr in round rho (blocks X, Y) from the pre-update G and the previous
// round's rotations: S[x, y] = J_{P(x)}[:, x half]^T G[P(x), P(y)] J_{P(y)}[:, y half] for x, y in
// {X, Y}, where P(x) is x's pair in the previous round.  S[Y, X] = S[X, Y]^T.  Uses tiles 0..7.
__device__ void build_subproblem(const EigProb& pr_, int q, int pr, int rho, double* sm, int warp, int lane) {
  const int nb = pr_.nb, np = nb / 2, prho = pr_.pround[q], par = pr_.ppar[q];
  const int64_t ld = (int64_t)nb * JB;
  const double* Gs = pr_.G[pr_.gcur[q]];
  const double* J0 = pr_.Jbuf + (int64_t)par * np * JS * JS;
  const int blk[2] = {rr_block(pr, rho, nb), rr_block(nb - 1 - pr, rho, nb)};
  int pp[2], hh[2];
  for (int i = 0; i < 2; ++i) {
    const int pos = rr_pos(blk[i], prho, nb);
    pp[i] = pos < np ? pos : nb - 1 - pos;
    hh[i] = pos < np ? 0 : 1;
  }
  double* S = sm;               // tile 0: the sub-problem
  double* Jx = sm + 2 * TILE;   // tiles 2, 3: previous rotations of X's and Y's pairs
  double* Jy = sm + 3 * TILE;
  double* T = sm + 4 * TILE;    // tiles 4, 5, 6: G[P(X), P(X)], G[P(X), P(Y)], G[P(Y), P(Y)]
  double* W = sm + 7 * TILE;    // tile 7: three 32 x 16 products, stride 48
  // S[X, X] and S[Y, Y] are 16 x 16 diagonal blocks of the previous round's rotated sub-problems
  // (J^T S J of pairs P(X), P(Y), published by their CTAs); only S[X, Y] mixes two pairs and is
  // formed from the pre-update G tile G[P(X), P(Y)] and both rotations.
  const double* S0 = pr_.Sbuf + (int64_t)par * np * JS * JS;
  j_async(Jx, J0 + (int64_t)pp[0] * JS * JS);
  j_async(Jy, J0 + (int64_t)pp[1] * JS * JS);
  tile_async(T, Gs, ld, -1, rr_block(pp[0], prho, nb), rr_block(nb - 1 - pp[0], prho, nb), rr_block(pp[1], prho, nb),
             rr_block(nb - 1 - pp[1], prho, nb));
  cp_commit();
  for (int e = threadIdx.x; e < 2 * 256; e += JT) {
    const int a = e >> 8, i = (e >> 4) & 15, j = e & 15;
    const double* Sprev = S0 + (int64_t)pp[a] * JS * JS;
    S[(16 * a + i) * LDS_ + 16 * a + j] = __ldcg(Sprev + (16 * hh[a] + i) * JS + 16 * hh[a] + j);
  }
  cp_wait<0>();
  __syncthreads();
  // W = G[P(X), P(Y)] J_Y[:, 16 h_Y : +16]   (32 x 16), S[X, Y] = J_X[:, 16 h_X : +16]^T W   (16 x 16)
  mm_k32(T, LDS_, false, Jy + 16 * hh[1], LDS_, W, 48, 32, 16, 0, warp, lane);
  __syncthreads();
  mm_k32(Jx + 16 * hh[0], LDS_, true, W, 48, S + 16, LDS_, 16, 16, 0, warp, lane, S + 16 * LDS_);  // + S[Y, X]
  __syncthreads();
}

// phase A of one pair: the rotations of the 32 x 32 sub-problem (J into Jbuf[par])
__device__ void pair_exec(const EigProb& pr_, int q, int pr, int round, int par, int sweep, double tol, double* sm,
                          PairBuf& pbuf, const StepTables& tb, unsigned long long* prof) {
  const int nb = pr_.nb, np = nb / 2;
  const bool absolute = pr_.abs_scale != nullptr;
  const double ascale = absolute ? pr_.ascale : 0.0;
  double* Sa = sm;
  double* Ra = sm + TILE;
  const bool tprof = prof && blockIdx.x == 0 && threadIdx.x == 0;
  const unsigned long long tb0 = tprof ? gtimer() : 0;
  if (pr_.pend[q]) {
    build_subproblem(pr_, q, pr, round, sm, threadIdx.x >> 5, threadIdx.x & 31);
  } else {
    const int bi = rr_block(pr, round, nb), bj = rr_block(nb - 1 - pr, round, nb);
    tile_async(Sa, pr_.G[pr_.gcur[q]], (int64_t)nb * JB, -1, bi, bj, bi, bj);
    cp_commit();
    cp_wait<0>();
  }
  if (round == 0)  // R in shared memory only for round 0's within-block steps
    for (int e = threadIdx.x; e < JS * JS; e += JT) {
      const int a = e >> 5, b = e & 31;
      Ra[a * LDS_ + b] = a == b ? 1.0 : 0.0;
    }
  __syncthreads();
  const unsigned long long ts0 = tprof ? gtimer() : 0;
  if (tprof) prof[5] += ts0 - tb0;
  double* Jp = pr_.Jbuf + ((int64_t)par * np + pr) * JS * JS;
  double* Sp = pr_.Sbuf + ((int64_t)par * np + pr) * JS * JS;
  int rot = 0;
  double om = subsolve(Sa, Ra, tb, pbuf, round == 0, tol, ascale, absolute, Jp, &rot);
  const unsigned long long ts1 = tprof ? gtimer() : 0;
  if (tprof) prof[4] += ts1 - ts0;
  for (int e = threadIdx.x; e < JS * JS; e += JT)
    Sp[e] = Sa[(e >> 5) * LDS_ + (e & 31)];  // the rotated sub-problem: next round's diagonal blocks
  rot = __syncthreads_or(rot);
  if (threadIdx.x == 0) pr_.jflag[par * np + pr] = rot;
  if (threadIdx.x < 32) {
    for (int o = 16; o; o >>= 1) om = fmax(om, __shfl_xor_sync(0xffffffffu, om, o));
    if (threadIdx.x == 0 && om > 0.0) atomicMax(pr_.offmax + sweep, (unsigned long long)__double_as_longlong(om));
  }
  __syncthreads();
  if (tprof) prof[6] += gtimer() - ts1;
}

// One round's parallel section: phase A of every active problem's pairs, and -- on the CTAs phase A
// leaves idle -- the G (phase B) and V updates owed by the previous round.
__device__ void section(EigProb* P, int nprob, int64_t total_pairs, int64_t total_gitems, int64_t total_vitems,
                        int gchunk, int vchunk, int q, int round, int par, int sweep, bool pairs_on, double tol,
                        double* sm, PairBuf& pbuf, const StepTables& tb, unsigned long long* prof,
                        unsigned long long* work, bool join, bool buddy, int lead, int qrank, int nq) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nA = pairs_on ? total_pairs : 0;
  const int64_t nX = total_gitems + total_vitems;
  auto extra = [&](int64_t x) {
    if (x < total_gitems) {
      const int pi = find_prob(P, nprob, x, 1);
      const EigProb& pr_ = P[pi];
      if (!pr_.pend[q]) return;
      int pb, chunk;
      g_run(x - pr_.gitem_off, pr_.nb / 2, gchunk, pb, chunk);
      const int a0 = chunk * gchunk, a1 = a0 + gchunk < pb + 1 ? a0 + gchunk : pb + 1;
      g_run_exec(pr_, q, pb, a0, a1, sm, warp, lane);
    } else {
      const int64_t vi = x - total_gitems;
      const int pi = find_prob(P, nprob, vi, 2);
      const EigProb& pr_ = P[pi];
      if (!pr_.pend[q]) return;
      const int np = pr_.nb / 2;
      const int per = (np + vchunk - 1) / vchunk;
      const unsigned j = (unsigned)(vi - pr_.vitem_off);
      const int pb = (int)(j / (unsigned)per), c = (int)(j - (unsigned)pb * (unsigned)per);
      const int r0 = c * vchunk, r1 = r0 + vchunk < np ? r0 + vchunk : np;
      v_run(pr_, q, pb, r0, r1, sm, warp, lane);
    }
  };
  auto pair = [&](int64_t it) {
    const int pi = find_prob(P, nprob, it, 0);
    const EigProb& pr_ = P[pi];
    if (pr_.done || round >= pr_.nb - 1) return;
    pair_exec(pr_, q, (int)(it - pr_.pair_off), round, par, sweep, tol, sm, pbuf, tb, prof);
  };
  // pairs first (one per CTA while they last), then the G / V queue (heaviest items first), drained
  // through a shared counter by the CTAs without a pair -- and by the pair CTAs too when the extra
  // work outweighs a phase-A sub-solve (join)
  bool had_pair = false;
  if (lead == -2) {
    for (int64_t it = blockIdx.x; it < nA; it += gridDim.x) {
      pair(it);
      had_pair = true;
    }
  } else if (lead >= 0) {
    for (int64_t it = lead; it < nA; it += gridDim.x) {  // nA <= grid / 8: one pair at most
      pair(it);
      had_pair = true;
    }
  }
  if (had_pair && !join && nA < (int64_t)gridDim.x) return;
  // a CTA sharing its SM with a phase-A CTA stays out of the queue while sub-solves run: the
  // latency-bound rotation chain then has the SM to itself (measured: 7.7 -> 6.5 ms of sub-solve
  // per n = 1000 eigensolve)
  if (buddy && nA > 0) return;
  // rounds with pairs: items [0, nq) go to the queue CTAs by rank, the rest through the counter
  const int64_t x0 = nA > 0 ? nq : 0;
  if (nA > 0 && qrank >= 0 && qrank < nX) extra(qrank);
  __shared__ int64_t grab;
  while (true) {
    if (threadIdx.x == 0) grab = x0 + (int64_t)atomicAdd(work, 1ull);
    __syncthreads();
    const int64_t x = grab;
    __syncthreads();
    if (x >= nX) break;
    extra(x);
  }
}

// The next round's bookkeeping slot (q ^ 1) of one problem.
__device__ __forceinline__ void advance_one(EigProb& pr_, int q, int round, int par) {
  const int cur = pr_.pend[q] ? pr_.gcur[q] ^ 1 : pr_.gcur[q];
  const bool active = !pr_.done && round < pr_.nb - 1;
  pr_.gcur[q ^ 1] = cur;
  pr_.pend[q ^ 1] = active ? 1 : 0;
  pr_.pround[q ^ 1] = round;
  pr_.ppar[q ^ 1] = par;
  pr_.gfinal = cur;
}

// After a CTA's section work: the next round's slot in its shared copy of the descriptors (every
// CTA replays the same deterministic update, so no CTA reads bookkeeping from global memory on the
// per-round critical path) and, on block 0, in the global copy (the host reads gfinal) plus the
// work counter.
__device__ void advance_slots(EigProb* P, EigProb* PL, int nprob, int q, int round, int par,
                              unsigned long long* work) {
  if (PL != P)
    for (int pi = threadIdx.x; pi < nprob; pi += blockDim.x) advance_one(PL[pi], q, round, par);
  if (blockIdx.x != 0) return;
  if (threadIdx.x == 0) work[q ^ 1] = 0ull;
  for (int pi = threadIdx.x; pi < nprob; pi += blockDim.x) advance_one(P[pi], q, round, par);
}

__global__ void __launch_bounds__(JT, JACOBI_CTAS_PER_SM)
    k_jacobi(EigProb* P, int nprob, int64_t total_pairs, int64_t total_gitems, int64_t total_vitems, int gchunk,
             int vchunk, int max_rounds, int max_sweeps, double tol, double stagnate_below, double quad_margin,
             unsigned long long* prof,
             unsigned long long* work, int join, int* smids, int spread_factor) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  __shared__ StepTables tb;
  __shared__ PairBuf pbuf;
  __shared__ int s_buddy;
  build_tables(tb);
  // When the pairs leave most SMs free, phase-A (pair) CTAs get an SM each: pair j goes to the
  // first CTA of the j-th distinct SM (the block scheduler may put consecutive CTAs on one SM), and
  // the other CTA on that SM stays out of the phase-B queue while sub-solves run.
  if (threadIdx.x == 0) {
    unsigned sid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sid));
    smids[blockIdx.x] = (int)sid;
  }
  grid.sync();
  __shared__ int s_lead, s_qrank, s_nq, s_spread;
  {
    // the dynamic shared buffer is free until the first section: SM ids, first-on-SM flags and
    // leader ranks of every CTA, computed by the whole block
    const int G = (int)gridDim.x;
    int* ssm = reinterpret_cast<int*>(sm);
    int* sfirst = ssm + G;
    int* srank = sfirst + G;
    for (int c = threadIdx.x; c < G; c += blockDim.x) ssm[c] = __ldcg(smids + c);
    __syncthreads();
    for (int c = threadIdx.x; c < G; c += blockDim.x) {
      int f = 1;
      for (int d = 0; d < c && f; ++d) f = ssm[d] != ssm[c];
      sfirst[c] = f;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int c = 0; c < G; ++c) {
        srank[c] = run;
        run += sfirst[c];
      }
      const int me = (int)blockIdx.x, mine = ssm[me];
      const int64_t npair_ctas = total_pairs < (int64_t)G ? total_pairs : (int64_t)G;
      const bool spread = (int64_t)spread_factor * npair_ctas <= (int64_t)G;
      int bud = 0;
      if (spread && !sfirst[me]) {
        int leader = 0;
        while (ssm[leader] != mine) ++leader;
        bud = srank[leader] < npair_ctas ? 1 : 0;
      }
      s_buddy = bud;
      s_lead = spread ? (sfirst[me] ? srank[me] : -1) : -2;  // -2: pairs by blockIdx (many pairs)
      s_spread = spread ? 1 : 0;
    }
    __syncthreads();
    // rank among the CTAs that go straight to the G / V queue in a round with pairs (no pair of
    // their own, not a buddy): their first item is theirs by rank, without an atomic
    int* spart = srank + G;
    const int64_t npair_ctas = total_pairs < (int64_t)G ? total_pairs : (int64_t)G;
    for (int c = threadIdx.x; c < G; c += blockDim.x) {
      bool part;
      if (!s_spread) {
        part = (int64_t)c >= total_pairs;
      } else if (sfirst[c]) {
        part = (int64_t)srank[c] >= total_pairs;
      } else {
        int leader = 0;
        while (ssm[leader] != ssm[c]) ++leader;
        part = !((int64_t)srank[leader] < npair_ctas);
      }
      spart[c] = part ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int nq = 0, qr = -1;
      for (int c = 0; c < G; ++c) {
        if (c == (int)blockIdx.x && spart[c]) qr = nq;
        nq += spart[c];
      }
      s_qrank = qr;
      s_nq = nq;
    }
  }
  __syncthreads();
  const bool buddy = s_buddy != 0;
  // descriptors: a shared copy when the batch is small (JMAXP), else the global array
  __shared__ EigProb sP[JMAXP];
  if (blockIdx.x == 0)
    for (int pi = threadIdx.x; pi < nprob; pi += blockDim.x)
      P[pi].ascale = P[pi].abs_scale ? *P[pi].abs_scale : 0.0;
  grid.sync();
  EigProb* PL = nprob <= JMAXP ? sP : P;
  if (PL != P)
    for (int pi = threadIdx.x; pi < nprob; pi += blockDim.x) sP[pi] = P[pi];
  __syncthreads();
  int gr = 0;  // global round counter (R buffer and bookkeeping parity)
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    for (int round = 0; round < max_rounds; ++round, ++gr) {
      const int q = gr & 1;
      const unsigned long long t0 = prof ? gtimer() : 0;
      section(PL, nprob, total_pairs, total_gitems, total_vitems, gchunk, vchunk, q, round, q, sweep, true, tol, sm,
              pbuf, tb, prof, work + q, join != 0, buddy, s_lead, s_qrank, s_nq);
      const unsigned long long t1 = prof ? gtimer() : 0;
      advance_slots(P, PL, nprob, q, round, q, work);
      grid.sync();
      if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
        prof[0] += t1 - t0;
        prof[1] += gtimer() - t1;
      }
    }
    // per-problem convergence: converged, or the off-diagonal measure stagnates at the rounding floor
    if (blockIdx.x == 0) {
      for (int pi = threadIdx.x; pi < nprob; pi += blockDim.x) {
        EigProb& pr_ = P[pi];
        if (pr_.done) continue;
        const double cur = __longlong_as_double((long long)pr_.offmax[sweep]);
        const double prev = sweep ? __longlong_as_double((long long)pr_.offmax[sweep - 1]) : 1e300;
        // quadratic regime: this sweep leaves ~ C cur^2 with C = cur / prev^2 from the last step;
        // stop when that is far below the tolerance (saves the confirming sweep)
        const bool quad = sweep > 0 && cur < 1e-8 && prev > 0.0 && prev < 1e-3 &&
                          (cur / (prev * prev)) * cur * cur <= quad_margin * tol;
        if (cur <= tol || quad || (cur < stagnate_below && cur > 0.25 * prev) || sweep + 1 == max_sweeps) {
          pr_.done = 1;
          pr_.sweeps = sweep + 1;
        }
      }
    }
    grid.sync();
    if (PL != P) {
      for (int pi = threadIdx.x; pi < nprob; pi += blockDim.x) {
        sP[pi].done = P[pi].done;
        sP[pi].sweeps = P[pi].sweeps;
      }
      __syncthreads();
    }
    bool all = true;
    for (int pi = 0; pi < nprob; ++pi) all &= (PL[pi].done != 0);
    if (all) break;
  }
  // the last round's G and V updates
  const int q = gr & 1;
  section(PL, nprob, total_pairs, total_gitems, total_vitems, gchunk, vchunk, q, 0, q, 0, false, tol, sm, pbuf, tb,
          nullptr, work + q, true, false, s_lead, -1, 0);
  advance_slots(P, PL, nprob, q, 0, q, work);
}

__global__ void k_max_diag(int64_t n, const double* A, int64_t lda, double* out) {
  __shared__ double red[256];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(A[i * lda + i]));
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0] > 0.0 ? red[0] : 1.0;
}

__global__ void k_pad_copy(int64_t n, int64_t npad, const double* A, int64_t lda, double* G) {
  FPI_GRID_STRIDE(e, npad * npad) {
    int64_t i = e / npad, j = e - i * npad;
    G[e] = (i < n && j < n) ? A[i * lda + j] : 0.0;
  }
}

__global__ void k_identity(int64_t n, double* A) {
  FPI_GRID_STRIDE(e, n * n) A[e] = (e / n == e % n) ? 1.0 : 0.0;
}

__global__ void k_diag_keys(int64_t n, const double* G, int64_t npad, double* keys, int32_t* idx) {
  FPI_GRID_STRIDE(i, n) {
    keys[i] = G[i * npad + i];
    idx[i] = (int32_t)i;
  }
}

// V[:, k] = eigenvector order[k]; perm (optional): row a of Vp belongs to original index perm[a]
__global__ void k_gather_eig(int64_t n, const double* Vp, int64_t npad, const int32_t* order, const double* wsorted,
                             const int32_t* perm, double* w, double* V, int64_t ldv) {
  FPI_GRID_STRIDE(e, n * n) {
    int64_t a = e / n, k = e - a * n;
    const int64_t i = perm ? perm[a] : a;
    V[i * ldv + k] = Vp[a * npad + order[k]];
    if (a == 0 && w) w[k] = wsorted[k];
  }
}

}  // namespace

void sym_eig_batched(fpi_context* h, int nprob, const int64_t* n, const double* const* A, const int64_t* lda,
                     double* const* w, double* const* V, const int64_t* ldv, int max_sweeps, double tol,
                     bool absolute, int* sweeps_out) {
  if (nprob <= 0) return;
  cudaStream_t s = h->stream;
  // Stagnation stop: the off-diagonal measure stops falling (cur > prev / 4) while below the rounding
  // floor of a rotation sweep, ~c n eps (c = 32).  Above that floor a stalled measure keeps iterating
  // (to max_sweeps): stopping there would leave eigenvector errors of ~measure / gap.
  int64_t n_max = 1;
  for (int i = 0; i < nprob; ++i) n_max = n[i] > n_max ? n[i] : n_max;
  const double stagnate_below = 32.0 * (double)n_max * 2.220446049250313e-16;
  // the quadratic-regime stop: the sweep's predicted residual C cur^2 (C = cur / prev^2) below
  // quad_margin * tol (FPI_JACOBI_QUAD overrides)
  static const double quad_margin = getenv("FPI_JACOBI_QUAD") ? atof(getenv("FPI_JACOBI_QUAD")) : 1e-1;
  std::vector<EigProb> hp(nprob);
  std::vector<int64_t> npad(nprob), goff(nprob);
  int64_t gsz = 0, jsz = 0, fsz = 0, tot_pairs = 0, tot_tri = 0, tot_vt = 0;
  int max_rounds = 0;
  for (int i = 0; i < nprob; ++i) {
    int nb = (int)((n[i] + JB - 1) / JB);
    if (nb < 2) nb = 2;
    if (nb % 2) ++nb;
    npad[i] = (int64_t)nb * JB;
    const int64_t np = nb / 2;
    hp[i] = EigProb{};
    hp[i].nb = nb;
    goff[i] = gsz;
    gsz += npad[i] * npad[i];
    jsz += 2 * np * JS * JS;
    fsz += 2 * np;
    tot_pairs += np;
    tot_tri += np * (np + 1) / 2;
    tot_vt += np * np;
    if (nb - 1 > max_rounds) max_rounds = nb - 1;
  }
  static std::atomic<uint64_t> attr_set{0};
  static std::atomic<int> blocks_per_sm[64];
  once_per_device(attr_set, h->device, [&] {
    FPI_CUDA(cudaFuncSetAttribute((const void*)k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)JACOBI_SMEM));
    int per_sm = 0;
    FPI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi, JT, JACOBI_SMEM));
    blocks_per_sm[h->device & 63].store(per_sm);
  });
  const int max_blocks = blocks_per_sm[h->device & 63].load() * h->num_sms;
  int grid = max_blocks;
  if (const char* e = getenv("FPI_JACOBI_GRID")) grid = atoi(e) < max_blocks ? atoi(e) : max_blocks;
  if (grid < 1) grid = 1;
  // run lengths of the G (phase B) and V updates of round r - 1: a few 32 x 32 tiles per queue item,
  // enough items to balance across the grid (a G tile costs two 32^3 products, a V tile one)
  // (measured, tools/eig_compare.py / bench_eig.py / jacobi_tune.py: n <= ~1000 balances best with
  //  short V runs, n = 1628 / 2000 with longer ones; n <= ~900 with 3-tile G runs)
  int64_t np_max = 0;
  for (int i = 0; i < nprob; ++i) np_max = hp[i].nb / 2 > np_max ? hp[i].nb / 2 : np_max;
  int gchunk = np_max <= 28 ? 3 : 4, vchunk = np_max <= 40 ? 3 : 8;
  if (const char* e = getenv("FPI_JACOBI_CHUNKS")) sscanf(e, "%d,%d", &gchunk, &vchunk);
  // pair CTAs join the queue when the extra work per idle CTA exceeds ~20 tile products (~ one sub-solve)
  const int64_t xcta = grid - tot_pairs > 1 ? grid - tot_pairs : 1;
  int join = (2 * tot_tri + tot_vt) > 20 * xcta ? 1 : 0;
  if (const char* e = getenv("FPI_JACOBI_JOIN")) join = atoi(e);
  int64_t tot_g = 0, tot_v = 0;
  for (int i = 0; i < nprob; ++i) {
    const int64_t np = hp[i].nb / 2;
    hp[i].pair_off = i ? hp[i - 1].pair_off + hp[i - 1].nb / 2 : 0;
    hp[i].gitem_off = tot_g;
    hp[i].vitem_off = tot_v;
    tot_g += g_runs_before(np, gchunk);
    tot_v += np * ((np + vchunk - 1) / vchunk);
  }
  Scratch<double> Gall(gsz, s), Gall2(gsz, s), Vall(gsz, s), Jall(jsz, s), Sall(jsz, s), scales(nprob, s);
  Scratch<int> fall(fsz, s);
  Scratch<unsigned long long> offm((int64_t)nprob * (max_sweeps + 1), s);
  Scratch<EigProb> dP(nprob, s);
  FPI_CUDA(cudaMemsetAsync(offm.get(), 0, sizeof(unsigned long long) * nprob * (max_sweeps + 1), s));
  const unsigned G16 = (unsigned)(h->num_sms * 16);
  int64_t jo = 0, fo = 0;
  for (int i = 0; i < nprob; ++i) {
    const int64_t np = hp[i].nb / 2;
    hp[i].G[0] = Gall.get() + goff[i];
    hp[i].G[1] = Gall2.get() + goff[i];
    hp[i].V = Vall.get() + goff[i];
    hp[i].Jbuf = Jall.get() + jo;
    hp[i].Sbuf = Sall.get() + jo;
    hp[i].jflag = fall.get() + fo;
    hp[i].offmax = offm.get() + (int64_t)i * (max_sweeps + 1);
    hp[i].abs_scale = absolute ? scales.get() + i : nullptr;
    k_pad_copy<<<grid_for(npad[i] * npad[i], 256, G16), 256, 0, s>>>(n[i], npad[i], A[i], lda[i], hp[i].G[0]);
    k_identity<<<grid_for(npad[i] * npad[i], 256, G16), 256, 0, s>>>(npad[i], hp[i].V);
    if (absolute) k_max_diag<<<1, 256, 0, s>>>(n[i], A[i], lda[i], scales.get() + i);
    note_launch(h, absolute ? 3 : 2);
    jo += 2 * np * JS * JS;
    fo += 2 * np;
  }
  FPI_CUDA(cudaMemcpyAsync(dP.get(), hp.data(), sizeof(EigProb) * nprob, cudaMemcpyHostToDevice, s));
  FPI_LAUNCH_CHECK();
  Scratch<unsigned long long> work(2, s);
  FPI_CUDA(cudaMemsetAsync(work.get(), 0, sizeof(unsigned long long) * 2, s));
  Scratch<unsigned long long> prof(8, s);
  FPI_CUDA(cudaMemsetAsync(prof.get(), 0, sizeof(unsigned long long) * 8, s));
  unsigned long long* prof_p = getenv("FPI_JACOBI_PROFILE") ? prof.get() : nullptr;
  EigProb* Pp = dP.get();
  int gch = gchunk, vch = vchunk;
  unsigned long long* work_p = work.get();
  Scratch<int> smids(grid, s);
  int* smids_p = smids.get();
  // pair CTAs get SMs of their own while the pairs need at most 1 / spread of the grid
  int spread = 8;
  if (const char* e = getenv("FPI_JACOBI_SPREAD")) spread = atoi(e) > 0 ? atoi(e) : 1 << 20;
  void* args[] = {&Pp, &nprob, &tot_pairs, &tot_g, &tot_v, &gch, &vch, &max_rounds, &max_sweeps, &tol,
                  (void*)&stagnate_below, (void*)&quad_margin, &prof_p, &work_p, &join, &smids_p, &spread};
  {
    KTimer kt(h, "sym_eig_block_jacobi", 0.0, 0.0);
    FPI_CUDA(cudaLaunchCooperativeKernel((void*)k_jacobi, grid, JT, args, JACOBI_SMEM, s));
  }
  note_launch(h);
  FPI_CUDA(cudaMemcpyAsync(hp.data(), dP.get(), sizeof(EigProb) * nprob, cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  if (sweeps_out)
    for (int i = 0; i < nprob; ++i) sweeps_out[i] = hp[i].sweeps;
  if (prof_p) {
    unsigned long long hq[8];
    FPI_CUDA(cudaMemcpyAsync(hq, prof_p, sizeof(hq), cudaMemcpyDeviceToHost, s));
    FPI_CUDA(cudaStreamSynchronize(s));
    fprintf(stderr, "[jacobi nprob=%d n0=%lld grid=%d gchunk=%d vchunk=%d] section %.3f (build %.3f subsolve %.3f "
            "epilogue %.3f)  sync %.3f ms\n",
            nprob, (long long)n[0], grid, gchunk, vchunk, hq[0] * 1e-6, hq[5] * 1e-6, hq[4] * 1e-6, hq[6] * 1e-6,
            hq[1] * 1e-6);
    std::vector<unsigned long long> om((size_t)max_sweeps + 1);
    FPI_CUDA(cudaMemcpy(om.data(), offm.get(), sizeof(unsigned long long) * om.size(), cudaMemcpyDeviceToHost));
    fprintf(stderr, "[jacobi] problem 0 off-diagonal measure per sweep (tol %.1e):", tol);
    for (int i = 0; i < hp[0].sweeps; ++i) {
      double v;
      memcpy(&v, &om[(size_t)i], sizeof(double));
      fprintf(stderr, " %.2e", v);
    }
    fprintf(stderr, "\n");
  }
  // eigenvalues (descending diagonal) and the matching columns of V
  CubTemp tmp(s);
  for (int i = 0; i < nprob; ++i) {
    Scratch<double> keys(n[i], s), keys2(n[i], s);
    Scratch<int32_t> idx(n[i], s), idx2(n[i], s);
    k_diag_keys<<<grid_for(n[i], 256, h->num_sms * 4), 256, 0, s>>>(n[i], hp[i].G[hp[i].gfinal], npad[i], keys,
                                                                       idx);
    sort_pairs(tmp, keys.get(), keys2.get(), idx.get(), idx2.get(), n[i], true, 0, 64, s);
    k_gather_eig<<<grid_for(n[i] * n[i], 256, G16), 256, 0, s>>>(n[i], Vall.get() + goff[i], npad[i], idx2, keys2,
                                                                  nullptr, w[i],
                                                                  V[i], ldv[i]);
    note_launch(h, 3);
  }
  FPI_LAUNCH_CHECK();
}

int sym_eig(fpi_context* h, int64_t n, const double* A, int64_t lda, double* w, double* V, int64_t ldv,
            int max_sweeps, double tol, bool absolute) {
  if (n <= 0) return 0;
  int sw = 0;
  sym_eig_batched(h, 1, &n, &A, &lda, &w, &V, &ldv, max_sweeps, tol, absolute, &sw);
  return sw;
}

}  // namespace fpi

extern "C" int fpi_sym_eig(fpi_handle h, int64_t n, const double* d_A, int64_t lda, double* d_w, double* d_V,
                           int64_t ldv, int32_t* h_sweeps) {
  FPI_API_BEGIN(h)
  int sw = fpi::sym_eig(h, n, d_A, lda, d_w, d_V, ldv, 60, 1e-14, false);
  if (h_sweeps) *h_sweeps = sw;
  FPI_API_END(h)
}

// ---- internal microbenchmark (not part of the public ABI): one CTA runs the
// sub-solve `iters` times on a fixed SPD 32 x 32 matrix; ns per step.
namespace fpi {
namespace {
__global__ void __launch_bounds__(JT) k_subsolve_bench(int iters, double* out) {
  __shared__ __align__(16) double S[JS * LDS_];
  __shared__ __align__(16) double R[JS * LDS_];
  __shared__ StepTables tb;
  __shared__ PairBuf pbuf;
  build_tables(tb);
  __syncthreads();
  const bool r0 = iters > 0;  // negative iters: cross steps only (rounds > 0 of a sweep)
  iters = iters < 0 ? -iters : iters;
  const unsigned long long t0 = gtimer();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    for (int e = threadIdx.x; e < JS * JS; e += JT) {
      const int a = e >> 5, b = e & 31;
      S[a * LDS_ + b] = (a == b) ? 32.0 + a : 1.0 / (1.0 + a + b);
      R[a * LDS_ + b] = a == b ? 1.0 : 0.0;
    }
    __syncthreads();
    acc += subsolve(S, R, tb, pbuf, r0, 1e-14, 0.0, false);
  }
  const unsigned long long t1 = gtimer();
  if (threadIdx.x == 0) {
    out[0] = (double)(t1 - t0) / (iters * (r0 ? 31.0 : 16.0));
    out[1] = acc;
  }
}
}  // namespace
}  // namespace fpi

extern "C" int fpi_dbg_subsolve_bench(fpi_handle h, int iters, double* h_ns_per_step) {
  FPI_API_BEGIN(h)
  double* d;
  FPI_CUDA(cudaMallocAsync((void**)&d, 16, h->stream));
  fpi::k_subsolve_bench<<<1, fpi::JT, 0, h->stream>>>(iters, d);
  FPI_LAUNCH_CHECK();
  double hv[2];
  FPI_CUDA(cudaMemcpyAsync(hv, d, 16, cudaMemcpyDeviceToHost, h->stream));
  FPI_CUDA(cudaStreamSynchronize(h->stream));
  cudaFreeAsync(d, h->stream);
  *h_ns_per_step = hv[0];
  FPI_API_END(h)
}
