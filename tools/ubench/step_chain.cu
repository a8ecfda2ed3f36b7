// Where the cross-step latency of the Jacobi sub-solve goes: the warp-0 producer chain of
// jacobi.cu's subsolve with clock64 stamps (tool only; includes the library source).
#include "../../paper_2011_04235_b200/csrc/jacobi.cu"

namespace fpi {
namespace {
__global__ void __launch_bounds__(JT) k_chain(int iters, unsigned long long* seg, double* sink) {
  __shared__ __align__(16) double S[JS * LDS_];
  __shared__ __align__(16) double R[JS * LDS_];
  __shared__ PairBuf pb;
  const int tid = threadIdx.x;
  for (int e = tid; e < JS * JS; e += JT) {
    const int a = e >> 5, b = e & 31;
    S[a * LDS_ + b] = (a == b) ? 32.0 + a : 1.0 / (1.0 + a + b);
    R[a * LDS_ + b] = a == b ? 1.0 : 0.0;
  }
  if (tid < 16) {
    for (int b = 0; b < 2; ++b) {
      pb.c[b][tid] = 0.9; pb.s[b][tid] = 0.1; pb.app[b][tid] = 2.0; pb.aqq[b][tid] = 1.0; pb.apq[b][tid] = 0.3;
    }
  }
  __syncthreads();
  const int k = tid & 15, l = (k + 1 + (tid >> 4)) & 15;
  const int u = tid - 32;
  unsigned long long s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    for (int st = 15; st < 31; ++st) {
      const unsigned long long T0 = clock64();
      const int t = st - 15, b = st & 1, nbuf = b ^ 1;
      const int pk = k, qk = 16 + ((k + t) & 15), pl = l, ql = 16 + ((l + t) & 15);
      const double ck = pb.c[b][k], sk = pb.s[b][k], cl = pb.c[b][l], sl = pb.s[b][l];
      const double a = S[pk * LDS_ + pl], bb = S[pk * LDS_ + ql], c2 = S[qk * LDS_ + pl], d = S[qk * LDS_ + ql];
      const double appk = pb.app[b][k], aqqk = pb.aqq[b][k], apqk = pb.apq[b][k];
      const double appl = pb.app[b][l], aqql = pb.aqq[b][l], apql = pb.apq[b][l];
      double rc_[3], rs_[3], rp_[3], rq_[3];
      int rpi[3], rqi[3];
      if (u >= 0) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const int idx = u + r * (JT - 32);
          const int kk = (idx >> 5) & 15, row = idx & 31;
          rpi[r] = kk * LDS_ + row;
          rqi[r] = (16 + ((kk + t) & 15)) * LDS_ + row;
          rc_[r] = pb.c[b][kk];
          rs_[r] = pb.s[b][kk];
          rp_[r] = R[rpi[r]];
          rq_[r] = R[rqi[r]];
        }
      }
      const double ra = ck * a - sk * c2, rb = ck * bb - sk * d;
      const double rc = sk * a + ck * c2, rd = sk * bb + ck * d;
      const double o1 = ra * sl + rb * cl;
      acc += o1;
      const unsigned long long T1 = clock64();
      S[pk * LDS_ + pl] = ra * cl - rb * sl;
      S[pk * LDS_ + ql] = o1;
      S[qk * LDS_ + pl] = rc * cl - rd * sl;
      S[qk * LDS_ + ql] = rc * sl + rd * cl;
      unsigned long long T2 = T1;
      if (tid < 16) {
        const double dx = new_diag(true, ck, sk, appk, aqqk, apqk);
        const double dy = new_diag(false, cl, sl, appl, aqql, apql);
        double c, sn;
        rotation(dx, dy, o1, 1e-14, 0.0, false, c, sn);
        acc += c + sn;
        T2 = clock64();
        // keep the state bounded and non-trivial
        pb.c[nbuf][k] = c; pb.s[nbuf][k] = sn; pb.app[nbuf][k] = dx; pb.aqq[nbuf][k] = dy; pb.apq[nbuf][k] = o1;
      } else if (u >= 0) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          if (u + r * (JT - 32) < 16 * JS) {
            R[rpi[r]] = rc_[r] * rp_[r] - rs_[r] * rq_[r];
            R[rqi[r]] = rs_[r] * rp_[r] + rc_[r] * rq_[r];
          }
        }
      }
      const unsigned long long T3 = clock64();
      __syncthreads();
      const unsigned long long T4 = clock64();
      s0 += T1 - T0; s1 += T2 - T1; s2 += T3 - T2; s3 += T4 - T3;
    }
    if ((it & 7) == 7) {  // re-seed so the rotations stay non-trivial
      for (int e = tid; e < JS * JS; e += JT) {
        const int a2 = e >> 5, b2 = e & 31;
        S[a2 * LDS_ + b2] = (a2 == b2) ? 32.0 + a2 : 1.0 / (1.0 + a2 + b2 + it);
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    seg[0] = s0; seg[1] = s1; seg[2] = s2; seg[3] = s3;
  }
  if (tid == 32) {
    seg[4] = s0; seg[5] = s1; seg[6] = s2; seg[7] = s3;
  }
  sink[tid] = acc;
}
}  // namespace
}  // namespace fpi

int main() {
  unsigned long long* seg;
  double* sink;
  cudaMalloc(&seg, 8 * 8);
  cudaMalloc(&sink, 256 * 8);
  const int iters = 400;
  fpi::k_chain<<<1, fpi::JT>>>(iters, seg, sink);
  fpi::k_chain<<<1, fpi::JT>>>(iters, seg, sink);
  unsigned long long h[8];
  cudaMemcpy(h, seg, sizeof(h), cudaMemcpyDeviceToHost);
  const double steps = iters * 16.0;
  printf("warp0 (producer): loads+o1 %.0f  rotation %.0f  stores %.0f  barrier %.0f  = %.0f cyc/step\n",
         h[0] / steps, h[1] / steps, h[2] / steps, h[3] / steps, (h[0] + h[1] + h[2] + h[3]) / steps);
  printf("warp1 (R updater): loads+o1 %.0f  -- %.0f  R stores %.0f  barrier %.0f\n", h[4] / steps, h[5] / steps,
         h[6] / steps, h[7] / steps);
  return 0;
}
