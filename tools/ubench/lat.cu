// Dependent-chain latency of FP64 / conversion / MUFU ops (cycles per op), one warp.
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void k(double* out, long long* cyc, double x0, float f0) {
  double x = x0; float f = f0;
  long long t0, t1;
  // DFMA
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-9);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DMUL
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = x * 1.0000001;
  t1 = clock64(); cyc[1] = t1 - t0;
  // FFMA
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) f = fmaf(f, 0.999999f, 1e-9f);
  t1 = clock64(); cyc[2] = t1 - t0;
  // F2F f64->f32->f64 roundtrip
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = (double)(float)x + 1e-30;
  t1 = clock64(); cyc[3] = t1 - t0;
  // MUFU.RSQ f32
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) { float r; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f)); f = r; }
  t1 = clock64(); cyc[4] = t1 - t0;
  // MUFU.RCP64H
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  t1 = clock64(); cyc[5] = t1 - t0;
  // LDS->use chain through shared
  __shared__ double sh[64];
  sh[threadIdx.x & 63] = x;
  __syncthreads();
  int idx = threadIdx.x & 63;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) { double v = sh[idx]; idx = ((int)v & 1) + (threadIdx.x & 31); }
  t1 = clock64(); cyc[6] = t1 - t0;
  // bar.sync alone (8 warps)
  t0 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  t1 = clock64(); cyc[7] = t1 - t0;
  // shfl double
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64(); cyc[8] = t1 - t0;
  out[threadIdx.x] = x + f + idx;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 16 * 8);
  k<<<1, 256>>>(o, c, 1.5, 1.5f);
  k<<<1, 256>>>(o, c, 1.5, 1.5f);
  long long h[16]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[] = {"DFMA", "DMUL", "FFMA", "F2F d->f->d (+DADD)", "MUFU.RSQ f32", "MUFU.RCP64H", "LDS dep", "BAR.SYNC(256 thr)", "SHFL f64"};
  for (int i = 0; i < 9; ++i) printf("%-22s %.1f cyc/op\n", nm[i], (double)h[i] / N);
  return 0;
}
