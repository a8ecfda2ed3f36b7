// DMMA m8n8k4 dependent-chain latency and independent-chain issue rate (one warp / 8 warps).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double d[CH][2];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
  long long h;
#define RUN(CH, TH) k<CH><<<1, TH>>>(o, c, 1.0, 1e-3); k<CH><<<1, TH>>>(o, c, 1.0, 1e-3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); \
  printf("chains=%d threads=%d: %.1f cyc per DMMA-step (per warp)\n", CH, TH, h / 256.0);
  RUN(1, 32) RUN(2, 32) RUN(4, 32) RUN(8, 32) RUN(1, 256) RUN(2, 256) RUN(4, 256) RUN(8, 256)
  return 0;
}
