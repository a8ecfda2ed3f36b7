// Relative error of the f64 MUFU approximations (rsqrt.approx.f64, rcp.approx.ftz.f64) on [1, 4).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(double* out) {
  double worst_rs = 0, worst_rc = 0;
  for (int i = threadIdx.x; i < 1 << 20; i += blockDim.x) {
    const double x = 1.0 + 3.0 * (double)i / (1 << 20);
    double rs, rc;
    asm("rsqrt.approx.f64 %0, %1;" : "=d"(rs) : "d"(x));
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(x));
    worst_rs = fmax(worst_rs, fabs(rs * sqrt(x) - 1.0));
    worst_rc = fmax(worst_rc, fabs(rc * x - 1.0));
  }
  __shared__ double a[256], b[256];
  a[threadIdx.x] = worst_rs; b[threadIdx.x] = worst_rc;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 256; ++i) { worst_rs = fmax(worst_rs, a[i]); worst_rc = fmax(worst_rc, b[i]); }
    out[0] = worst_rs; out[1] = worst_rc;
  }
}
int main() {
  double* d; cudaMalloc(&d, 16);
  k<<<1, 256>>>(d);
  double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("rsqrt.approx.f64 max rel err %.3e (2^%.1f)\nrcp.approx.ftz.f64 max rel err %.3e (2^%.1f)\n", h[0], log2(h[0]), h[1], log2(h[1]));
}
