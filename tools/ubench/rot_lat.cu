// Pure dependent-chain latency of jacobi.cu's rotation() (one warp, no other warps).
#include "../../paper_2011_04235_b200/csrc/jacobi.cu"
namespace fpi { namespace {
__global__ void k_rot(int iters, long long* cyc, double* sink, int nwarps_busy) {
  double app = 2.0 + threadIdx.x * 1e-3, aqq = 1.0, apq = 0.3;
  double acc = 0.0;
  const bool timed = threadIdx.x < 32;
  if (!timed && (int)(threadIdx.x >> 5) > nwarps_busy) return;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double c, s;
    rotation(app, aqq, apq, 1e-14, 0.0, false, c, s);
    const double dx = new_diag(true, c, s, app, aqq, apq);
    const double dy = new_diag(false, c, s, app, aqq, apq);
    acc += c;
    app = dy + 1.0; aqq = dx; apq = 0.3 * c + 0.1 * s;  // keep it a dependent chain
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  sink[threadIdx.x] = acc + app;
}
}}
int main() {
  long long* c; double* s;
  cudaMalloc(&c, 8); cudaMalloc(&s, 256 * 8);
  for (int busy : {0, 7}) {
    fpi::k_rot<<<1, 256>>>(1000, c, s, busy);
    fpi::k_rot<<<1, 256>>>(1000, c, s, busy);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("busy warps %d: rotation+new_diag+glue %.0f cycles per iteration\n", busy, h / 1000.0);
  }
}
