// Per-kernel-class timing with CUDA events (bench.py's roofline leg) and the
// FP64 tensor-pipe peak microbenchmark (DMMA issue rate from registers).
#include <map>

#include "common.cuh"
#include "capi_guard.cuh"
#include "instrument.cuh"

#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace fpi {
void trace_point(fpi_context* h, const char* label) {
  static const bool on = getenv("FPI_TRACE") != nullptr;
  static const bool host = getenv("FPI_TRACE_HOST") != nullptr;
  if (host) {  // host wall time between points, no synchronisation: where does the host block?
    static auto lasth = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(now - lasth).count();
    if (ms > 5.0) fprintf(stderr, "[trace-host] %-28s %9.3f ms\n", label, ms);
    lasth = now;
    return;
  }
  if (!on) return;
  static auto last = std::chrono::steady_clock::now();
  cudaStreamSynchronize(h->stream);
  const auto now = std::chrono::steady_clock::now();
  fprintf(stderr, "[trace] %-28s %9.3f ms\n", label, std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}


struct TimingState {
  struct Rec {
    cudaEvent_t a, b;
    std::string name;
    double flops, bytes;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  struct Stat {
    int64_t launches = 0;
    double ms = 0, flops = 0, bytes = 0;
  };
  std::map<std::string, Stat> stats;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    FPI_CUDA(cudaEventCreate(&e));
    return e;
  }
};

static std::map<fpi_context*, TimingState*> g_timing;

static TimingState* state(fpi_context* h) {
  auto it = g_timing.find(h);
  return it == g_timing.end() ? nullptr : it->second;
}

KTimer::KTimer(fpi_context* h_, const char* name_, double flops_, double bytes_)
    : h(h_), name(name_), flops(flops_), bytes(bytes_) {
  TimingState* st = state(h);
  if (!st) return;
  active = true;
  ev_a = st->get();
  FPI_CUDA(cudaEventRecord((cudaEvent_t)ev_a, h->stream));
}

KTimer::~KTimer() {
  if (!active) return;
  TimingState* st = state(h);
  if (!st) return;
  cudaEvent_t b = st->get();
  cudaEventRecord(b, h->stream);
  st->pending.push_back({(cudaEvent_t)ev_a, b, name, flops, bytes});
}

namespace {
__global__ void k_dmma_peak(int iters, double* out) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[0] = s;
}
}  // namespace

}  // namespace fpi

extern "C" int fpi_timing_enable(fpi_handle h, int on) {
  FPI_API_BEGIN(h)
  if (on) {
    if (!fpi::state(h)) fpi::g_timing[h] = new fpi::TimingState();
    h->timing_on = true;
  } else {
    h->timing_on = false;
    auto it = fpi::g_timing.find(h);
    if (it != fpi::g_timing.end()) {
      for (auto& r : it->second->pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
      }
      for (auto e : it->second->pool) cudaEventDestroy(e);
      delete it->second;
      fpi::g_timing.erase(it);
    }
  }
  FPI_API_END(h)
}

// Resolves pending events; writes up to cap records "name\tlaunches\tms\tflops\tbytes\n" into buf.
extern "C" int fpi_timing_report(fpi_handle h, char* buf, int64_t cap, int reset) {
  FPI_API_BEGIN(h)
  fpi::TimingState* st = fpi::state(h);
  FPI_REQUIRE(st, FPI_EDOMAIN, "timing not enabled");
  FPI_CUDA(cudaStreamSynchronize(h->stream));
  for (auto& r : st->pending) {
    float ms = 0;
    FPI_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    auto& s = st->stats[r.name];
    s.launches += 1;
    s.ms += ms;
    s.flops += r.flops;
    s.bytes += r.bytes;
    st->pool.push_back(r.a);
    st->pool.push_back(r.b);
  }
  st->pending.clear();
  std::string out;
  for (auto& kv : st->stats) {
    char line[256];
    snprintf(line, sizeof(line), "%s\t%lld\t%.6f\t%.6e\t%.6e\n", kv.first.c_str(), (long long)kv.second.launches,
             kv.second.ms, kv.second.flops, kv.second.bytes);
    out += line;
  }
  if (buf && cap > 0) {
    size_t n = out.size() < (size_t)(cap - 1) ? out.size() : (size_t)(cap - 1);
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  if (reset) st->stats.clear();
  FPI_API_END(h)
}

// FP64 tensor (DMMA) issue-rate peak in TFLOP/s over `ms_target` milliseconds of work.
extern "C" int fpi_dmma_peak(fpi_handle h, double* h_tflops) {
  FPI_API_BEGIN(h)
  cudaStream_t s = h->stream;
  double* out;
  FPI_CUDA(cudaMallocAsync((void**)&out, 8, s));
  const int blocks = h->num_sms * 4, threads = 256, iters = 4096;
  fpi::k_dmma_peak<<<blocks, threads, 0, s>>>(16, out);  // warm-up
  cudaEvent_t a, b;
  FPI_CUDA(cudaEventCreate(&a));
  FPI_CUDA(cudaEventCreate(&b));
  FPI_CUDA(cudaEventRecord(a, s));
  fpi::k_dmma_peak<<<blocks, threads, 0, s>>>(iters, out);
  FPI_CUDA(cudaEventRecord(b, s));
  FPI_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  FPI_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFreeAsync(out, s);
  const double flops = (double)blocks * (threads / 32) * iters * 8 * (2.0 * 8 * 8 * 4);
  *h_tflops = flops / (ms * 1e-3) / 1e12;
  FPI_API_END(h)
}
