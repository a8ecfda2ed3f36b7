// Shared plumbing for the FastPI B200 core: status codes, the handle, a
// stream-ordered scratch allocator and small device helpers.
#pragma once
#include <atomic>
#include <cstring>
#include <mutex>

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>
#include <stdexcept>

#include "../../include/fastpi_b200.h"

namespace fpi {

// Thrown inside the library, converted to a status code at the C-ABI edge.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

#define FPI_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess)                                                          \
      throw ::fpi::Error(FPI_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e) + \
                                        " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define FPI_REQUIRE(cond, code, msg)                 \
  do {                                               \
    if (!(cond)) throw ::fpi::Error((code), (msg));  \
  } while (0)

#define FPI_LAUNCH_CHECK() FPI_CUDA(cudaGetLastError())

// One-time initialisation per CUDA device (kernel attributes such as the dynamic shared-memory
// opt-in are per device, and the handles are per device): runs f() the first time a call site is
// reached with `dev` current, under a lock, then marks the device done in `mask`.
template <class F>
inline void once_per_device(std::atomic<uint64_t>& mask, int dev, F&& f) {
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (mask.load(std::memory_order_relaxed) & bit) return;
  f();
  mask.fetch_or(bit, std::memory_order_release);
}

}  // namespace fpi

namespace fpi {
struct FastpiResult;  // fastpi_capi.cu
struct Comm;          // comm.cuh
void fastpi_free(fpi_context* h);
void comm_free(fpi_context* h);
}  // namespace fpi

// The handle: one stream, device properties, scratch memory and the results
// that are fetched in a second call (variable-size outputs).
struct fpi_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  std::string last_error;
  // reorder results kept until fpi_reorder_fetch
  std::vector<int64_t> gcc_sizes;
  int64_t* d_spans = nullptr;
  int64_t n_spans = 0;
  int64_t spans_cap = 0;
  void* host_scalars = nullptr;  // pinned scratch for per-iteration device scalars (reorder)
  cudaStream_t copy_stream = nullptr;  // device->host copies overlapped with the compute stream
  fpi::FastpiResult* fastpi = nullptr;  // factors of the last fpi_fastpi call (fpi_fastpi_get)
  cudaEvent_t copy_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // numerics diagnostics of the last randomized / dense SVD
  fpi_svd_diag diag{};
  int64_t sparse_core[4] = {0, 0, 0, 0};  // last column update's dense core (fpi_sparse_core_info)
  // fpi_fastpi_values_hook: the caller's "values are on their way" callback of a deferred upload
  int (*values_hook)(void*, void**) = nullptr;
  void* values_hook_ctx = nullptr;
  // cross-rank communicator of a sharded solve (comm.cu), null for one rank
  fpi::Comm* comm = nullptr;
  // counters
  int64_t kernel_launches = 0;
  bool timing_on = false;
};

namespace fpi {

// Stream-ordered scratch buffer (cudaMallocAsync from the device pool).
template <typename T>
struct Scratch {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  Scratch() = default;
  Scratch(size_t count, cudaStream_t st) { alloc(count, st); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) FPI_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T) + 16, st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~Scratch() { release(); }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  Scratch(Scratch&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  Scratch& operator=(Scratch&& o) noexcept {
    release();
    p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0;
    return *this;
  }
  T* get() const { return p; }
  operator T*() const { return p; }
};

inline unsigned grid_for(int64_t n, int threads, int64_t cap = 148 * 32) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

template <typename T>
inline T host_read(const T* d, cudaStream_t s) {
  // through a pinned per-thread slot: a pageable destination makes the driver stage the copy
  static thread_local void* slot = nullptr;
  if (!slot) FPI_CUDA(cudaMallocHost(&slot, 256));
  static_assert(sizeof(T) <= 256, "host_read of a large object");
  FPI_CUDA(cudaMemcpyAsync(slot, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  T v;
  memcpy(&v, slot, sizeof(T));
  return v;
}

// n (<= 256 bytes of) device values to the host through the same pinned slot, one synchronisation
template <typename T>
inline void host_read_n(const T* d, T* out, int n, cudaStream_t s) {
  static thread_local void* slot = nullptr;
  if (!slot) FPI_CUDA(cudaMallocHost(&slot, 256));
  if ((size_t)n * sizeof(T) > 256) throw Error(FPI_ECUDA, "host_read_n: too many values");
  FPI_CUDA(cudaMemcpyAsync(slot, d, sizeof(T) * n, cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  memcpy(out, slot, sizeof(T) * n);
}

void note_launch(fpi_context* h, int count = 1);

}  // namespace fpi

#define FPI_GRID_STRIDE(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)(n); i += (int64_t)gridDim.x * blockDim.x)
