// fpi_fastpi: Algorithm 1 end to end behind one C call (reference pinv.py:278-347, fastpi()), for a
// C / C++ / FFI host that does not want to sequence the stage entry points itself.  The stages are
// exactly the ones the Python mirror (paper_2011_04235_b200/pinv.py fastpi_device) calls, in the
// same order and with the same rank logic, so the two produce identical bits.
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "capi_guard.cuh"

namespace fpi {
namespace {

// Device buffer owned by the handle's fastpi result until fpi_fastpi_release / fpi_fastpi_take.
// Stream-ordered (cudaMallocAsync from the device pool, whose release threshold fpi_create raises):
// a cudaMalloc / cudaFree pair would synchronise the device at every solve.
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  void alloc(size_t bytes, cudaStream_t st) {
    release();
    s = st;
    if (bytes) FPI_CUDA(cudaMallocAsync(&p, bytes, st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
  }
  void* take() {
    void* q = p;
    p = nullptr;
    return q;
  }
  ~DevBuf() { release(); }
};

// Stage boundaries of one solve as events on the handle stream (pinv.py:95-98 StageTime).
constexpr int kStages = 5;  // reorder, block_svd, row_update, column_update, pinv_assembly

// Checks a status returned by one of the library's own entry points and rethrows it with its message.
void ok(fpi_context* h, int rc) {
  if (rc != FPI_OK) throw Error(rc, h->last_error);
}

}  // namespace

struct FastpiResult {
  DevBuf U, sigma, Vt, sdag, row_fwd, col_fwd, spans;
  std::vector<int64_t> gcc;
  cudaEvent_t ev[kStages + 1] = {};
  fpi_fastpi_info info{};
  FastpiResult() {
    for (auto& e : ev) FPI_CUDA(cudaEventCreate(&e));
  }
  ~FastpiResult() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  void mark(int i, cudaStream_t s) { FPI_CUDA(cudaEventRecord(ev[i], s)); }
};

void fastpi_free(fpi_context* h) {
  delete h->fastpi;
  h->fastpi = nullptr;
}

}  // namespace fpi

namespace fpi {
namespace {
// the two halves of the canonical-form check (sparse.cu k_check_canonical) for a deferred upload
__global__ void k_check_pattern(int64_t m, const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                                int* __restrict__ bad) {
  FPI_GRID_STRIDE(r, m) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    for (int64_t p = b + 1; p < e; ++p)
      if (idx[p] <= idx[p - 1]) {
        *bad = 1;
        break;
      }
  }
}
__global__ void k_check_values(int64_t nnz, const double* __restrict__ val, int* __restrict__ bad) {
  bool z = false;
  FPI_GRID_STRIDE(i, nnz) z |= val[i] == 0.0;
  if (z) *bad = 1;
}
}  // namespace
}  // namespace fpi

extern "C" int fpi_fastpi_values_hook(fpi_handle h, fpi_values_hook hook, void* ctx) {
  FPI_API_BEGIN(h)
  h->values_hook = hook;
  h->values_hook_ctx = ctx;
  FPI_API_END(h)
}

extern "C" int fpi_fastpi_ex(fpi_handle h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                             const int32_t* d_indices, const double* d_values, double alpha, double k, int64_t seed,
                             double low_rank_threshold, double pinv_cutoff, int32_t flags, fpi_fastpi_info* h_info) {
  FPI_API_BEGIN(h)
  using fpi::Scratch;
  FPI_REQUIRE(m > 0 && n > 0, FPI_EDOMAIN, "cannot factorize a zero-dimension matrix");
  FPI_REQUIRE(m >= n, FPI_EDOMAIN, "fpi_fastpi expects m >= n (factor A^T and swap the factors otherwise)");
  FPI_REQUIRE(alpha > 0.0 && alpha <= 1.0, FPI_EDOMAIN, "target rank ratio alpha must be in (0, 1]");
  cudaStream_t s = h->stream;
  const fpi_values_hook values_hook = h->values_hook;
  void* const values_ctx = h->values_hook_ctx;
  h->values_hook = nullptr;
  h->values_hook_ctx = nullptr;
  const bool deferred = (flags & FPI_FASTPI_DEFERRED_VALUES) != 0;
  FPI_REQUIRE(!deferred || ((flags & FPI_FASTPI_CANONICAL) != 0 && values_hook != nullptr), FPI_EDOMAIN,
              "FPI_FASTPI_DEFERRED_VALUES needs FPI_FASTPI_CANONICAL and a hook (fpi_fastpi_values_hook)");
  delete h->fastpi;
  h->fastpi = nullptr;
  if (deferred) {  // pattern half of check_csr before anything is speculated on it
    Scratch<int> bad(1, s);
    FPI_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    fpi::k_check_pattern<<<fpi::grid_for(m, 256, (int64_t)h->num_sms * 16), 256, 0, s>>>(m, d_indptr, d_indices, bad);
    FPI_LAUNCH_CHECK();
    fpi::note_launch(h);
    if (fpi::host_read(bad.get(), s)) throw fpi::Error(FPI_ERETRY, "deferred upload: the CSR pattern is not canonical");
  }
  auto* res = new fpi::FastpiResult();
  h->fastpi = res;
  fpi_fastpi_info& info = res->info;
  info.m = m;
  info.n = n;
  res->mark(0, s);

  // check_csr (validation.py:38-55): canonical copy (sorted, duplicates summed, explicit zeros dropped),
  // skipped when the caller says its CSR is canonical already (DeviceCSR.from_host canonicalizes)
  const bool canonical = (flags & FPI_FASTPI_CANONICAL) != 0;
  Scratch<int64_t> ap(canonical ? 0 : m + 1, s);
  Scratch<int32_t> ai(canonical ? 0 : nnz, s);
  Scratch<double> av(canonical ? 0 : nnz, s);
  int64_t cnnz = nnz;
  const int64_t* cp = d_indptr;
  const int32_t* ci = d_indices;
  const double* cv = d_values;
  if (!canonical) {
    fpi::ok(h, fpi_csr_canonicalize(h, m, n, nnz, d_indptr, d_indices, d_values, ap, ai, av, &cnnz));
    cp = ap;
    ci = ai;
    cv = av;
  }

  // reorder + partition (reorder.py:158-337)
  res->row_fwd.alloc(sizeof(int64_t) * m, s);
  res->col_fwd.alloc(sizeof(int64_t) * n, s);
  int64_t* row_fwd = static_cast<int64_t*>(res->row_fwd.p);
  int64_t* col_fwd = static_cast<int64_t*>(res->col_fwd.p);
  fpi_reorder_info ri{};
  fpi::ok(h, fpi_reorder(h, m, n, cnnz, cp, ci, k, row_fwd, col_fwd, &ri));
  res->spans.alloc(sizeof(int64_t) * (4 * ri.n_spans + 4), s);
  int64_t* spans = static_cast<int64_t*>(res->spans.p);
  res->gcc.assign((size_t)ri.n_gcc + 1, 0);
  fpi::ok(h, fpi_reorder_fetch(h, spans, res->gcc.data()));
  res->gcc.resize((size_t)ri.n_gcc);
  info.n_gcc = ri.n_gcc;
  info.edges_visited = ri.edges_visited;
  info.nodes_visited = ri.nodes_visited;
  const int64_t m1 = ri.m1, n1 = ri.n1, m2 = ri.m2, n2 = ri.n2;
  info.m1 = m1;
  info.n1 = n1;
  info.m2 = m2;
  info.n2 = n2;
  info.n_iterations = ri.n_iterations;
  info.n_spans = ri.n_spans;
  fpi_partition_info pi{};
  fpi::ok(h, fpi_partition_count(h, m, n, cnnz, cp, ci, row_fwd, col_fwd, m1, n1, ri.n_spans, spans, &pi));
  const int64_t nT = pi.nnz_a12 + pi.nnz_a22;
  if (deferred) {
    // the values were uploading on the caller's stream while the reorder ran: wait for them, then the
    // value half of check_csr (no explicit zeros)
    void* ev = nullptr;
    if (values_hook(values_ctx, &ev) != 0 || ev == nullptr) {
      fpi::fastpi_free(h);
      throw fpi::Error(FPI_ECUDA, "deferred upload: the values hook failed");
    }
    FPI_CUDA(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev), 0));
    Scratch<int> bad(1, s);
    FPI_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    fpi::k_check_values<<<fpi::grid_for(cnnz, 256, (int64_t)h->num_sms * 16), 256, 0, s>>>(cnnz, cv, bad);
    FPI_LAUNCH_CHECK();
    fpi::note_launch(h);
    if (fpi::host_read(bad.get(), s)) {
      fpi::fastpi_free(h);
      throw fpi::Error(FPI_ERETRY, "deferred upload: the CSR holds explicit zeros");
    }
  }
  Scratch<int64_t> a11p(m1 + 1, s), tp(m + 1, s), ttp(n2 + 1, s), a21p(m2 + 1, s), a21tp(n1 + 1, s);
  Scratch<int32_t> a11i(pi.nnz_a11, s), ti(nT, s), tti(nT, s), a21i(pi.nnz_a21, s), a21ti(pi.nnz_a21, s);
  Scratch<double> a11v(pi.nnz_a11, s), tv(nT, s), ttv(nT, s), a21v(pi.nnz_a21, s), a21tv(pi.nnz_a21, s);
  fpi::ok(h, fpi_partition(h, m, n, cnnz, cp, ci, cv, row_fwd, col_fwd, m1, n1, ri.n_spans, spans, a11p, a11i, a11v,
                           tp, ti, tv, ttp, tti, ttv, a21p, a21i, a21v, a21tp, a21ti, a21tv));
  res->mark(1, s);

  // block-diagonal SVD of A11 (svd.py:141-193)
  fpi_block_plan bp{};
  fpi::ok(h, fpi_block_svd_plan(h, ri.n_spans, spans, alpha, &bp));
  const int64_t rank11 = bp.rank11;
  Scratch<double> sig11(rank11, s), u11v(bp.nnz_u11, s), v11v(bp.nnz_vt11, s);
  Scratch<int64_t> u11p(m1 + 1, s), v11p(rank11 + 1, s);
  Scratch<int32_t> u11i(bp.nnz_u11, s), v11i(bp.nnz_vt11, s);
  fpi::ok(h, fpi_block_svd(h, m1, n1, a11p, a11i, a11v, ri.n_spans, spans, alpha, sig11, u11p, u11i, u11v, v11p,
                           v11i, v11v, &bp));
  info.rank11 = rank11;
  res->mark(2, s);

  // row update (pinv.py:318-331): s = min(ceil(alpha n1), rank11 + m2, n1), seed + 1
  const int64_t want_s = (int64_t)std::ceil(alpha * (double)n1);
  int64_t srank = want_s;
  if (rank11 + m2 < srank) srank = rank11 + m2;
  if (n1 < srank) srank = n1;
  info.rank_clamped = srank < want_s ? 1 : 0;
  info.s = srank;
  Scratch<double> Ur(m * srank, s), sigr(srank, s), Vtr(srank * n1, s);
  int32_t eng_r = 0;
  if (srank > 0)
    fpi::ok(h, fpi_row_update(h, m1, n1, rank11, sig11, u11p, u11i, u11v, v11p, v11i, v11v, m2, a21p, a21i, a21v,
                              srank, low_rank_threshold, seed + 1, Ur, sigr, Vtr, &eng_r));
  info.row_engine = eng_r;
  res->mark(3, s);

  // column update (pinv.py:333-339): r = min(ceil(alpha n), s + n2, m), seed + 2
  int64_t r = (int64_t)std::ceil(alpha * (double)n);
  if (srank + n2 < r) r = srank + n2;
  if (m < r) r = m;
  info.rank = r;
  res->U.alloc(sizeof(double) * m * r, s);
  res->sigma.alloc(sizeof(double) * r, s);
  res->Vt.alloc(sizeof(double) * r * n, s);
  res->sdag.alloc(sizeof(double) * r, s);
  int32_t eng_c = 0;
  if (r > 0)
    fpi::ok(h, fpi_column_update(h, m, srank, n1, Ur, sigr, Vtr, n2, tp, ti, tv, ttp, tti, ttv, r, low_rank_threshold,
                                 seed + 2, static_cast<double*>(res->U.p), static_cast<double*>(res->sigma.p),
                                 static_cast<double*>(res->Vt.p), &eng_c));
  info.col_engine = eng_c;
  res->mark(4, s);

  // pseudoinverse assembly (pinv.py:211-231)
  double tol = 0.0;
  int32_t af = 0;
  if (r > 0)
    fpi::ok(h, fpi_pinv_assemble(h, r, static_cast<double*>(res->sigma.p), m, n, pinv_cutoff,
                                 static_cast<double*>(res->sdag.p), &tol, &af));
  info.tolerance_used = tol;
  info.all_filtered = af;  // pinv.py:222-224: False for an empty sigma
  res->mark(5, s);
  // no stream synchronisation: the scratch above is freed stream-ordered (cudaFreeAsync) after its
  // last use, and the factors are read by later work on the same stream
  if (h_info) *h_info = info;
  FPI_API_END(h)
}

extern "C" int fpi_fastpi(fpi_handle h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                          const int32_t* d_indices, const double* d_values, double alpha, double k, int64_t seed,
                          double low_rank_threshold, double pinv_cutoff, fpi_fastpi_info* h_info) {
  return fpi_fastpi_ex(h, m, n, nnz, d_indptr, d_indices, d_values, alpha, k, seed, low_rank_threshold, pinv_cutoff,
                       0, h_info);
}

extern "C" int fpi_fastpi_get(fpi_handle h, const double** d_U, const double** d_sigma, const double** d_Vt,
                              const double** d_sigma_dagger, const int64_t** d_row_fwd, const int64_t** d_col_fwd) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(h->fastpi != nullptr, FPI_EDOMAIN, "no fpi_fastpi result on this handle");
  fpi::FastpiResult* r = h->fastpi;
  if (d_U) *d_U = static_cast<const double*>(r->U.p);
  if (d_sigma) *d_sigma = static_cast<const double*>(r->sigma.p);
  if (d_Vt) *d_Vt = static_cast<const double*>(r->Vt.p);
  if (d_sigma_dagger) *d_sigma_dagger = static_cast<const double*>(r->sdag.p);
  if (d_row_fwd) *d_row_fwd = static_cast<const int64_t*>(r->row_fwd.p);
  if (d_col_fwd) *d_col_fwd = static_cast<const int64_t*>(r->col_fwd.p);
  FPI_API_END(h)
}

extern "C" int fpi_fastpi_take(fpi_handle h, fpi_fastpi_buffers* out, int64_t* h_gcc, int64_t gcc_cap,
                               float* h_stage_ms) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(h->fastpi != nullptr, FPI_EDOMAIN, "no fpi_fastpi result on this handle");
  FPI_REQUIRE(out != nullptr, FPI_EDOMAIN, "fpi_fastpi_take needs an output descriptor");
  fpi::FastpiResult* r = h->fastpi;
  FPI_REQUIRE(h_gcc == nullptr || gcc_cap >= (int64_t)r->gcc.size(), FPI_EDOMAIN, "gcc buffer too small");
  if (h_gcc)
    for (size_t i = 0; i < r->gcc.size(); ++i) h_gcc[i] = r->gcc[i];
  if (h_stage_ms) {
    FPI_CUDA(cudaEventSynchronize(r->ev[fpi::kStages]));
    for (int i = 0; i < fpi::kStages; ++i) FPI_CUDA(cudaEventElapsedTime(&h_stage_ms[i], r->ev[i], r->ev[i + 1]));
  }
  out->U = static_cast<double*>(r->U.take());
  out->sigma = static_cast<double*>(r->sigma.take());
  out->Vt = static_cast<double*>(r->Vt.take());
  out->sigma_dagger = static_cast<double*>(r->sdag.take());
  out->row_fwd = static_cast<int64_t*>(r->row_fwd.take());
  out->col_fwd = static_cast<int64_t*>(r->col_fwd.take());
  out->spans = static_cast<int64_t*>(r->spans.take());
  delete r;  // events only: the buffers now belong to the caller
  h->fastpi = nullptr;
  FPI_API_END(h)
}

extern "C" int fpi_device_free(fpi_handle h, void* d_ptr) {
  FPI_API_BEGIN(h)
  if (d_ptr) FPI_CUDA(cudaFreeAsync(d_ptr, h->stream));
  FPI_API_END(h)
}

extern "C" int fpi_fastpi_release(fpi_handle h) {
  FPI_API_BEGIN(h)
  FPI_CUDA(cudaStreamSynchronize(h->stream));
  delete h->fastpi;
  h->fastpi = nullptr;
  FPI_API_END(h)
}
