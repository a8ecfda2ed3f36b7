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

// Device buffer owned by the handle's fastpi result (cudaMalloc: it outlives the call).
struct DevBuf {
  void* p = nullptr;
  void alloc(size_t bytes) {
    release();
    if (bytes) FPI_CUDA(cudaMalloc(&p, bytes));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
  }
  ~DevBuf() { release(); }
};

// Checks a status returned by one of the library's own entry points and rethrows it with its message.
void ok(fpi_context* h, int rc) {
  if (rc != FPI_OK) throw Error(rc, h->last_error);
}

}  // namespace

struct FastpiResult {
  DevBuf U, sigma, Vt, sdag, row_fwd, col_fwd;
  fpi_fastpi_info info{};
};

void fastpi_free(fpi_context* h) {
  delete h->fastpi;
  h->fastpi = nullptr;
}

}  // namespace fpi

extern "C" int fpi_fastpi(fpi_handle h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                          const int32_t* d_indices, const double* d_values, double alpha, double k, int64_t seed,
                          double low_rank_threshold, double pinv_cutoff, fpi_fastpi_info* h_info) {
  FPI_API_BEGIN(h)
  using fpi::Scratch;
  FPI_REQUIRE(m > 0 && n > 0, FPI_EDOMAIN, "cannot factorize a zero-dimension matrix");
  FPI_REQUIRE(m >= n, FPI_EDOMAIN, "fpi_fastpi expects m >= n (factor A^T and swap the factors otherwise)");
  FPI_REQUIRE(alpha > 0.0 && alpha <= 1.0, FPI_EDOMAIN, "target rank ratio alpha must be in (0, 1]");
  cudaStream_t s = h->stream;
  delete h->fastpi;
  h->fastpi = nullptr;
  auto* res = new fpi::FastpiResult();
  h->fastpi = res;
  fpi_fastpi_info& info = res->info;
  info.m = m;
  info.n = n;

  // check_csr (validation.py:38-55): canonical copy (sorted, duplicates summed, explicit zeros dropped)
  Scratch<int64_t> ap(m + 1, s);
  Scratch<int32_t> ai(nnz, s);
  Scratch<double> av(nnz, s);
  int64_t cnnz = 0;
  fpi::ok(h, fpi_csr_canonicalize(h, m, n, nnz, d_indptr, d_indices, d_values, ap, ai, av, &cnnz));

  // reorder + partition (reorder.py:158-337)
  res->row_fwd.alloc(sizeof(int64_t) * m);
  res->col_fwd.alloc(sizeof(int64_t) * n);
  int64_t* row_fwd = static_cast<int64_t*>(res->row_fwd.p);
  int64_t* col_fwd = static_cast<int64_t*>(res->col_fwd.p);
  fpi_reorder_info ri{};
  fpi::ok(h, fpi_reorder(h, m, n, cnnz, ap, ai, k, row_fwd, col_fwd, &ri));
  Scratch<int64_t> spans(4 * ri.n_spans + 4, s);
  std::vector<int64_t> gcc((size_t)ri.n_gcc + 1);
  fpi::ok(h, fpi_reorder_fetch(h, spans, gcc.data()));
  const int64_t m1 = ri.m1, n1 = ri.n1, m2 = ri.m2, n2 = ri.n2;
  info.m1 = m1;
  info.n1 = n1;
  info.m2 = m2;
  info.n2 = n2;
  info.n_iterations = ri.n_iterations;
  info.n_spans = ri.n_spans;
  fpi_partition_info pi{};
  fpi::ok(h, fpi_partition_count(h, m, n, cnnz, ap, ai, row_fwd, col_fwd, m1, n1, ri.n_spans, spans, &pi));
  const int64_t nT = pi.nnz_a12 + pi.nnz_a22;
  Scratch<int64_t> a11p(m1 + 1, s), tp(m + 1, s), ttp(n2 + 1, s), a21p(m2 + 1, s), a21tp(n1 + 1, s);
  Scratch<int32_t> a11i(pi.nnz_a11, s), ti(nT, s), tti(nT, s), a21i(pi.nnz_a21, s), a21ti(pi.nnz_a21, s);
  Scratch<double> a11v(pi.nnz_a11, s), tv(nT, s), ttv(nT, s), a21v(pi.nnz_a21, s), a21tv(pi.nnz_a21, s);
  fpi::ok(h, fpi_partition(h, m, n, cnnz, ap, ai, av, row_fwd, col_fwd, m1, n1, ri.n_spans, spans, a11p, a11i, a11v,
                           tp, ti, tv, ttp, tti, ttv, a21p, a21i, a21v, a21tp, a21ti, a21tv));

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

  // column update (pinv.py:333-339): r = min(ceil(alpha n), s + n2, m), seed + 2
  int64_t r = (int64_t)std::ceil(alpha * (double)n);
  if (srank + n2 < r) r = srank + n2;
  if (m < r) r = m;
  info.rank = r;
  res->U.alloc(sizeof(double) * m * r);
  res->sigma.alloc(sizeof(double) * r);
  res->Vt.alloc(sizeof(double) * r * n);
  res->sdag.alloc(sizeof(double) * r);
  int32_t eng_c = 0;
  if (r > 0)
    fpi::ok(h, fpi_column_update(h, m, srank, n1, Ur, sigr, Vtr, n2, tp, ti, tv, ttp, tti, ttv, r, low_rank_threshold,
                                 seed + 2, static_cast<double*>(res->U.p), static_cast<double*>(res->sigma.p),
                                 static_cast<double*>(res->Vt.p), &eng_c));
  info.col_engine = eng_c;

  // pseudoinverse assembly (pinv.py:211-231)
  double tol = 0.0;
  int32_t af = 0;
  if (r > 0)
    fpi::ok(h, fpi_pinv_assemble(h, r, static_cast<double*>(res->sigma.p), m, n, pinv_cutoff,
                                 static_cast<double*>(res->sdag.p), &tol, &af));
  info.tolerance_used = tol;
  info.all_filtered = af;  // pinv.py:222-224: False for an empty sigma
  FPI_CUDA(cudaStreamSynchronize(s));  // the scratch above is released at scope exit, after its last use
  if (h_info) *h_info = info;
  FPI_API_END(h)
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

extern "C" int fpi_fastpi_release(fpi_handle h) {
  FPI_API_BEGIN(h)
  FPI_CUDA(cudaStreamSynchronize(h->stream));
  delete h->fastpi;
  h->fastpi = nullptr;
  FPI_API_END(h)
}
