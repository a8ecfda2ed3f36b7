// Sparse structure kernels: check_csr canonicalisation (validation.py:38-55),
// CSR transpose (to_bipartite's A.T, reorder.py:123-134), the permutation
// (apply_permutation, reorder.py:290-307) and the 2x2 partition with its
// structural check (partition, reorder.py:310-337).
//
// Every sorted CSR is produced the same way: (major, minor) coordinates ->
// 64-bit key (major << minor_bits | minor) -> stable radix sort of (key,
// position) -> gather values; row pointers from a per-major histogram and a
// scan.  Keys are unique, so the result is deterministic regardless of the
// order in which entries were appended.
#include "common.cuh"
#include "capi_guard.cuh"
#include "cub_util.cuh"
#include "sparse.cuh"
#include "instrument.cuh"

namespace fpi {
namespace {

__global__ void k_expand_rows(int64_t m, const int64_t* __restrict__ indptr, int32_t* __restrict__ rows) {
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < m; r += nw)
    for (int64_t p = indptr[r] + lane; p < indptr[r + 1]; p += 32) rows[p] = (int32_t)r;
}

__global__ void k_make_keys(int64_t cnt, const int32_t* __restrict__ major, const int32_t* __restrict__ minor,
                            int minor_bits, uint64_t* __restrict__ keys, int32_t* __restrict__ pos) {
  FPI_GRID_STRIDE(i, cnt) {
    keys[i] = ((uint64_t)(uint32_t)major[i] << minor_bits) | (uint32_t)minor[i];
    pos[i] = (int32_t)i;
  }
}

// Row pointers from the sorted keys: ptr[r] = first position whose major is >= r, by a binary search
// per row (no per-entry atomics -- a transpose's popular columns made those serialise).
__global__ void k_ptr_from_sorted(int64_t cnt, const uint64_t* __restrict__ keys, int minor_bits, int64_t nmajor,
                                  int64_t* __restrict__ ptr) {
  FPI_GRID_STRIDE(r, nmajor + 1) {
    const uint64_t target = (uint64_t)r << minor_bits;
    int64_t lo = 0, hi = cnt;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    ptr[r] = lo;
  }
}

__global__ void k_iota_pos(int64_t n, int32_t* __restrict__ pos) {
  FPI_GRID_STRIDE(i, n) pos[i] = (int32_t)i;
}

__global__ void k_gather_transposed(int64_t nnz, const int32_t* __restrict__ pos, const int32_t* __restrict__ rows,
                                    const double* __restrict__ vals, int32_t* __restrict__ t_idx,
                                    double* __restrict__ t_val) {
  FPI_GRID_STRIDE(i, nnz) {
    const int32_t p = pos[i];
    t_idx[i] = rows[p];
    if (t_val) t_val[i] = vals ? vals[p] : 0.0;
  }
}

// t_ptr[c] = first position whose (sorted) column is >= c
__global__ void k_ptr_from_sorted32(int64_t cnt, const uint32_t* __restrict__ keys, int64_t ncols,
                                    int64_t* __restrict__ ptr) {
  FPI_GRID_STRIDE(c, ncols + 1) {
    int64_t lo = 0, hi = cnt;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)keys[mid] < c) lo = mid + 1; else hi = mid;
    }
    ptr[c] = lo;
  }
}

__global__ void k_scatter_sorted(int64_t cnt, const uint64_t* __restrict__ keys, const int32_t* __restrict__ pos,
                                 const double* __restrict__ vals, uint64_t minor_mask, int32_t* __restrict__ out_idx,
                                 double* __restrict__ out_val) {
  FPI_GRID_STRIDE(i, cnt) {
    out_idx[i] = (int32_t)(keys[i] & minor_mask);
    if (out_val) out_val[i] = vals ? vals[pos[i]] : 0.0;
  }
}

__global__ void k_counts_to_ptr_first(int64_t* ptr) { ptr[0] = 0; }

// Canonical-form check: strictly increasing indices within rows, no zero values.
__global__ void k_check_canonical(int64_t m, const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                                  const double* __restrict__ val, int* __restrict__ bad) {
  FPI_GRID_STRIDE(r, m) {
    int64_t b = indptr[r], e = indptr[r + 1];
    for (int64_t p = b; p < e; ++p) {
      if (val[p] == 0.0 || (p > b && idx[p] <= idx[p - 1])) {
        *bad = 1;
        break;
      }
    }
  }
}

__global__ void k_coo_keys(int64_t nnz, const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                           int minor_bits, uint64_t* __restrict__ keys, int32_t* __restrict__ pos) {
  FPI_GRID_STRIDE(i, nnz) {
    keys[i] = ((uint64_t)(uint32_t)rows[i] << minor_bits) | (uint32_t)cols[i];
    pos[i] = (int32_t)i;
  }
}

// After sorting: sum runs of equal keys (in sorted order), keep non-zero sums.
__global__ void k_run_heads(int64_t n, const uint64_t* __restrict__ keys, int32_t* __restrict__ head) {
  FPI_GRID_STRIDE(i, n) head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_sum_runs(int64_t n, const uint64_t* __restrict__ keys, const int32_t* __restrict__ pos,
                           const double* __restrict__ vals, const int32_t* __restrict__ head,
                           double* __restrict__ run_sum, uint64_t* __restrict__ run_key,
                           const int32_t* __restrict__ run_id) {
  FPI_GRID_STRIDE(i, n) {
    if (!head[i]) continue;
    double s = vals[pos[i]];
    for (int64_t j = i + 1; j < n && !head[j]; ++j) s += vals[pos[j]];
    run_sum[run_id[i]] = s;
    run_key[run_id[i]] = keys[i];
  }
}

struct NonZeroAt {
  const double* v;
  __device__ bool operator()(int32_t i) const { return v[i] != 0.0; }
};

__global__ void k_emit_canonical(int64_t cnt, const int32_t* __restrict__ keep, const uint64_t* __restrict__ run_key,
                                 const double* __restrict__ run_sum, int minor_bits, int32_t* __restrict__ out_idx,
                                 double* __restrict__ out_val, int32_t* __restrict__ counts) {
  FPI_GRID_STRIDE(i, cnt) {
    int32_t r = keep[i];
    uint64_t k = run_key[r];
    out_idx[i] = (int32_t)(k & ((1ull << minor_bits) - 1));
    out_val[i] = run_sum[r];
    atomicAdd(counts + (int32_t)(k >> minor_bits), 1);
  }
}

// Partition classification (reordered coordinates).
struct PartBufs {
  int32_t *a11_r, *a11_c;
  double* a11_v;
  int32_t *t_r, *t_c;
  double* t_v;
  int32_t *a21_r, *a21_c;
  double* a21_v;
  unsigned long long* counters;  // [0] a11, [1] t, [2] a21, [3] structural violations, [4] a12
};

// Slots for up to 5 per-thread flags: one global atomic per CTA and counter (a per-warp atomic on
// five shared addresses serialised at L2); slots are unordered, build_csr sorts afterwards.
template <int NC>
__device__ __forceinline__ void block_slots(unsigned long long* ctr, const bool (&want)[NC],
                                            unsigned long long (&slot)[NC]) {
  __shared__ unsigned int wc[NC][32];
  __shared__ unsigned long long bb[NC];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  unsigned masks[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    masks[c] = __ballot_sync(0xffffffffu, want[c]);
    if (lane == 0) wc[c][warp] = __popc(masks[c]);
  }
  __syncthreads();
  if (threadIdx.x < NC) {
    const int c = threadIdx.x;
    unsigned int run = 0;
    for (int w = 0; w < nw; ++w) {
      const unsigned int x = wc[c][w];
      wc[c][w] = run;
      run += x;
    }
    bb[c] = run ? atomicAdd(ctr + c, (unsigned long long)run) : 0ull;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NC; ++c) slot[c] = bb[c] + wc[c][warp] + __popc(masks[c] & lt);
  __syncthreads();
}

__global__ void k_partition(int64_t nnz, const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                            const double* __restrict__ vals, const int64_t* __restrict__ row_fwd,
                            const int64_t* __restrict__ col_fwd, int64_t m1, int64_t n1,
                            const int32_t* __restrict__ row_span, const int64_t* __restrict__ spans, bool emit,
                            PartBufs b) {
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < nnz; base += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = base + threadIdx.x;
    bool valid = e < nnz;
    int64_t r = 0, c = 0;
    if (valid) {
      r = row_fwd[rows[e]];
      c = col_fwd[cols[e]];
    }
    bool in11 = valid && r < m1 && c < n1;
    bool inT = valid && c >= n1;
    bool in21 = valid && r >= m1 && c < n1;
    bool viol = false;
    if (in11) {
      int32_t s = row_span[r];
      if (s < 0) {
        viol = true;
      } else {
        int64_t cs = spans[4 * s + 2], cl = spans[4 * s + 3];
        viol = (c < cs) || (c >= cs + cl);
      }
    }
    const bool want[5] = {in11, inT, in21, viol, inT && r < m1};
    unsigned long long slot[5];
    block_slots<5>(b.counters, want, slot);
    if (!emit) continue;
    const unsigned long long s11 = slot[0], sT = slot[1], s21 = slot[2];
    double v = valid && vals ? vals[e] : 0.0;
    if (in11 && b.a11_r) {
      b.a11_r[s11] = (int32_t)r;
      b.a11_c[s11] = (int32_t)c;
      b.a11_v[s11] = v;
    }
    if (inT && b.t_r) {
      b.t_r[sT] = (int32_t)r;
      b.t_c[sT] = (int32_t)(c - n1);
      b.t_v[sT] = v;
    }
    if (in21 && b.a21_r) {
      b.a21_r[s21] = (int32_t)(r - m1);
      b.a21_c[s21] = (int32_t)c;
      b.a21_v[s21] = v;
    }
  }
}

__global__ void k_row_span(int64_t nspans, const int64_t* __restrict__ spans, int32_t* __restrict__ row_span) {
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < nspans; s += nw) {
    int64_t rs = spans[4 * s], rl = spans[4 * s + 1];
    for (int64_t r = rs + lane; r < rs + rl; r += 32) row_span[r] = (int32_t)s;
  }
}

__global__ void k_fill_i32(int32_t* a, int64_t n, int32_t v) {
  FPI_GRID_STRIDE(i, n) a[i] = v;
}

__global__ void k_remap(int64_t nnz, const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                        const int64_t* __restrict__ row_fwd, const int64_t* __restrict__ col_fwd,
                        int32_t* __restrict__ r_out, int32_t* __restrict__ c_out) {
  FPI_GRID_STRIDE(e, nnz) {
    r_out[e] = (int32_t)row_fwd[rows[e]];
    c_out[e] = (int32_t)col_fwd[cols[e]];
  }
}

}  // namespace

void expand_rows(fpi_context* h, int64_t m, const int64_t* indptr, int32_t* rows) {
  if (m == 0) return;
  k_expand_rows<<<grid_for(m * 32, 256, (int64_t)h->num_sms * 16), 256, 0, h->stream>>>(m, indptr, rows);
  FPI_LAUNCH_CHECK();
  note_launch(h);
}

// Sorted CSR (nmajor x nminor) from unsorted unique (major, minor, value) triples.
void build_csr(fpi_context* h, CubTemp& tmp, int64_t cnt, const int32_t* major, const int32_t* minor,
               const double* vals, int64_t nmajor, int64_t nminor, int64_t* out_ptr, int32_t* out_idx,
               double* out_val) {
  cudaStream_t s = h->stream;
  const int T = 256;
  const int64_t G = (int64_t)h->num_sms * 16;
  if (cnt > 0) {
    const int minor_bits = bits_for((uint64_t)(nminor > 0 ? nminor : 1));
    const int major_bits = bits_for((uint64_t)(nmajor > 0 ? nmajor : 1));
    FPI_REQUIRE(minor_bits + major_bits <= 64, FPI_ECAPACITY, "sort key exceeds 64 bits");
    Scratch<uint64_t> keys(cnt, s), keys2(cnt, s);
    Scratch<int32_t> pos(cnt, s), pos2(cnt, s);
    k_make_keys<<<grid_for(cnt, T, G), T, 0, s>>>(cnt, major, minor, minor_bits, keys, pos);
    sort_pairs(tmp, keys.get(), keys2.get(), pos.get(), pos2.get(), cnt, false, 0, minor_bits + major_bits, s);
    k_scatter_sorted<<<grid_for(cnt, T, G), T, 0, s>>>(cnt, keys2, pos2, vals, (1ull << minor_bits) - 1, out_idx,
                                                      out_val);
    k_ptr_from_sorted<<<grid_for(nmajor + 1, T, G), T, 0, s>>>(cnt, keys2, minor_bits, nmajor, out_ptr);
    FPI_LAUNCH_CHECK();
    note_launch(h, 4);
  } else {
    FPI_CUDA(cudaMemsetAsync(out_ptr, 0, sizeof(int64_t) * (nmajor + 1), s));
  }
}

// Transpose of a CSR: the entries are already in row-major order, so one STABLE radix sort on the
// column index alone (bits_for(q) bits instead of column + row bits) leaves every column's rows
// ascending.
void csr_transpose(fpi_context* h, int64_t p, int64_t q, int64_t nnz, const int64_t* indptr, const int32_t* indices,
                   const double* values, int64_t* t_ptr, int32_t* t_idx, double* t_val) {
  cudaStream_t s = h->stream;
  const int T = 256;
  const int64_t G = (int64_t)h->num_sms * 16;
  if (nnz == 0) {
    FPI_CUDA(cudaMemsetAsync(t_ptr, 0, sizeof(int64_t) * (q + 1), s));
    return;
  }
  CubTemp tmp(s);
  Scratch<int32_t> rows(nnz, s), pos(nnz, s), pos2(nnz, s);
  Scratch<uint32_t> keys2(nnz, s);
  expand_rows(h, p, indptr, rows);
  k_iota_pos<<<grid_for(nnz, T, G), T, 0, s>>>(nnz, pos);
  sort_pairs(tmp, reinterpret_cast<const uint32_t*>(indices), keys2.get(), pos.get(), pos2.get(), nnz, false, 0,
             bits_for((uint64_t)(q > 0 ? q : 1)), s);
  k_gather_transposed<<<grid_for(nnz, T, G), T, 0, s>>>(nnz, pos2, rows, values, t_idx, t_val);
  k_ptr_from_sorted32<<<grid_for(q + 1, T, G), T, 0, s>>>(nnz, keys2, q, t_ptr);
  FPI_LAUNCH_CHECK();
  note_launch(h, 5);
}

void csr_canonicalize(fpi_context* h, int64_t m, int64_t n, int64_t nnz, const int64_t* indptr,
                      const int32_t* indices, const double* values, int64_t* out_ptr, int32_t* out_idx,
                      double* out_val, int64_t* out_nnz) {
  cudaStream_t s = h->stream;
  const int T = 256;
  const int64_t G = (int64_t)h->num_sms * 16;
  Scratch<int> bad(1, s);
  FPI_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  if (m) k_check_canonical<<<grid_for(m, T, G), T, 0, s>>>(m, indptr, indices, values, bad);
  FPI_LAUNCH_CHECK();
  note_launch(h);
  if (!host_read(bad.get(), s)) {
    FPI_CUDA(cudaMemcpyAsync(out_ptr, indptr, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToDevice, s));
    if (nnz) {
      FPI_CUDA(cudaMemcpyAsync(out_idx, indices, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, s));
      FPI_CUDA(cudaMemcpyAsync(out_val, values, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
    }
    *out_nnz = nnz;
    return;
  }
  CubTemp tmp(s);
  Scratch<int32_t> rows(nnz, s), pos(nnz, s), pos2(nnz, s), head(nnz, s), run_id(nnz, s);
  Scratch<uint64_t> keys(nnz, s), keys2(nnz, s);
  expand_rows(h, m, indptr, rows);
  const int minor_bits = bits_for((uint64_t)(n > 0 ? n : 1));
  const int major_bits = bits_for((uint64_t)(m > 0 ? m : 1));
  k_coo_keys<<<grid_for(nnz, T, G), T, 0, s>>>(nnz, rows, indices, minor_bits, keys, pos);
  sort_pairs(tmp, keys.get(), keys2.get(), pos.get(), pos2.get(), nnz, false, 0, minor_bits + major_bits, s);
  k_run_heads<<<grid_for(nnz, T, G), T, 0, s>>>(nnz, keys2, head);
  exclusive_sum(tmp, head.get(), run_id.get(), nnz, s);
  const int64_t nruns = host_read(run_id.get() + nnz - 1, s) + host_read(head.get() + nnz - 1, s);
  Scratch<double> run_sum(nruns, s);
  Scratch<uint64_t> run_key(nruns, s);
  k_sum_runs<<<grid_for(nnz, T, G), T, 0, s>>>(nnz, keys2, pos2, values, head, run_sum, run_key, run_id);
  Scratch<int32_t> keep(nruns, s), nkeep(1, s), counts(m + 1, s);
  select_if(tmp, cub::CountingInputIterator<int32_t>(0), keep.get(), nkeep.get(), nruns, NonZeroAt{run_sum.get()}, s);
  const int64_t kept = host_read(nkeep.get(), s);
  FPI_CUDA(cudaMemsetAsync(counts.get(), 0, sizeof(int32_t) * (m + 1), s));
  if (kept)
    k_emit_canonical<<<grid_for(kept, T, G), T, 0, s>>>(kept, keep, run_key, run_sum, minor_bits, out_idx, out_val,
                                                        counts);
  k_counts_to_ptr_first<<<1, 1, 0, s>>>(out_ptr);
  inclusive_sum(tmp, counts.get(), out_ptr + 1, m, s);
  FPI_LAUNCH_CHECK();
  note_launch(h, 7);
  *out_nnz = kept;
}

// Region counts + structural check (pass 1), then optional emission into
// sorted CSR outputs (pass 2).
void partition(fpi_context* h, int64_t m, int64_t n, int64_t nnz, const int64_t* indptr, const int32_t* indices,
               const double* values, const int64_t* row_fwd, const int64_t* col_fwd, int64_t m1, int64_t n1,
               int64_t nspans, const int64_t* spans, fpi_partition_info* info, const PartOut* out) {
  cudaStream_t s = h->stream;
  const int T = 256;
  const int64_t G = (int64_t)h->num_sms * 16;
  CubTemp tmp(s);
  Scratch<int32_t> rows(nnz, s), row_span(m1 > 0 ? m1 : 1, s);
  Scratch<unsigned long long> counters(5, s);
  FPI_CUDA(cudaMemsetAsync(counters.get(), 0, sizeof(unsigned long long) * 5, s));
  expand_rows(h, m, indptr, rows);
  if (m1) {
    k_fill_i32<<<grid_for(m1, T, G), T, 0, s>>>(row_span, m1, -1);
    if (nspans) k_row_span<<<grid_for(nspans * 32, T, G), T, 0, s>>>(nspans, spans, row_span);
  }
  PartBufs b{};
  b.counters = counters;
  if (nnz)
    k_partition<<<grid_for(nnz, T, G), T, 0, s>>>(nnz, rows, indices, values, row_fwd, col_fwd, m1, n1, row_span,
                                                  spans, false, b);
  FPI_LAUNCH_CHECK();
  note_launch(h, 3);
  unsigned long long hc[5];
  FPI_CUDA(cudaMemcpyAsync(hc, counters.get(), sizeof(hc), cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  if (hc[3])
    throw Error(FPI_ESTRUCT, std::to_string(hc[3]) + " spoke-region nonzeros lie outside every block span");
  info->nnz_a11 = (int64_t)hc[0];
  info->nnz_a12 = (int64_t)hc[4];
  info->nnz_a21 = (int64_t)hc[2];
  info->nnz_a22 = (int64_t)(hc[1] - hc[4]);
  if (!out) return;
  const int64_t m2 = m - m1, n2 = n - n1;
  const int64_t n11 = (int64_t)hc[0], nT = (int64_t)hc[1], n21 = (int64_t)hc[2];
  Scratch<int32_t> a11_r, a11_c, t_r, t_c, a21_r, a21_c;
  Scratch<double> a11_v, t_v, a21_v;
  if (out->a11_ptr) {
    a11_r.alloc(n11, s); a11_c.alloc(n11, s); a11_v.alloc(n11, s);
    b.a11_r = a11_r; b.a11_c = a11_c; b.a11_v = a11_v;
  }
  if (out->t_ptr || out->tt_ptr) {
    t_r.alloc(nT, s); t_c.alloc(nT, s); t_v.alloc(nT, s);
    b.t_r = t_r; b.t_c = t_c; b.t_v = t_v;
  }
  if (out->a21_ptr || out->a21t_ptr) {
    a21_r.alloc(n21, s); a21_c.alloc(n21, s); a21_v.alloc(n21, s);
    b.a21_r = a21_r; b.a21_c = a21_c; b.a21_v = a21_v;
  }
  FPI_CUDA(cudaMemsetAsync(counters.get(), 0, sizeof(unsigned long long) * 5, s));
  if (nnz)
    k_partition<<<grid_for(nnz, T, G), T, 0, s>>>(nnz, rows, indices, values, row_fwd, col_fwd, m1, n1, row_span,
                                                  spans, true, b);
  FPI_LAUNCH_CHECK();
  note_launch(h);
  if (out->a11_ptr) build_csr(h, tmp, n11, a11_r, a11_c, a11_v, m1, n1, out->a11_ptr, out->a11_idx, out->a11_val);
  if (out->t_ptr) build_csr(h, tmp, nT, t_r, t_c, t_v, m, n2, out->t_ptr, out->t_idx, out->t_val);
  if (out->tt_ptr) {
    if (out->t_ptr)  // from the sorted T: one column-key sort
      csr_transpose(h, m, n2, nT, out->t_ptr, out->t_idx, out->t_val, out->tt_ptr, out->tt_idx, out->tt_val);
    else
      build_csr(h, tmp, nT, t_c, t_r, t_v, n2, m, out->tt_ptr, out->tt_idx, out->tt_val);
  }
  if (out->a21_ptr) build_csr(h, tmp, n21, a21_r, a21_c, a21_v, m2, n1, out->a21_ptr, out->a21_idx, out->a21_val);
  if (out->a21t_ptr) {
    if (out->a21_ptr)
      csr_transpose(h, m2, n1, n21, out->a21_ptr, out->a21_idx, out->a21_val, out->a21t_ptr, out->a21t_idx,
                    out->a21t_val);
    else
      build_csr(h, tmp, n21, a21_c, a21_r, a21_v, n1, m2, out->a21t_ptr, out->a21t_idx, out->a21t_val);
  }
}

void permute(fpi_context* h, int64_t m, int64_t n, int64_t nnz, const int64_t* indptr, const int32_t* indices,
             const double* values, const int64_t* row_fwd, const int64_t* col_fwd, int64_t* out_ptr,
             int32_t* out_idx, double* out_val) {
  cudaStream_t s = h->stream;
  CubTemp tmp(s);
  Scratch<int32_t> rows(nnz, s), r2(nnz, s), c2(nnz, s);
  expand_rows(h, m, indptr, rows);
  if (nnz) k_remap<<<grid_for(nnz, 256, (int64_t)h->num_sms * 16), 256, 0, h->stream>>>(nnz, rows, indices, row_fwd, col_fwd, r2, c2);
  FPI_LAUNCH_CHECK();
  build_csr(h, tmp, nnz, r2, c2, values, m, n, out_ptr, out_idx, out_val);
}

}  // namespace fpi

extern "C" int fpi_csr_canonicalize(fpi_handle h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                                    const int32_t* d_indices, const double* d_values, int64_t* d_out_indptr,
                                    int32_t* d_out_indices, double* d_out_values, int64_t* h_out_nnz) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(m >= 0 && n >= 0 && nnz >= 0, FPI_EDOMAIN, "bad CSR shape");
  fpi::csr_canonicalize(h, m, n, nnz, d_indptr, d_indices, d_values, d_out_indptr, d_out_indices, d_out_values,
                        h_out_nnz);
  FPI_API_END(h)
}

extern "C" int fpi_csr_transpose(fpi_handle h, int64_t p, int64_t q, int64_t nnz, const int64_t* d_indptr,
                                 const int32_t* d_indices, const double* d_values, int64_t* d_t_indptr,
                                 int32_t* d_t_indices, double* d_t_values) {
  FPI_API_BEGIN(h)
  fpi::csr_transpose(h, p, q, nnz, d_indptr, d_indices, d_values, d_t_indptr, d_t_indices, d_t_values);
  FPI_API_END(h)
}

extern "C" int fpi_partition_count(fpi_handle h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                                   const int32_t* d_indices, const int64_t* d_row_fwd, const int64_t* d_col_fwd,
                                   int64_t m1, int64_t n1, int64_t n_spans, const int64_t* d_spans,
                                   fpi_partition_info* info) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(info, FPI_EDOMAIN, "null info");
  FPI_REQUIRE(0 <= m1 && m1 <= m && 0 <= n1 && n1 <= n, FPI_EDOMAIN, "region sizes out of range");
  fpi::partition(h, m, n, nnz, d_indptr, d_indices, nullptr, d_row_fwd, d_col_fwd, m1, n1, n_spans, d_spans, info,
                 nullptr);
  FPI_API_END(h)
}

extern "C" int fpi_partition(fpi_handle h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                             const int32_t* d_indices, const double* d_values, const int64_t* d_row_fwd,
                             const int64_t* d_col_fwd, int64_t m1, int64_t n1, int64_t n_spans,
                             const int64_t* d_spans, int64_t* a11_ptr, int32_t* a11_idx, double* a11_val,
                             int64_t* t_ptr, int32_t* t_idx, double* t_val, int64_t* tt_ptr, int32_t* tt_idx,
                             double* tt_val, int64_t* a21_ptr, int32_t* a21_idx, double* a21_val, int64_t* a21t_ptr,
                             int32_t* a21t_idx, double* a21t_val) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(0 <= m1 && m1 <= m && 0 <= n1 && n1 <= n, FPI_EDOMAIN, "region sizes out of range");
  fpi::PartOut out{a11_ptr, a11_idx, a11_val, t_ptr, t_idx, t_val, tt_ptr, tt_idx, tt_val,
                   a21_ptr, a21_idx, a21_val, a21t_ptr, a21t_idx, a21t_val};
  fpi_partition_info info{};
  fpi::KTimer kt(h, "permute_partition(all kernels)", 0.0, 2.0 * 12.0 * nnz + 8.0 * (m + n));
  fpi::partition(h, m, n, nnz, d_indptr, d_indices, d_values, d_row_fwd, d_col_fwd, m1, n1, n_spans, d_spans, &info,
                 &out);
  FPI_API_END(h)
}

extern "C" int fpi_permute(fpi_handle h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                           const int32_t* d_indices, const double* d_values, const int64_t* d_row_fwd,
                           const int64_t* d_col_fwd, int64_t* d_out_indptr, int32_t* d_out_indices,
                           double* d_out_values) {
  FPI_API_BEGIN(h)
  fpi::permute(h, m, n, nnz, d_indptr, d_indices, d_values, d_row_fwd, d_col_fwd, d_out_indptr, d_out_indices,
               d_out_values);
  FPI_API_END(h)
}
