// Dense core of a skewed sparse block.
//
// The column update's sparse block T = [A12; A22] (pinv.py:202-203) joins the hub columns of A
// to all rows; on Zipf-by-Zipf inputs (BASELINE configs[3]) its heavy rows x heavy columns
// rectangle is nearly dense -- at c4 4,373 rows x 1,610 columns hold 62% of T's 4.6M entries at
// 41% density -- and every entry of a gather SpMM with k = 2r columns moves 8k bytes through
// L1 / L2 (sparse.py:20-39's products are gather-bound).  A dense cell costs
// 2k DMMA flops instead: ~0.08 ns against ~0.67 ns per entry at k = 1000, so a rectangle denser
// than ~1/8 is cheaper on the tensor pipe.  build_sparse_core picks the rectangle, scatters it
// into a dense panel and rewrites S and S^T without its entries; InnerOp::apply / applyT
// (svd_engine.cu) then run  remainder SpMM + gathered DMMA product.
//
// Selection (all counts on the device, one host read):
//   R0 = rows with at least max(64, q2 / 40) entries
//   C  = columns with at least |R0| / 8 entries inside R0
//   R  = rows with at least |C| / 8 entries inside C
// The remainder S' is compacted row by row from S, its transpose by the stable CSR transpose.
// Every product keeps a fixed summation order (the core's GEMM is the deterministic split-K
// DMMA kernel, the remainder keeps its CSR order), so results stay bit-reproducible.
#include <cstdlib>

#include "common.cuh"
#include "cub_util.cuh"
#include "instrument.cuh"
#include "sparse.cuh"
#include "sparse_core.cuh"

namespace fpi {
namespace {

constexpr int FRAC = 8;  // a core row / column is at least 1 / FRAC dense inside the rectangle

__global__ void k_flag_by_degree(int64_t n, const int64_t* __restrict__ ptr, int64_t thr, int32_t* __restrict__ flag) {
  FPI_GRID_STRIDE(i, n) flag[i] = (ptr[i + 1] - ptr[i] >= thr) ? 1 : 0;
}

// cnt[row] = entries of the row whose column is flagged; one warp per row
__global__ void k_count_flagged(int64_t nrows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                const int32_t* __restrict__ flag, int32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows; r += nw) {
    int c = 0;
    for (int64_t e = ptr[r] + lane; e < ptr[r + 1]; e += 32) c += flag[idx[e]];
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[r] = c;
  }
}

// ccnt[c] += entries of flagged rows in column c; one warp per flagged row of S (rows are at most
// q2 long, while a hub row of S^T can hold most of the matrix: counting from the S side keeps
// every warp's walk short).  Integer atomics: the counts do not depend on the order.
__global__ void k_count_cols_in_rows(int64_t nrows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                     const int32_t* __restrict__ rowflag, int32_t* __restrict__ ccnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows; r += nw) {
    if (!rowflag[r]) continue;
    for (int64_t e = ptr[r] + lane; e < ptr[r + 1]; e += 32) atomicAdd(ccnt + idx[e], 1);
  }
}

__global__ void k_flag_by_count(int64_t n, const int32_t* __restrict__ cnt, const int* __restrict__ total, int min_cnt,
                                int32_t* __restrict__ flag) {
  const int t = *total;
  FPI_GRID_STRIDE(i, n) flag[i] = (t > 0 && cnt[i] >= min_cnt && (int64_t)cnt[i] * FRAC >= t) ? 1 : 0;
}

// rem[i] = entries the row keeps; core[i] = entries it hands to the dense panel
__global__ void k_split_counts(int64_t n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ cnt,
                               const int32_t* __restrict__ flag, int64_t* __restrict__ rem,
                               int64_t* __restrict__ core) {
  FPI_GRID_STRIDE(i, n + 1) {
    if (i == n) {
      rem[i] = 0;
      if (core) core[i] = 0;
      continue;
    }
    const int64_t c = flag[i] ? cnt[i] : 0;
    rem[i] = ptr[i + 1] - ptr[i] - c;
    if (core) core[i] = c;
  }
}

__global__ void k_iota32(int32_t* a, int64_t n) {
  FPI_GRID_STRIDE(i, n) a[i] = (int32_t)i;
}

struct Flagged {
  const int32_t* f;
  __device__ bool operator()(int32_t i) const { return f[i] != 0; }
};

__global__ void k_positions(int64_t n, const int32_t* __restrict__ list, int32_t* __restrict__ pos) {
  FPI_GRID_STRIDE(i, n) pos[list[i]] = (int32_t)i;
}

// Row-ordered compaction of the entries outside the rectangle; the ones inside go to the panel.
template <bool DENSE>
__global__ void k_fill_remainder(int64_t nrows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                 const double* __restrict__ val, const int32_t* __restrict__ rowflag,
                                 const int32_t* __restrict__ colflag, const int64_t* __restrict__ optr,
                                 int32_t* __restrict__ oidx, double* __restrict__ oval,
                                 const int32_t* __restrict__ rowpos, const int32_t* __restrict__ colpos,
                                 double* __restrict__ dense, int64_t ldd) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows; r += nw) {
    const bool in_core_row = rowflag[r] != 0;
    const int64_t b = ptr[r], e = ptr[r + 1];
    int64_t o = optr[r];
    for (int64_t base = b; base < e; base += 32) {
      const int64_t my = base + lane;
      const bool valid = my < e;
      int32_t c = 0;
      double v = 0.0;
      if (valid) {
        c = idx[my];
        v = val[my];
      }
      const bool core = valid && in_core_row && colflag[c] != 0;
      const bool keep = valid && !core;
      const unsigned mask = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int64_t at = o + __popc(mask & lt);
        oidx[at] = c;
        oval[at] = v;
      }
      o += __popc(mask);
      if (DENSE && core) dense[(int64_t)rowpos[r] * ldd + colpos[c]] = v;
    }
  }
}

__global__ void k_pack3(const int* a, const int* b, const int64_t* c, int64_t* out) {
  out[0] = *a;
  out[1] = *b;
  out[2] = *c;
}

template <typename T, typename O>
void reduce_sum(CubTemp& tmp, const T* in, O* out, int64_t n, cudaStream_t s) {
  size_t b = 0;
  FPI_CUDA(cub::DeviceReduce::Sum(nullptr, b, in, out, (int)n, s));
  FPI_CUDA(cub::DeviceReduce::Sum(tmp.need(b), b, in, out, (int)n, s));
}

}  // namespace

void build_sparse_core(fpi_context* h, int64_t p, int64_t q2, int64_t nnz, const int64_t* s_ptr,
                       const int32_t* s_idx, const double* s_val, const int64_t* st_ptr, const int32_t* st_idx,
                       const double* st_val, SparseCore& core) {
  core.use = false;
  // FPI_SPMM_CORE: 0 = never, force = also on small / sparse inputs (tests), unset = cost rule
  const char* env = getenv("FPI_SPMM_CORE");
  const bool off = env && env[0] == '0';
  const bool force = env && env[0] == 'f';
  if (off || !s_ptr || !st_ptr || p <= 0 || q2 <= 0 || nnz <= 0) return;
  if (p >= (1ll << 31) || q2 >= (1ll << 31) || nnz >= (1ll << 31)) return;
  if (!force && nnz < (1 << 20)) return;  // the whole SpMM is a few hundred microseconds
  cudaStream_t s = h->stream;
  const unsigned G = (unsigned)(h->num_sms * 16);
  CubTemp tmp(s);
  const int64_t thr = force ? 2 : std::max<int64_t>(64, q2 / 40);
  const int min_cnt = force ? 1 : 8;
  Scratch<int32_t> rflag(p, s), cflag(q2, s), rcnt(p, s), ccnt(q2, s);
  Scratch<int> nR0(1, s), nC(1, s), nR(1, s);
  Scratch<int64_t> rrem(p + 1, s), rcore(p + 1, s), ncore(1, s), packed(3, s);
  k_flag_by_degree<<<grid_for(p, 256, G), 256, 0, s>>>(p, s_ptr, thr, rflag);
  reduce_sum(tmp, rflag.get(), nR0.get(), p, s);
  FPI_CUDA(cudaMemsetAsync(ccnt.get(), 0, sizeof(int32_t) * q2, s));
  k_count_cols_in_rows<<<grid_for(p * 32, 256, G), 256, 0, s>>>(p, s_ptr, s_idx, rflag, ccnt);
  k_flag_by_count<<<grid_for(q2, 256, G), 256, 0, s>>>(q2, ccnt, nR0, min_cnt, cflag);
  reduce_sum(tmp, cflag.get(), nC.get(), q2, s);
  k_count_flagged<<<grid_for(p * 32, 256, G), 256, 0, s>>>(p, s_ptr, s_idx, cflag, rcnt);
  k_flag_by_count<<<grid_for(p, 256, G), 256, 0, s>>>(p, rcnt, nC, min_cnt, rflag);
  reduce_sum(tmp, rflag.get(), nR.get(), p, s);
  k_split_counts<<<grid_for(p + 1, 256, G), 256, 0, s>>>(p, s_ptr, rcnt, rflag, rrem, rcore);
  reduce_sum(tmp, rcore.get(), ncore.get(), p, s);
  k_pack3<<<1, 1, 0, s>>>(nR, nC, ncore, packed);
  FPI_LAUNCH_CHECK();
  note_launch(h, 12);
  int64_t hv[3];
  host_read_n(packed.get(), hv, 3, s);
  const int64_t n_r = hv[0], n_c = hv[1], n_core = hv[2];
  if (n_r <= 0 || n_c <= 0 || n_core <= 0) return;
  const double cells = (double)n_r * (double)n_c;
  if (!force) {
    // worth it when the rectangle takes a real share of the gathers and a dense cell (2k flops at
    // ~25 TFLOP/s) undercuts what its entries cost as gathers (8k bytes at ~12 TB/s): density > 1/8
    if ((double)n_core < 0.2 * (double)nnz || (double)n_core < 0.15 * cells) return;
    if (cells * 8.0 > 4e9) return;
  }
  core.nR = n_r;
  core.nC = n_c;
  core.core_nnz = n_core;
  core.rem_nnz = nnz - n_core;
  core.rows.alloc(n_r, s);
  core.cols.alloc(n_c, s);
  Scratch<int32_t> ids(std::max(p, q2), s), rpos(p, s), cpos(q2, s);
  Scratch<int> cnt(1, s);
  k_iota32<<<grid_for(std::max(p, q2), 256, G), 256, 0, s>>>(ids, std::max(p, q2));
  select_if(tmp, ids.get(), core.rows.get(), cnt.get(), p, Flagged{rflag.get()}, s);
  select_if(tmp, ids.get(), core.cols.get(), cnt.get(), q2, Flagged{cflag.get()}, s);
  FPI_CUDA(cudaMemsetAsync(rpos.get(), 0xFF, sizeof(int32_t) * p, s));
  FPI_CUDA(cudaMemsetAsync(cpos.get(), 0xFF, sizeof(int32_t) * q2, s));
  k_positions<<<grid_for(n_r, 256, G), 256, 0, s>>>(n_r, core.rows, rpos);
  k_positions<<<grid_for(n_c, 256, G), 256, 0, s>>>(n_c, core.cols, cpos);
  core.r_ptr.alloc(p + 1, s);
  core.rt_ptr.alloc(q2 + 1, s);
  exclusive_sum(tmp, rrem.get(), core.r_ptr.get(), p + 1, s);
  core.r_idx.alloc(core.rem_nnz + 1, s);
  core.r_val.alloc(core.rem_nnz + 1, s);
  core.rt_idx.alloc(core.rem_nnz + 1, s);
  core.rt_val.alloc(core.rem_nnz + 1, s);
  core.dense.alloc((size_t)n_r * n_c, s);
  FPI_CUDA(cudaMemsetAsync(core.dense.get(), 0, sizeof(double) * n_r * n_c, s));
  k_fill_remainder<true><<<grid_for(p * 32, 256, G), 256, 0, s>>>(p, s_ptr, s_idx, s_val, rflag, cflag, core.r_ptr,
                                                                  core.r_idx, core.r_val, rpos, cpos, core.dense,
                                                                  n_c);
  FPI_LAUNCH_CHECK();
  note_launch(h, 8);
  // S'^T by the stable transpose (one radix sort on the column key): a warp-per-row compaction of
  // S^T would serialise on its hub rows
  csr_transpose(h, p, q2, core.rem_nnz, core.r_ptr, core.r_idx, core.r_val, core.rt_ptr, core.rt_idx, core.rt_val);
  core.use = true;
}

}  // namespace fpi
