// Hub/spoke reordering of the bipartite graph (Algorithm 2), bit-exact with
// the reference reorder (reorder.py:158-287).
//
// Node ids are combined: instance (row) i -> i, feature (column) j -> m + j,
// exactly the universe the reference hands to connected_components
// (reorder.py:216-219).  Per iteration, on the current giant component:
//   1. degrees against active neighbours over the compacted edge list
//      (reorder.py:201-202; edges with an inactive endpoint were dropped when
//      the previous iteration compacted the list),
//   2. hubs = top ceil(k*count) active positive-degree nodes by
//      (degree desc, id asc): a stable descending radix sort of the
//      ascending candidate list (reorder.py:149-155), the first hub taking
//      the highest free id (reorder.py:206-212),
//   3. connected components of the residual with lock-free union-find
//      (link larger root under smaller root, so the representative is the
//      smallest member id -- the reference's GCC / spoke tie-break key,
//      reorder.py:229-234),
//   4. spoke components ordered by (size desc, min id asc) via a stable
//      descending sort of the ascending root list, laid out with exclusive
//      scans; members ascending within each side (reorder.py:246-257),
//   5. next active set = giant component; stop when it is below the quota
//      (reorder.py:259-269).  The terminal GCC takes the middle ids
//      (reorder.py:271-275).
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "capi_guard.cuh"
#include "cub_util.cuh"
#include "instrument.cuh"
#include "reorder.cuh"
#include <cmath>

namespace fpi {
namespace {

__global__ void k_expand_edges(int64_t m, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                               uint64_t* __restrict__ edges) {
  // one warp per row; edge = (row << 32) | col
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < m; r += nwarps) {
    int64_t b = indptr[r], e = indptr[r + 1];
    for (int64_t p = b + lane; p < e; p += 32) edges[p] = ((uint64_t)r << 32) | (uint32_t)indices[p];
  }
}

__global__ void k_fill_iota(int32_t* __restrict__ a, int64_t n) {
  FPI_GRID_STRIDE(i, n) a[i] = (int32_t)i;
}

__global__ void k_set_u8(uint8_t* __restrict__ a, int64_t n, uint8_t v) {
  FPI_GRID_STRIDE(i, n) a[i] = v;
}

__device__ __forceinline__ void warp_agg_inc(int32_t* ctr, int32_t key) {
  unsigned mask = __activemask();
  unsigned peers = __match_any_sync(mask, key);
  int leader = __ffs(peers) - 1;
  if ((int)(threadIdx.x & 31) == leader) atomicAdd(ctr + key, __popc(peers));
}

__global__ void k_gather_keys(const int32_t* __restrict__ ids, int64_t n, const int32_t* __restrict__ deg,
                              uint32_t* __restrict__ keys) {
  FPI_GRID_STRIDE(i, n) keys[i] = (uint32_t)deg[ids[i]];
}

// Union-find: parent[x] <= x always, so a root is the smallest id of its set.
__device__ __forceinline__ int32_t find_root(int32_t x, int32_t* parent) {
  int32_t cur = parent[x];
  if (cur != x) {
    int32_t prev = x, nxt;
    while (cur > (nxt = parent[cur])) {
      parent[prev] = nxt;  // path halving; benign race (values only move toward the root)
      prev = cur;
      cur = nxt;
    }
  }
  return cur;
}

struct IsSpokeRoot {
  const int32_t* parent;
  int32_t gcc;
  __device__ bool operator()(int32_t v) const { return parent[v] == v && v != gcc; }
};
struct InComp {
  const int32_t* parent;
  int32_t gcc;
  __device__ bool operator()(int32_t v) const { return parent[v] == gcc; }
};
struct IsActive {
  const uint8_t* state;
  __device__ bool operator()(int32_t v) const { return state[v] != 0; }
};
struct EdgeLive {
  const uint8_t* state;
  int32_t m;
  __device__ bool operator()(uint64_t e) const {
    return state[(int32_t)(e >> 32)] && state[(int32_t)(e & 0xffffffffu) + m];
  }
};

// Per spoke component (rank order): rows, cols and size, laid out by one exclusive scan of triples.
struct Tri {
  int64_t r, c, n;
};
struct TriSum {
  __host__ __device__ Tri operator()(const Tri& a, const Tri& b) const { return Tri{a.r + b.r, a.c + b.c, a.n + b.n}; }
};

__global__ void k_comp_table(const int32_t* __restrict__ roots_sorted, int64_t nc, const int32_t* __restrict__ csize,
                             const int32_t* __restrict__ crows, int32_t* __restrict__ rank_of_root,
                             Tri* __restrict__ tri) {
  FPI_GRID_STRIDE(i, nc) {
    int32_t r = roots_sorted[i];
    rank_of_root[r] = (int32_t)i;
    int64_t rows = crows[r], sz = csize[r];
    tri[i] = Tri{rows, sz - rows, sz};
  }
}

__global__ void k_write_spans(int64_t nc, const Tri* __restrict__ off, const Tri* __restrict__ tri, int64_t lo_t,
                              int64_t lo_f, int64_t* __restrict__ spans) {
  FPI_GRID_STRIDE(i, nc) {
    spans[4 * i + 0] = lo_t + off[i].r;
    spans[4 * i + 1] = tri[i].r;
    spans[4 * i + 2] = lo_f + off[i].c;
    spans[4 * i + 3] = tri[i].c;
  }
}

__global__ void k_node_rank_keys(const int32_t* __restrict__ nodes, int64_t cnt, const int32_t* __restrict__ parent,
                                 const int32_t* __restrict__ rank_of_root, uint32_t* __restrict__ keys) {
  FPI_GRID_STRIDE(i, cnt) keys[i] = (uint32_t)rank_of_root[parent[nodes[i]]];
}

__global__ void k_emit_spokes(const int32_t* __restrict__ nodes, const uint32_t* __restrict__ ranks, int64_t cnt,
                              int32_t m, const Tri* __restrict__ off, const Tri* __restrict__ tri, int64_t lo_t,
                              int64_t lo_f, int64_t* __restrict__ row_fwd, int64_t* __restrict__ col_fwd,
                              uint8_t* __restrict__ state) {
  FPI_GRID_STRIDE(p, cnt) {
    int32_t v = nodes[p];
    uint32_t c = ranks[p];
    int64_t pos = p - off[c].n;
    if (v < m) {
      row_fwd[v] = lo_t + off[c].r + pos;
    } else {
      col_fwd[v - m] = lo_f + off[c].c + pos - tri[c].r;
    }
    state[v] = 0;
  }
}

// Hub sort keys of both sides in one list: ascending (side, mask - degree) = rows first, each side
// degree-descending; the radix sort is stable, so ties keep the ascending id order.
__global__ void k_hub_keys(const int32_t* __restrict__ act, int64_t cnt_t, int64_t cnt, const int32_t* __restrict__ deg,
                           int deg_bits, uint32_t* __restrict__ keys) {
  const uint32_t mask = (deg_bits >= 32) ? 0xffffffffu : ((1u << deg_bits) - 1u);
  FPI_GRID_STRIDE(i, cnt) keys[i] = ((uint32_t)(i >= cnt_t) << deg_bits) | (mask - (uint32_t)deg[act[i]]);
}

// Hubs of both sides: the first min(q, #positive) of each side's segment of the sorted list; hub i
// of a side takes the id hi - i (reorder.py:206-212).
__global__ void k_assign_hubs2(const int32_t* __restrict__ ids, const uint32_t* __restrict__ keys, int64_t cnt_t,
                               int64_t qt, int64_t qf, int64_t hi_t, int64_t hi_f, int32_t m, int deg_bits,
                               int64_t* __restrict__ row_fwd, int64_t* __restrict__ col_fwd,
                               uint8_t* __restrict__ state, int* __restrict__ nhubs) {
  const uint32_t mask = (deg_bits >= 32) ? 0xffffffffu : ((1u << deg_bits) - 1u);
  FPI_GRID_STRIDE(i, qt + qf) {
    const bool col = i >= qt;
    const int64_t j = col ? i - qt : i;
    const int64_t pos = col ? cnt_t + j : j;
    if ((keys[pos] & mask) == mask) continue;  // degree 0: not a hub
    const int32_t v = ids[pos];
    if (col)
      col_fwd[v - m] = hi_f - j;
    else
      row_fwd[v] = hi_t - j;
    state[v] = 0;
    atomicAdd(nhubs + (col ? 1 : 0), 1);
  }
}

__global__ void k_assign_tail(const int32_t* __restrict__ act, int64_t cnt, int32_t m, int64_t cnt_t, int64_t lo_t,
                              int64_t lo_f, int64_t* __restrict__ row_fwd, int64_t* __restrict__ col_fwd) {
  FPI_GRID_STRIDE(i, cnt) {
    int32_t v = act[i];
    if (i < cnt_t)
      row_fwd[v] = lo_t + i;
    else
      col_fwd[v - m] = lo_f + (i - cnt_t);
  }
}

}  // namespace

// device-side kernels used by the one-sync-per-iteration driver
namespace {

// degrees over the compacted edge list whose length lives on the device
__global__ void k_degree_dev(const uint64_t* __restrict__ edges, const int* __restrict__ ne_p, int32_t m,
                             int32_t* __restrict__ deg) {
  const int64_t ne = *ne_p;
  FPI_GRID_STRIDE(e, ne) {
    uint64_t ed = edges[e];
    warp_agg_inc(deg, (int32_t)(ed >> 32));
    warp_agg_inc(deg, (int32_t)(ed & 0xffffffffu) + m);
  }
}

__global__ void k_hook_dev(const uint64_t* __restrict__ edges, const int* __restrict__ ne_p, int32_t m,
                           const uint8_t* __restrict__ state, int32_t* parent) {
  const int64_t ne = *ne_p;
  FPI_GRID_STRIDE(e, ne) {
    uint64_t ed = edges[e];
    int32_t u = (int32_t)(ed >> 32);
    int32_t v = (int32_t)(ed & 0xffffffffu) + m;
    if (!state[u] || !state[v]) continue;
    int32_t ru = find_root(u, parent), rv = find_root(v, parent);
    while (ru != rv) {
      if (ru < rv) {
        int32_t old = atomicCAS(parent + rv, rv, ru);
        if (old == rv) break;
        rv = find_root(old, parent);
      } else {
        int32_t old = atomicCAS(parent + ru, ru, rv);
        if (old == ru) break;
        ru = find_root(old, parent);
      }
    }
  }
}

__global__ void k_label_stats_dev(const int32_t* __restrict__ act, const int* __restrict__ cnt_p, int32_t m,
                                  int32_t* parent, int32_t* __restrict__ csize, int32_t* __restrict__ crows) {
  const int64_t cnt = *cnt_p;
  FPI_GRID_STRIDE(i, cnt) {
    int32_t v = act[i];
    int32_t r = v;
    while (parent[r] != r) r = parent[r];
    parent[v] = r;
    warp_agg_inc(csize, r);
    if (v < m) warp_agg_inc(crows, r);
  }
}

__global__ void k_pick_gcc_dev(const int32_t* __restrict__ act, const int* __restrict__ cnt_p,
                               const int32_t* __restrict__ parent, const int32_t* __restrict__ csize,
                               unsigned long long* best, int32_t* nroots) {
  const int64_t cnt = *cnt_p;
  unsigned long long local = 0;
  int32_t nr = 0;
  FPI_GRID_STRIDE(i, cnt) {
    int32_t v = act[i];
    if (parent[v] == v) {
      unsigned long long key = ((unsigned long long)(uint32_t)csize[v] << 32) | (uint32_t)(0x7fffffff - v);
      local = key > local ? key : local;
      ++nr;
    }
  }
  for (int o = 16; o; o >>= 1) {
    unsigned long long other = __shfl_xor_sync(0xffffffffu, local, o);
    local = other > local ? other : local;
    nr += __shfl_xor_sync(0xffffffffu, nr, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(best, local);
    atomicAdd(nroots, nr);
  }
}

struct IterScalars {
  unsigned long long best;
  int32_t nroots, h_t, h_f, acnt, ne, gcc_rows, pad0, pad1;
};

__global__ void k_collect(IterScalars* out, const unsigned long long* best, const int32_t* nroots, const int* hubs,
                          const int* acnt, const int* ne, const int32_t* crows) {
  if (threadIdx.x || blockIdx.x) return;
  out->best = *best;
  out->nroots = *nroots;
  out->h_t = hubs[0];
  out->h_f = hubs[1];
  out->acnt = *acnt;
  out->ne = *ne;
  const int32_t gcc = (int32_t)(0x7fffffff - (int64_t)(*best & 0xffffffffull));
  out->gcc_rows = (*best) ? crows[gcc] : 0;
}

// also clears the iteration's device counters (hub counts, GCC key, root count)
__global__ void k_reset_nodes_dev(const int32_t* __restrict__ act, int64_t cnt, int32_t* __restrict__ deg,
                                  int32_t* __restrict__ parent, int32_t* __restrict__ csize,
                                  int32_t* __restrict__ crows, int32_t* __restrict__ dsc,
                                  unsigned long long* __restrict__ best) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    dsc[0] = dsc[1] = dsc[4] = 0;
    *best = 0ull;
  }
  FPI_GRID_STRIDE(i, cnt) {
    int32_t v = act[i];
    deg[v] = 0;
    parent[v] = v;
    csize[v] = 0;
    crows[v] = 0;
  }
}

}  // namespace

// One host synchronisation per iteration: every count the host needs (hubs taken, active
// nodes left, component count, giant component) is gathered into one pinned readback; edge
// and node kernels take their lengths from device memory.
static void run_reorder(fpi_context* h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                        const int32_t* d_indices, double k, int64_t* d_row_fwd, int64_t* d_col_fwd,
                        ReorderOut& out) {
  cudaStream_t s = h->stream;
  const auto t_enter = std::chrono::steady_clock::now();
  FPI_REQUIRE(k > 0.0 && k < 1.0, FPI_EDOMAIN, "hub selection ratio k must be in (0, 1)");
  FPI_REQUIRE(m > 0 && n > 0, FPI_EDOMAIN, "graph has an empty node side");
  FPI_REQUIRE(m + n < (int64_t)INT32_MAX, FPI_ECAPACITY, "m + n exceeds the int32 node-id range");
  FPI_REQUIRE(nnz < (int64_t)INT32_MAX, FPI_ECAPACITY, "nnz exceeds the int32 edge-count range");
  const int64_t V = m + n;
  const int T = 256;
  const unsigned G = (unsigned)(h->num_sms * 8);
  CubTemp tmp(s);

  Scratch<uint64_t> edges(nnz, s), edges2(nnz, s);
  Scratch<uint8_t> state(V, s);
  Scratch<int32_t> deg(V, s), parent(V, s), csize(V, s), crows(V, s), rank_of_root(V, s);
  Scratch<int32_t> act(V, s), act2(V, s), cand(V, s), cand_sorted(V, s);
  Scratch<uint32_t> keys(V, s), keys_sorted(V, s);
  Scratch<Tri> tri(V, s), tri_off(V, s);
  // device scalars: [0] hubs rows, [1] hubs cols, [2] active count, [3] spoke roots (partition),
  // [4] nroots, [5] edge count
  Scratch<int32_t> dsc(8, s);
  Scratch<unsigned long long> d_best(1, s);
  Scratch<IterScalars> d_it(1, s);
  // pinned once per handle: a per-call cudaMallocHost / cudaFreeHost costs milliseconds and the
  // free synchronises the device
  if (!h->host_scalars) FPI_CUDA(cudaMallocHost(&h->host_scalars, 256));
  IterScalars* hs = static_cast<IterScalars*>(h->host_scalars);

  if (h->spans_cap < V) {
    if (h->d_spans) cudaFree(h->d_spans);
    FPI_CUDA(cudaMalloc((void**)&h->d_spans, sizeof(int64_t) * 4 * (V + 1)));
    h->spans_cap = V;
  }
  h->n_spans = 0;
  h->gcc_sizes.clear();

  if (nnz) k_expand_edges<<<G, T, 0, s>>>(m, d_indptr, d_indices, edges);
  k_set_u8<<<G, T, 0, s>>>(state, V, 1);
  k_fill_iota<<<G, T, 0, s>>>(act, V);
  int32_t* ne_d = dsc.get() + 5;
  {
    int32_t v = (int32_t)nnz;
    FPI_CUDA(cudaMemcpyAsync(ne_d, &v, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    FPI_CUDA(cudaStreamSynchronize(s));
  }
  FPI_LAUNCH_CHECK();
  note_launch(h, 3);

  int64_t cnt_t = m, cnt_f = n;
  int64_t lo_t = 0, lo_f = 0, hi_t = m - 1, hi_f = n - 1;
  int64_t iters = 0;
  bool any_edges = nnz > 0;
  const int deg_bits = bits_for((uint64_t)(m > n ? m : n));
  const int rank_bits = bits_for((uint64_t)V);

  const char* trace_env = getenv("FPI_TRACE_REORDER");
  const bool trace = trace_env != nullptr;
  const double trace_min_ms = trace ? atof(trace_env) : 0.0;  // print iterations at least this long
  auto titer = std::chrono::steady_clock::now();
  if (trace) fprintf(stderr, "[reorder] setup %.2f ms\n", std::chrono::duration<double, std::milli>(titer - t_enter).count());
  while (true) {
    ++iters;
    const int64_t q_t = (int64_t)std::ceil(k * (double)cnt_t);  // math.ceil(k * cnt), reorder.py:198-199
    const int64_t q_f = (int64_t)std::ceil(k * (double)cnt_f);
    const int64_t cnt = cnt_t + cnt_f;
    out.v_sum += cnt;  // SURVEY 8(d) accounting (E_t added once the iteration's edge count is read)

    // 1. degrees over the compacted edge list
    k_reset_nodes_dev<<<grid_for(cnt, T, G), T, 0, s>>>(act, cnt, deg, parent, csize, crows, dsc, d_best);
    if (any_edges) k_degree_dev<<<G, T, 0, s>>>(edges, ne_d, (int32_t)m, deg);
    // 2. hubs of both sides from one stable sort of the (ascending) active list
    {
      const int64_t qt = (cnt_t > 0 && q_t > 0) ? (q_t < cnt_t ? q_t : cnt_t) : 0;
      const int64_t qf = (cnt_f > 0 && q_f > 0) ? (q_f < cnt_f ? q_f : cnt_f) : 0;
      if (qt + qf > 0) {
        k_hub_keys<<<grid_for(cnt, T, G), T, 0, s>>>(act, cnt_t, cnt, deg, deg_bits, keys);
        sort_pairs(tmp, keys.get(), keys_sorted.get(), act.get(), cand_sorted.get(), cnt, /*descending=*/false, 0,
                   deg_bits + 1, s);
        k_assign_hubs2<<<grid_for(qt + qf, T, G), T, 0, s>>>(cand_sorted, keys_sorted, cnt_t, qt, qf, hi_t, hi_f,
                                                             (int32_t)m, deg_bits, d_row_fwd, d_col_fwd, state,
                                                             dsc.get());
      }
    }
    // active list without the hubs (count on device)
    select_if(tmp, act.get(), act2.get(), dsc.get() + 2, cnt, IsActive{state}, s);
    std::swap(act, act2);
    // 3. connected components of the residual
    if (any_edges) k_hook_dev<<<G, T, 0, s>>>(edges, ne_d, (int32_t)m, state, parent);
    k_label_stats_dev<<<grid_for(cnt, T, G), T, 0, s>>>(act, dsc.get() + 2, (int32_t)m, parent, csize, crows);
    k_pick_gcc_dev<<<grid_for(cnt, T, G), T, 0, s>>>(act, dsc.get() + 2, parent, csize, d_best, dsc.get() + 4);
    k_collect<<<1, 1, 0, s>>>(d_it, d_best, dsc.get() + 4, dsc.get(), dsc.get() + 2, ne_d, crows);
    FPI_CUDA(cudaMemcpyAsync(hs, d_it.get(), sizeof(IterScalars), cudaMemcpyDeviceToHost, s));
    const auto tsync0 = std::chrono::steady_clock::now();
    FPI_CUDA(cudaStreamSynchronize(s));  // the one host synchronisation of the iteration
    if (trace) {
      const auto now = std::chrono::steady_clock::now();
      const double it_ms = std::chrono::duration<double, std::milli>(now - titer).count();
      const double sy_ms = std::chrono::duration<double, std::milli>(now - tsync0).count();
      if (it_ms >= trace_min_ms) fprintf(stderr, "[reorder] iteration %lld: %.2f ms (sync wait %.2f ms)\n", (long long)iters, it_ms, sy_ms);
      titer = now;
    }
    FPI_LAUNCH_CHECK();
    note_launch(h, 8);
    const int64_t h_t = hs->h_t, h_f = hs->h_f;
    out.e_sum += any_edges ? (int64_t)hs->ne : 0;
    hi_t -= h_t;
    hi_f -= h_f;
    cnt_t -= h_t;
    cnt_f -= h_f;
    const int64_t acnt = cnt_t + cnt_f;
    if (acnt == 0) {  // reorder.py:224-226
      h->gcc_sizes.push_back(0);
      break;
    }
    const int32_t gcc = (int32_t)(0x7fffffff - (int64_t)(hs->best & 0xffffffffull));
    const int64_t gcc_size = (int64_t)(hs->best >> 32);
    const int64_t gcc_t = hs->gcc_rows, gcc_f = gcc_size - gcc_t;
    const int64_t nsc = (int64_t)hs->nroots - 1;
    const int64_t nsp = acnt - gcc_size;

    // 4. one pass over the active list: the giant component (next active set) | spoke roots |
    //    other spoke nodes, each in ascending id order (this CUB writes the unselected part in input
    //    order; tests/test_reorder_gpu.py pins it); roots and other spokes land contiguously in
    //    cand (roots first), which orders every component root-first = ascending.
    three_way_partition(tmp, act.get(), act2.get(), cand.get(), cand.get() + nsc,
                        dsc.get() + 2, acnt, InComp{parent, gcc}, IsSpokeRoot{parent, gcc}, s);
    note_launch(h, 2);
    if (nsc > 0) {
      // spoke components -> blocks (size desc, min id asc), members ascending within each side
      k_gather_keys<<<grid_for(nsc, T, G), T, 0, s>>>(cand, nsc, csize, keys);
      sort_pairs(tmp, keys.get(), keys_sorted.get(), cand.get(), cand_sorted.get(), nsc, true, 0, rank_bits, s);
      k_comp_table<<<grid_for(nsc, T, G), T, 0, s>>>(cand_sorted, nsc, csize, crows, rank_of_root, tri);
      exclusive_scan(tmp, tri.get(), tri_off.get(), TriSum{}, Tri{0, 0, 0}, nsc, s);
      k_write_spans<<<grid_for(nsc, T, G), T, 0, s>>>(nsc, tri_off, tri, lo_t, lo_f, h->d_spans + 4 * h->n_spans);
      k_node_rank_keys<<<grid_for(nsp, T, G), T, 0, s>>>(cand, nsp, parent, rank_of_root, keys);
      sort_pairs(tmp, keys.get(), keys_sorted.get(), cand.get(), cand_sorted.get(), nsp, false, 0, rank_bits, s);
      k_emit_spokes<<<grid_for(nsp, T, G), T, 0, s>>>(cand_sorted, keys_sorted, nsp, (int32_t)m, tri_off, tri, lo_t,
                                                      lo_f, d_row_fwd, d_col_fwd, state);
      FPI_LAUNCH_CHECK();
      note_launch(h, 8);
      h->n_spans += nsc;
    }
    lo_t += cnt_t - gcc_t;
    lo_f += cnt_f - gcc_f;

    // 5. giant component becomes the active set (its count was written to dsc[2] by the partition)
    std::swap(act, act2);
    h->gcc_sizes.push_back(gcc_size);
    cnt_t = gcc_t;
    cnt_f = gcc_f;
    if (gcc_t < q_t || gcc_f < q_f) break;  // reorder.py:268-269
    // compact edges to the new active set (length stays on the device)
    if (any_edges) {
      select_if(tmp, edges.get(), edges2.get(), ne_d, hs->ne, EdgeLive{state, (int32_t)m}, s);
      std::swap(edges, edges2);
      note_launch(h, 1);
    }
  }
  // terminal GCC: middle ids, ascending (reorder.py:271-275)
  const int64_t rem = cnt_t + cnt_f;
  if (rem) {
    k_assign_tail<<<grid_for(rem, T, G), T, 0, s>>>(act, rem, (int32_t)m, cnt_t, lo_t, lo_f, d_row_fwd, d_col_fwd);
    FPI_LAUNCH_CHECK();
    note_launch(h, 1);
  }
  FPI_CUDA(cudaStreamSynchronize(s));
  if (trace)
    fprintf(stderr, "[reorder] loop+tail done %.2f ms after entry\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_enter).count());
  out.m1 = lo_t;
  out.n1 = lo_f;
  out.m2 = m - lo_t;
  out.n2 = n - lo_f;
  out.T = iters;
}

}  // namespace fpi

extern "C" int fpi_reorder(fpi_handle h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                           const int32_t* d_indices, double k, int64_t* d_row_fwd, int64_t* d_col_fwd,
                           fpi_reorder_info* info) {
  FPI_API_BEGIN(h)
  fpi::ReorderOut o{};
  // algorithmic bytes: sum_t (3 * 8 * E_t + 4 * 8 * V_t), known once the loop ends
  fpi::KTimer kt(h, "reorder_loop(all kernels)", 0.0, 0.0);
  // the persistent device loop unless it is outside its static limits (or the host loop is forced)
  const bool hostloop = getenv("FPI_REORDER_HOSTLOOP") != nullptr;
  if (hostloop || !fpi::run_reorder_persistent(h, m, n, nnz, d_indptr, d_indices, k, d_row_fwd, d_col_fwd, o))
    fpi::run_reorder(h, m, n, nnz, d_indptr, d_indices, k, d_row_fwd, d_col_fwd, o);
  kt.bytes = 24.0 * (double)o.e_sum + 32.0 * (double)o.v_sum;
  if (info) {
    info->m1 = o.m1;
    info->n1 = o.n1;
    info->m2 = o.m2;
    info->n2 = o.n2;
    info->n_iterations = o.T;
    info->n_spans = h->n_spans;
    info->n_gcc = (int64_t)h->gcc_sizes.size();
    info->edges_visited = o.e_sum;
    info->nodes_visited = o.v_sum;
  }
  FPI_API_END(h)
}

extern "C" int fpi_reorder_fetch(fpi_handle h, int64_t* d_spans, int64_t* h_gcc) {
  FPI_API_BEGIN(h)
  if (d_spans && h->n_spans)
    FPI_CUDA(cudaMemcpyAsync(d_spans, h->d_spans, sizeof(int64_t) * 4 * h->n_spans, cudaMemcpyDeviceToDevice,
                             h->stream));
  if (h_gcc)
    for (size_t i = 0; i < h->gcc_sizes.size(); ++i) h_gcc[i] = h->gcc_sizes[i];
  FPI_CUDA(cudaStreamSynchronize(h->stream));
  FPI_API_END(h)
}
