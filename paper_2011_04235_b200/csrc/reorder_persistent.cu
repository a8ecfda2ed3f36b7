// Hub/spoke reordering (Algorithm 2, reference reorder.py:158-287) as ONE persistent cooperative
// kernel: the whole iteration loop runs on the device with grid barriers between its phases, so
// an iteration costs ~20 barriers instead of ~25 kernel launches (several of them multi-kernel
// CUB sorts) plus a host round trip.  Bit-exact with the host-driven loop in reorder.cu and with
// the reference: every ordering decision is re-derived from (degree, id) / (size, min id) keys.
//
// Per iteration, on the active node list `act` (ascending combined ids; row i -> i, column j ->
// m + j) and the live edge list (both endpoints active):
//   P1  degrees over the live edges (reorder.py:201-202)
//   P2  hub threshold per side by an 11-bit-per-level radix select over the degrees: the
//       quota-th largest degree d*, how many nodes lie above it, how many d* nodes to take
//   P3  (only if d* ties must be split) per-CTA counts of d* nodes -> ascending-id ranks
//   P4  hubs appended to a per-side list
//   P5  hub ranks by (degree desc, id asc) (reorder.py:149-155), one warp per hub; the first
//       hub takes the highest free id (reorder.py:206-212)
//   P6  union-find hooking over the residual edges (root = smallest member id)
//   P7  labels (full path compression), component sizes and row counts
//   P8  giant component = max (size, -min id) (reorder.py:228-234)
//   P9/P10 ordered three-way partition of the active list: giant component (next `act`) |
//       spoke roots | other spoke nodes, all ascending
//       Spoke roots / nodes are only logged here: their blocks and ids depend on nothing later
//       iterations change, so they are laid out once after the loop (below).
//   P15 edge list compacted to the new giant component (unordered: neither degrees nor the
//       union-find result depend on edge order); the next iteration's degrees counted on the way.
// After the loop, all spoke components of all iterations are ordered by (iteration, size desc,
// min id asc) with two grid-wide stable radix sorts; one exclusive scan of their (rows, cols) gives
// the spans (the scan across iterations is exactly each iteration's lo_t / lo_f), and one more
// stable sort groups the logged spoke nodes by component (reorder.py:236-257).
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "cub_util.cuh"
#include "instrument.cuh"
#include "reorder.cuh"

namespace cg = cooperative_groups;

namespace fpi {
namespace {

#ifndef RP_HALVING
#define RP_HALVING 1
#endif
constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int HBITS = 11;
constexpr int HB = 1 << HBITS;
constexpr int HUB_CAP = 1 << 15;      // hubs per side per iteration (ranked by brute force)

struct Ctl {
  int nhub[2];
  int nroots;
  int maxsz;
  int ne_next[2];
  unsigned long long best;
  long long out[8];  // lo_t, lo_f, iterations, spans, gcc entries, sum E_t, sum V_t
};

struct Params {
  int32_t m, n;
  double k;
  int levels;  // hub-degree radix-select levels (11 bits each)
  int hk;      // edges in flight per thread when hooking
  int hshort;  // skip an edge whose endpoints already share a parent
  int ne0;
  uint64_t* e0;
  uint64_t* e1;
  uint8_t* state;
  int32_t* deg;
  int32_t* parent;
  int32_t* csize;
  int32_t* crows;
  int32_t* act0;
  int32_t* act1;
  int32_t* cand;
  uint32_t* k0;
  uint32_t* k1;
  int32_t* v0;
  int32_t* v1;
  int32_t* rank_of_root;
  int32_t* rlog;   // spoke roots of every iteration (ascending within an iteration)
  int32_t* riter;  // their iteration
  uint64_t* tri;   // per spoke component (rank order): rows << 32 | cols
  uint64_t* toff;  // exclusive prefix of tri
  int64_t* row_fwd;
  int64_t* col_fwd;
  int64_t* spans;
  int64_t* gcc_sizes;
  int32_t* hist;  // [3][2][HB]
  int32_t* dig;   // [256][G] + [256]
  int64_t* blk;   // [G][4]
  uint64_t* hubkeys;  // [2][HUB_CAP]
  Ctl* ctl;
  unsigned long long* prof;  // optional per-phase nanoseconds (FPI_REORDER_PROFILE)
};

using BlockScanU64 = cub::BlockScan<unsigned long long, NT>;
using BlockScanInt = cub::BlockScan<int, NT>;

struct Smem {
  int hist[2][HB];
  int wcnt[NW][256];
  int run[256];
  int base[256];
  int tile[256];
  long long bc[8];
  unsigned long long red[NW];
  union {
    typename BlockScanU64::TempStorage u64;
    typename BlockScanInt::TempStorage i32;
  } scan;
};

// Plain (L1-cacheable) loads: grid.sync's fences order them after the previous phase's writes,
// and hot addresses (the giant component's root, hub states) are then served by L1 instead of
// serialising on one L2 slice.
template <typename T>
__device__ __forceinline__ T ld_(const T* p) {
  return *p;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void agg_inc(int32_t* ctr, int32_t key) {
  const unsigned mask = __activemask();
  const unsigned peers = __match_any_sync(mask, key);
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(ctr + key, __popc(peers));
}

__device__ __forceinline__ int32_t find_root_cg(int32_t x, int32_t* parent) {
  int32_t cur = ld_(parent + x);
  if (cur != x) {
    int32_t prev = x, nxt;
    while (cur > (nxt = ld_(parent + cur))) {
      if (RP_HALVING) parent[prev] = nxt;  // path halving (benign race: values only move toward the root)
      prev = cur;
      cur = nxt;
    }
  }
  return cur;
}

// find_root_cg with the first parent load already done
__device__ __forceinline__ int32_t find_root_from(int32_t x, int32_t cur, int32_t* parent) {
  if (cur != x) {
    int32_t prev = x, nxt;
    while (cur > (nxt = ld_(parent + cur))) {
      if (RP_HALVING) parent[prev] = nxt;
      prev = cur;
      cur = nxt;
    }
  }
  return cur;
}

// Block-wide sum (every thread gets the total).  Callers separate consecutive uses by the
// __syncthreads at its entry.
__device__ unsigned long long block_sum(unsigned long long v, Smem& sm) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long tot = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) tot += sm.red[w];
  return tot;
}

__device__ unsigned long long block_max(unsigned long long v, Smem& sm) {
  for (int o = 16; o; o >>= 1) {
    const unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long r = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) r = sm.red[w] > r ? sm.red[w] : r;
  return r;
}

// Sum of field `f` of the per-CTA counters of the CTAs before `b` (ordered chunk offsets).
__device__ int64_t cta_prefix(const int64_t* blk, int f, int b, Smem& sm) {
  unsigned long long v = 0;
  for (int c = threadIdx.x; c < b; c += NT) v += (unsigned long long)ld_(blk + 4 * c + f);
  return (int64_t)block_sum(v, sm);
}

__device__ __forceinline__ int field21(unsigned long long x, int f) { return (int)((x >> (21 * f)) & 0x1fffffull); }

// One stable LSD radix pass (8 bits at `shift`) of (kin, vin)[0, n) into (kout, vout).
// GRID: each CTA takes a contiguous chunk, digit offsets through `dig` (three grid barriers).
// !GRID: the calling CTA sorts the whole list (block barriers only).
template <bool GRID>
__device__ void radix_pass(cg::grid_group& grid, const uint32_t* kin, const int32_t* vin, uint32_t* kout,
                           int32_t* vout, int64_t n, int shift, int32_t* dig, Smem& sm) {
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  const int G = GRID ? (int)gridDim.x : 1, b = GRID ? (int)blockIdx.x : 0;
  const int64_t c0 = n * b / G, c1 = n * (b + 1) / G;
  if (t < 256) sm.run[t] = 0;
  __syncthreads();
  for (int64_t i = c0 + t; i < c1; i += NT) atomicAdd(&sm.run[(ld_(kin + i) >> shift) & 255], 1);
  __syncthreads();
  if (GRID) {
    if (t < 256) dig[t * G + b] = sm.run[t];
    grid.sync();
    const int gw = (int)((blockIdx.x * NT + t) >> 5), nwg = G * NW;
    for (int d = gw; d < 256; d += nwg) {
      int carry = 0;
      for (int cb = 0; cb < G; cb += 32) {
        const int c = cb + lane;
        const int x = c < G ? ld_(dig + d * G + c) : 0;
        int incl = x;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (c < G) dig[d * G + c] = carry + incl - x;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) dig[256 * G + d] = carry;
    }
    grid.sync();
  }
  {
    int tot = 0;
    if (t < 256) tot = GRID ? ld_(dig + 256 * G + t) : sm.run[t];
    int ex;
    BlockScanInt(sm.scan.i32).ExclusiveSum(tot, ex);
    __syncthreads();
    if (t < 256) {
      sm.base[t] = ex + (GRID ? ld_(dig + t * G + b) : 0);
      sm.run[t] = 0;
    }
    for (int i = t; i < NW * 256; i += NT) (&sm.wcnt[0][0])[i] = 0;
    __syncthreads();
  }
  for (int64_t i0 = c0; i0 < c1; i0 += NT) {
    const int64_t i = i0 + t;
    const bool valid = i < c1;
    uint32_t key = 0;
    int32_t val = 0;
    int d = 256;
    if (valid) {
      key = ld_(kin + i);
      val = ld_(vin + i);
      d = (int)((key >> shift) & 255u);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int lr = __popc(peers & lanemask_lt());
    if (valid && lr == 0) sm.wcnt[w][d] = __popc(peers);
    __syncthreads();
    if (t < 256) {
      int r = 0;
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) {
        const int c = sm.wcnt[ww][t];
        sm.wcnt[ww][t] = r;
        r += c;
      }
      sm.tile[t] = r;
    }
    __syncthreads();
    if (valid) {
      const int64_t pos = (int64_t)sm.base[d] + sm.run[d] + sm.wcnt[w][d] + lr;
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
    if (t < 256) {
      sm.run[t] += sm.tile[t];
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) sm.wcnt[ww][t] = 0;
    }
    __syncthreads();
  }
  if (GRID) {
    grid.sync();
  } else {
    __threadfence();
    __syncthreads();
  }
}

__device__ __forceinline__ int key_bits(int64_t maxkey) {
  int b = 0;
  while (b < 63 && (maxkey >> b) != 0) ++b;
  return b;
}

// Sorts (k, v)[0, n) by the low `bits` key bits; returns which buffer pair holds the result
// (0 = k0/v0, 1 = k1/v1).  Input in k0/v0.
template <bool GRID>
__device__ int radix_sort(cg::grid_group& grid, const Params& P, int64_t n, int bits, Smem& sm) {
  int cur = 0;
  for (int shift = 0; shift < bits; shift += 8) {
    if (cur == 0)
      radix_pass<GRID>(grid, P.k0, P.v0, P.k1, P.v1, n, shift, P.dig, sm);
    else
      radix_pass<GRID>(grid, P.k1, P.v1, P.k0, P.v0, n, shift, P.dig, sm);
    cur ^= 1;
  }
  return cur;
}

// Ordered exclusive scan of tri over [c0, c1) from `carry`; writes toff and the spans.
__device__ void comp_offsets(const Params& P, int64_t c0, int64_t c1, unsigned long long carry, int64_t lo_t,
                             int64_t lo_f, int64_t span0, Smem& sm) {
  for (int64_t i0 = c0; i0 < c1; i0 += NT) {
    const int64_t i = i0 + threadIdx.x;
    const bool valid = i < c1;
    const unsigned long long x = valid ? ld_(P.tri + i) : 0ull;
    unsigned long long ex, tot;
    BlockScanU64(sm.scan.u64).ExclusiveSum(x, ex, tot);
    if (valid) {
      const unsigned long long o = carry + ex;
      P.toff[i] = o;
      int64_t* sp = P.spans + 4 * (span0 + i);
      sp[0] = lo_t + (int64_t)(o >> 32);
      sp[1] = (int64_t)(x >> 32);
      sp[2] = lo_f + (int64_t)(o & 0xffffffffull);
      sp[3] = (int64_t)(x & 0xffffffffull);
    }
    carry += tot;
    __syncthreads();
  }
}

__device__ __forceinline__ void node_keys(const Params& P, int64_t c0, int64_t c1, int64_t stride) {
  for (int64_t p = c0; p < c1; p += stride) {
    const int32_t v = ld_(P.cand + p);
    P.k0[p] = (uint32_t)ld_(P.rank_of_root + ld_(P.parent + v));
    P.v0[p] = v;
  }
}

__device__ __forceinline__ void emit_nodes(const Params& P, const uint32_t* ks, const int32_t* vs, int64_t c0,
                                           int64_t c1, int64_t stride, int64_t lo_t, int64_t lo_f) {
  for (int64_t p = c0; p < c1; p += stride) {
    const int32_t v = ld_(vs + p);
    const uint32_t c = ld_(ks + p);
    const unsigned long long o = ld_(P.toff + c);
    const int64_t rb = (int64_t)(o >> 32), cb = (int64_t)(o & 0xffffffffull);
    const int64_t pos = p - (rb + cb);
    if (v < P.m)
      P.row_fwd[v] = lo_t + rb + pos;
    else
      P.col_fwd[v - P.m] = lo_f + cb + pos - (int64_t)(ld_(P.tri + c) >> 32);
  }
}

// Union-find hooking over the live edges.  HK edges per thread in flight: the first two levels of
// every find are issued as independent loads.
template <int HK>
__device__ __forceinline__ void hook_edges(const Params& P, const uint64_t* E, int64_t ne, int64_t gtid, int64_t gsz) {
  const int32_t m = P.m;
  for (int64_t e0 = gtid; e0 < ne; e0 += (int64_t)HK * gsz) {
    int32_t u[HK], v[HK], pu[HK], pv[HK];
    bool ok[HK];
#pragma unroll
    for (int j = 0; j < HK; ++j) {
      const int64_t e = e0 + j * gsz;
      ok[j] = e < ne;
      const uint64_t ed = ok[j] ? ld_(E + e) : 0ull;
      u[j] = (int32_t)(ed >> 32);
      v[j] = (int32_t)(ed & 0xffffffffu) + m;
    }
#pragma unroll
    for (int j = 0; j < HK; ++j) ok[j] = ok[j] && ld_(P.state + u[j]) && ld_(P.state + v[j]);
#pragma unroll
    for (int j = 0; j < HK; ++j) {
      pu[j] = ok[j] ? ld_(P.parent + u[j]) : u[j];
      pv[j] = ok[j] ? ld_(P.parent + v[j]) : v[j];
    }
#pragma unroll
    for (int j = 0; j < HK; ++j) {
      if (!ok[j]) continue;
      if (P.hshort && pu[j] == pv[j]) continue;  // a common parent: already one component
      int32_t ru = find_root_from(u[j], pu[j], P.parent), rv = find_root_from(v[j], pv[j], P.parent);
      while (ru != rv) {
        if (ru < rv) {
          const int32_t old = atomicCAS(P.parent + rv, rv, ru);
          if (old == rv) break;
          rv = find_root_cg(old, P.parent);
        } else {
          const int32_t old = atomicCAS(P.parent + ru, ru, rv);
          if (old == ru) break;
          ru = find_root_cg(old, P.parent);
        }
      }
    }
  }
}

#ifndef RP_CTAS_PER_SM
#define RP_CTAS_PER_SM 1
#endif
__global__ void __launch_bounds__(NT, RP_CTAS_PER_SM) k_reorder_persistent(Params P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Smem sm;
  const int t = threadIdx.x, b = blockIdx.x, G = gridDim.x, lane = t & 31;
  const int64_t gtid = (int64_t)b * NT + t, gsz = (int64_t)G * NT;
  const int32_t m = P.m;
  Ctl* ctl = P.ctl;

  int64_t cnt_t = m, cnt_f = P.n, lo_t = 0, lo_f = 0, hi_t = (int64_t)m - 1, hi_f = (int64_t)P.n - 1;
  int64_t ne = P.ne0, nspans = 0, ngcc = 0, iters = 0;
  int32_t* act = P.act0;
  int32_t* act_nx = P.act1;
  uint64_t* E = P.e0;
  uint64_t* E_nx = P.e1;
  int hl = 0;  // hub histogram buffer rotation
  int64_t nroots_log = 0, nnodes_log = 0, maxsz_all = 0;  // spoke log (laid out after the loop)
  int64_t dprev[2] = {0, 0};                                // previous hub thresholds (0: none)
  int64_t e_sum = 0, v_sum = 0;                             // sum_t E_t, sum_t V_t
  unsigned long long tlast = (P.prof && gtid == 0) ? gtimer() : 0ull;
#define RP_PROF(i)                                     \
  if (P.prof && gtid == 0) {                           \
    const unsigned long long now_ = gtimer();          \
    P.prof[i] += now_ - tlast;                         \
    tlast = now_;                                      \
  }

  while (true) {
    ++iters;
    const int par = (int)(iters & 1);
    const int64_t q_t = (int64_t)ceil(P.k * (double)cnt_t);  // math.ceil(k * cnt), reorder.py:198-199
    const int64_t q_f = (int64_t)ceil(P.k * (double)cnt_f);
    const int64_t L = cnt_t + cnt_f;  // length of the active list this iteration
    e_sum += ne;  // edges with both endpoints active (the list is compacted to the previous GCC)
    v_sum += L;

    // ---- P1: degrees; clear this iteration's accumulators
    if (gtid == 0) {
      ctl->nhub[0] = ctl->nhub[1] = 0;
      ctl->nroots = 0;
      ctl->maxsz = 0;
      ctl->best = 0ull;
      ctl->ne_next[par] = 0;
    }
    if (iters == 1) {  // later iterations count degrees while compacting the edge list (P15)
      for (int64_t e = gtid; e < ne; e += gsz) {
        const uint64_t ed = ld_(E + e);
        agg_inc(P.deg, (int32_t)(ed >> 32));
        agg_inc(P.deg, (int32_t)(ed & 0xffffffffu) + m);
      }
      grid.sync();
    }
    RP_PROF(0)

    // ---- P2: per-side hub threshold (radix select over the degrees, highest level first)
    int64_t need[2], pre[2] = {0, 0}, htot[2], eqcnt[2] = {0, 0};
    need[0] = (cnt_t > 0 && q_t > 0) ? (q_t < cnt_t ? q_t : cnt_t) : 0;
    need[1] = (cnt_f > 0 && q_f > 0) ? (q_f < cnt_f ? q_f : cnt_f) : 0;
    htot[0] = need[0];
    htot[1] = need[1];
    // Window pass: degrees only fall from one iteration to the next and every node left active had
    // degree <= the previous threshold, so the new threshold usually lies in the 2048 degrees
    // (dprev - 2048, dprev]: one histogram level instead of P.levels.
    bool gen[2] = {need[0] > 0, need[1] > 0};
    if ((need[0] > 0 && dprev[0] > 0) || (need[1] > 0 && dprev[1] > 0)) {
      int64_t wbase[2];
      bool win[2];
      for (int sd = 0; sd < 2; ++sd) {
        win[sd] = need[sd] > 0 && dprev[sd] > 0;
        wbase[sd] = dprev[sd] - (HB - 1) > 1 ? dprev[sd] - (HB - 1) : 1;
      }
      int32_t* buf = P.hist + (hl % 3) * 2 * HB;
      int32_t* zbuf = P.hist + ((hl + 1) % 3) * 2 * HB;
      for (int64_t i = gtid; i < 2 * HB; i += gsz) zbuf[i] = 0;
      for (int i = t; i < 2 * HB; i += NT) (&sm.hist[0][0])[i] = 0;
      __syncthreads();
      for (int64_t i = gtid; i < L; i += gsz) {
        const int32_t v = ld_(act + i);
        const int side = v >= m;
        if (!win[side]) continue;
        const int64_t d = ld_(P.deg + v);
        if (d < wbase[side]) continue;
        atomicAdd(&sm.hist[side][d - wbase[side]], 1);
      }
      __syncthreads();
      for (int i = t; i < 2 * HB; i += NT) {
        const int c = (&sm.hist[0][0])[i];
        if (c) atomicAdd(buf + i, c);
      }
      grid.sync();
      ++hl;
      for (int side = 0; side < 2; ++side) {
        if (!win[side]) continue;
        int c4[4];
        unsigned long long mine = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          c4[j] = ld_(buf + side * HB + (HB - 1 - 4 * t - j));
          mine += (unsigned long long)c4[j];
        }
        unsigned long long ex, tot;
        BlockScanU64(sm.scan.u64).ExclusiveSum(mine, ex, tot);
        const int64_t nd = need[side];
        if ((int64_t)tot >= nd && (int64_t)ex < nd && nd <= (int64_t)(ex + mine)) {
          int64_t run = (int64_t)ex;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (run + c4[j] >= nd) {
              sm.bc[0] = HB - 1 - 4 * t - j;
              sm.bc[1] = run;
              sm.bc[2] = c4[j];
              break;
            }
            run += c4[j];
          }
        }
        __syncthreads();
        if ((int64_t)tot >= nd) {  // found in the window (otherwise the general select below)
          pre[side] = wbase[side] + sm.bc[0];
          need[side] = nd - sm.bc[1];
          eqcnt[side] = sm.bc[2];
          gen[side] = false;
        }
        __syncthreads();
      }
    }
    if (gen[0] || gen[1]) {
      for (int lev = P.levels - 1; lev >= 0; --lev) {
        const int shift = lev * HBITS;
        int32_t* buf = P.hist + (hl % 3) * 2 * HB;
        int32_t* zbuf = P.hist + ((hl + 1) % 3) * 2 * HB;
        for (int64_t i = gtid; i < 2 * HB; i += gsz) zbuf[i] = 0;
        for (int i = t; i < 2 * HB; i += NT) (&sm.hist[0][0])[i] = 0;
        __syncthreads();
        for (int64_t i = gtid; i < L; i += gsz) {
          const int32_t v = ld_(act + i);
          const int side = v >= m;
          if (!gen[side] || need[side] == 0) continue;
          const int32_t d = ld_(P.deg + v);
          if (d <= 0) continue;
          if (lev < P.levels - 1 && ((int64_t)d >> (shift + HBITS)) != pre[side]) continue;
          atomicAdd(&sm.hist[side][(d >> shift) & (HB - 1)], 1);
        }
        __syncthreads();
        for (int i = t; i < 2 * HB; i += NT) {
          const int c = (&sm.hist[0][0])[i];
          if (c) atomicAdd(buf + i, c);
        }
        grid.sync();
        ++hl;
        // decision, identical in every CTA: the bin holding the need-th largest degree
        for (int side = 0; side < 2; ++side) {
          if (!gen[side] || need[side] == 0) continue;
          int c4[4];
          unsigned long long mine = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            c4[j] = ld_(buf + side * HB + (HB - 1 - 4 * t - j));
            mine += (unsigned long long)c4[j];
          }
          unsigned long long ex, tot;
          BlockScanU64(sm.scan.u64).ExclusiveSum(mine, ex, tot);
          if (lev == P.levels - 1) {
            if ((int64_t)tot < need[side]) need[side] = (int64_t)tot;  // fewer positive-degree nodes than the quota
            htot[side] = need[side];
          }
          const int64_t nd = need[side];
          if (nd > 0 && (int64_t)ex < nd && nd <= (int64_t)(ex + mine)) {
            int64_t run = (int64_t)ex;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (run + c4[j] >= nd) {
                sm.bc[0] = HB - 1 - 4 * t - j;
                sm.bc[1] = run;
                sm.bc[2] = c4[j];
                break;
              }
              run += c4[j];
            }
          }
          __syncthreads();
          if (nd > 0) {
            pre[side] = (pre[side] << HBITS) | sm.bc[0];
            need[side] = nd - sm.bc[1];
            eqcnt[side] = sm.bc[2];
          }
          __syncthreads();
        }
      }
    }
    dprev[0] = htot[0] > 0 ? pre[0] : 0;
    dprev[1] = htot[1] > 0 ? pre[1] : 0;
    RP_PROF(1)
    // hubs of side s: degree > pre[s], plus the first need[s] (ascending id) of degree == pre[s]
    const bool split_ties = (htot[0] > 0 && need[0] < eqcnt[0]) || (htot[1] > 0 && need[1] < eqcnt[1]);
    if (htot[0] > 0 || htot[1] > 0) {
      if (!split_ties) {
        for (int64_t i = gtid; i < L; i += gsz) {
          const int32_t v = ld_(act + i);
          const int side = v >= m;
          if (htot[side] == 0) continue;
          const int32_t d = ld_(P.deg + v);
          if (d > 0 && (int64_t)d >= pre[side]) {
            const int pos = atomicAdd(&ctl->nhub[side], 1);
            P.hubkeys[side * HUB_CAP + pos] = ((uint64_t)(0xffffffffu - (uint32_t)d) << 32) | (uint32_t)v;
            P.state[v] = 0;  // retired now: the hooking below (same phase as the ranks) skips it
          }
        }
      } else {
        // ---- P3: per-CTA counts of tie-degree nodes (ordered chunks)
        const int64_t c0 = L * b / G, c1 = L * (b + 1) / G;
        unsigned long long e0 = 0, e1 = 0;
        for (int64_t i = c0 + t; i < c1; i += NT) {
          const int32_t v = ld_(act + i);
          const int side = v >= m;
          if (htot[side] > 0 && (int64_t)ld_(P.deg + v) == pre[side]) (side ? e1 : e0) += 1;
        }
        e0 = block_sum(e0, sm);
        e1 = block_sum(e1, sm);
        if (t == 0) {
          P.blk[4 * b + 0] = (int64_t)e0;
          P.blk[4 * b + 1] = (int64_t)e1;
        }
        grid.sync();
        // ---- P4: collect hubs; ties taken in ascending id order
        int64_t base0 = cta_prefix(P.blk, 0, b, sm), base1 = cta_prefix(P.blk, 1, b, sm);
        for (int64_t i0 = c0; i0 < c1; i0 += NT) {
          const int64_t i = i0 + t;
          int32_t v = 0, d = 0;
          int side = 0;
          bool eq = false;
          if (i < c1) {
            v = ld_(act + i);
            side = v >= m;
            d = ld_(P.deg + v);
            eq = htot[side] > 0 && (int64_t)d == pre[side];
          }
          const unsigned long long x = eq ? (side ? (1ull << 21) : 1ull) : 0ull;
          unsigned long long ex, tot;
          BlockScanU64(sm.scan.u64).ExclusiveSum(x, ex, tot);
          if (i < c1 && htot[side] > 0 && d > 0) {
            const int64_t eqrank = (side ? base1 : base0) + field21(ex, side);
            if ((int64_t)d > pre[side] || (eq && eqrank < need[side])) {
              const int pos = atomicAdd(&ctl->nhub[side], 1);
              P.hubkeys[side * HUB_CAP + pos] = ((uint64_t)(0xffffffffu - (uint32_t)d) << 32) | (uint32_t)v;
              P.state[v] = 0;
            }
          }
          base0 += field21(tot, 0);
          base1 += field21(tot, 1);
          __syncthreads();
        }
      }
      grid.sync();
      RP_PROF(2)
      // ---- P5: hub ranks (degree desc, id asc) and ids from the top
      const int64_t H = htot[0] + htot[1];
      for (int64_t gw = gtid >> 5; gw < H; gw += gsz >> 5) {
        const int side = gw >= htot[0];
        const int64_t i = side ? gw - htot[0] : gw;
        const uint64_t* lst = P.hubkeys + side * HUB_CAP;
        const uint64_t key = ld_(lst + i);
        int r = 0;
        for (int64_t j = lane; j < htot[side]; j += 32) r += ld_(lst + j) < key;
        for (int o = 16; o; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        if (lane == 0) {
          const int32_t v = (int32_t)(key & 0xffffffffull);
          if (side)
            P.col_fwd[v - m] = hi_f - r;
          else
            P.row_fwd[v] = hi_t - r;
        }
      }
      // (no barrier: the ranks only write the permutations, the hooking below reads states that
      // were final at the collection barrier)
      RP_PROF(3)
      hi_t -= htot[0];
      hi_f -= htot[1];
      cnt_t -= htot[0];
      cnt_f -= htot[1];
    }

    // ---- P6: connected components of the residual (lock-free union-find, min-id roots)
    if (P.hk == 4)
      hook_edges<4>(P, E, ne, gtid, gsz);
    else if (P.hk == 2)
      hook_edges<2>(P, E, ne, gtid, gsz);
    else
      hook_edges<1>(P, E, ne, gtid, gsz);
    grid.sync();
    if (P.prof && gtid == 0 && iters <= 5) P.prof[10 + iters] = gtimer() - tlast;
    RP_PROF(4)
    // ---- P7: labels, sizes, row counts, and the giant component (max size, then min id,
    // reorder.py:228-234) with the component count -- in one pass: a root's final size is the value
    // its last (aggregated) size increment produces, so the max over every increment's result is
    // the max over the final sizes
    {
      unsigned long long best = 0, nr = 0;
      for (int64_t i = gtid; i < L; i += gsz) {
        const int32_t v = ld_(act + i);
        if (!ld_(P.state + v)) continue;
        int32_t r = v, p;
        while ((p = ld_(P.parent + r)) != r) r = p;
        P.parent[v] = r;
        P.deg[v] = 0;  // this iteration's degrees are spent; the compaction below counts the next ones
        const unsigned peers = __match_any_sync(__activemask(), r);
        if (lane == __ffs(peers) - 1) {
          const unsigned nsz = (unsigned)atomicAdd(P.csize + r, __popc(peers)) + (unsigned)__popc(peers);
          const unsigned long long key = ((unsigned long long)nsz << 32) | (uint32_t)(0x7fffffff - r);
          best = key > best ? key : best;
        }
        if (v < m) agg_inc(P.crows, r);
        nr += r == v;
      }
      best = block_max(best, sm);
      nr = block_sum(nr, sm);
      if (t == 0) {
        if (best) atomicMax(&ctl->best, best);
        if (nr) atomicAdd(&ctl->nroots, (int)nr);
      }
    }
    grid.sync();
    RP_PROF(5)
    const int64_t acnt = cnt_t + cnt_f;
    if (acnt == 0) {  // reorder.py:224-226
      if (gtid == 0) P.gcc_sizes[ngcc] = 0;
      ++ngcc;
      break;
    }
    const unsigned long long best = __ldcg(&ctl->best);
    const int32_t gcc = (int32_t)(0x7fffffff - (int64_t)(best & 0xffffffffull));
    const int64_t gsize = (int64_t)(best >> 32);
    const int64_t g_t = ld_(P.crows + gcc), g_f = gsize - g_t;
    const int64_t nsc = (int64_t)__ldcg(&ctl->nroots) - 1;
    const int64_t nsp = acnt - gsize;

    // ---- P9: three-way partition counts (giant | spoke roots | other spokes), ordered chunks
    const int64_t c0 = L * b / G, c1 = L * (b + 1) / G;
    {
      unsigned long long n0 = 0, n1 = 0, n2 = 0, mx = 0;
      for (int64_t i = c0 + t; i < c1; i += NT) {
        const int32_t v = ld_(act + i);
        if (!ld_(P.state + v)) continue;
        const int32_t p = ld_(P.parent + v);
        if (p == gcc) {
          ++n0;
        } else if (p == v) {
          ++n1;
          const unsigned long long sz = (unsigned long long)ld_(P.csize + v);
          mx = sz > mx ? sz : mx;
        } else {
          ++n2;
        }
      }
      n0 = block_sum(n0, sm);
      n1 = block_sum(n1, sm);
      n2 = block_sum(n2, sm);
      mx = block_max(mx, sm);
      if (t == 0) {
        P.blk[4 * b + 0] = (int64_t)n0;
        P.blk[4 * b + 1] = (int64_t)n1;
        P.blk[4 * b + 2] = (int64_t)n2;
        if (mx) atomicMax(&ctl->maxsz, (int)mx);
      }
    }
    // ---- P15: compact the edge list to the new giant component (unordered), counting the next
    // iteration's degrees on the way (reorder.py:201-202).  Runs in the same phase as the partition
    // counts: an edge stays iff both endpoints' labels are the giant root (hubs retired this
    // iteration keep parent == self, spoke nodes carry their own roots), read before P10 resets them.
    for (int64_t e0 = gtid - lane; e0 < ne; e0 += gsz) {
      const int64_t e = e0 + lane;
      bool keep = false;
      uint64_t ed = 0;
      if (e < ne) {
        ed = ld_(E + e);
        keep = ld_(P.parent + (int32_t)(ed >> 32)) == gcc && ld_(P.parent + (int32_t)(ed & 0xffffffffu) + m) == gcc;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      int base = 0;
      if (lane == 0 && bal) base = atomicAdd(&ctl->ne_next[par], __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        E_nx[base + __popc(bal & lanemask_lt())] = ed;
        agg_inc(P.deg, (int32_t)(ed >> 32));
        agg_inc(P.deg, (int32_t)(ed & 0xffffffffu) + m);
      }
    }
    grid.sync();
    RP_PROF(7)
    // ---- P10: partition write; giant members reset for the next iteration, spokes retired
    const int64_t maxsz = __ldcg(&ctl->maxsz);
    {
      int64_t b0 = cta_prefix(P.blk, 0, b, sm);
      int64_t b1 = cta_prefix(P.blk, 1, b, sm);
      int64_t b2 = nsc + cta_prefix(P.blk, 2, b, sm);
      for (int64_t i0 = c0; i0 < c1; i0 += NT) {
        const int64_t i = i0 + t;
        int cls = -1;
        int32_t v = 0;
        if (i < c1) {
          v = ld_(act + i);
          if (ld_(P.state + v)) {
            const int32_t p = ld_(P.parent + v);
            cls = p == gcc ? 0 : (p == v ? 1 : 2);
          }
        }
        const unsigned long long x = cls < 0 ? 0ull : (1ull << (21 * cls));
        unsigned long long ex, tot;
        BlockScanU64(sm.scan.u64).ExclusiveSum(x, ex, tot);
        if (cls == 0) {
          act_nx[b0 + field21(ex, 0)] = v;
          P.parent[v] = v;
          P.csize[v] = 0;
          P.crows[v] = 0;
        } else if (cls == 1) {
          // spoke roots and spoke nodes are logged; their blocks and ids are laid out once, after
          // the loop (a spoke's parent / size / row count are never touched again)
          const int64_t p = b1 + field21(ex, 1);
          P.rlog[nroots_log + p] = v;
          P.riter[nroots_log + p] = (int32_t)iters;
          P.cand[nnodes_log + p] = v;
          P.state[v] = 0;
        } else if (cls == 2) {
          P.cand[nnodes_log + b2 + field21(ex, 2)] = v;
          P.state[v] = 0;
        }
        b0 += field21(tot, 0);
        b1 += field21(tot, 1);
        b2 += field21(tot, 2);
        __syncthreads();
      }
    }
    grid.sync();
    RP_PROF(8)
    ne = __ldcg(&ctl->ne_next[par]);
    {
      uint64_t* tmp = E;
      E = E_nx;
      E_nx = tmp;
    }

    const bool stop = g_t < q_t || g_f < q_f;  // reorder.py:268-269
    maxsz_all = maxsz > maxsz_all ? maxsz : maxsz_all;
    nroots_log += nsc;
    nnodes_log += nsp;
    if (gtid == 0) P.gcc_sizes[ngcc] = gsize;
    ++ngcc;
    nspans += nsc;
    lo_t += cnt_t - g_t;
    lo_f += cnt_f - g_f;
    cnt_t = g_t;
    cnt_f = g_f;
    {
      int32_t* tmp = act;
      act = act_nx;
      act_nx = tmp;
    }
    if (stop) break;

  }
  // ---- spoke blocks of all iterations at once (reorder.py:236-257): components ordered by
  // (iteration, size desc, min id asc) -- two stable LSD sorts of the root log (size key, then
  // iteration key) -- and the global exclusive scan of their (rows, cols) IS lo_t / lo_f of their
  // iteration plus the offset inside it; then the logged spoke nodes are stably grouped by their
  // component's rank (roots first within an iteration's log, so members stay ascending).
  RP_PROF(9)
  if (nroots_log > 0) {
    const int64_t R = nroots_log, Nn = nnodes_log;
    for (int64_t i = gtid; i < R; i += gsz) {
      P.k0[i] = (uint32_t)(maxsz_all - ld_(P.csize + ld_(P.rlog + i)));
      P.v0[i] = (int32_t)i;
    }
    grid.sync();
    int cur = radix_sort<true>(grid, P, R, maxsz_all > 1 ? key_bits(maxsz_all - 1) : 0, sm);
    {
      const int32_t* vs = cur ? P.v1 : P.v0;
      for (int64_t i = gtid; i < R; i += gsz) {
        const int32_t li = ld_(vs + i);
        P.k0[i] = (uint32_t)ld_(P.riter + li);
        P.v0[i] = li;
      }
    }
    grid.sync();
    cur = radix_sort<true>(grid, P, R, key_bits(iters), sm);
    const int32_t* order = cur ? P.v1 : P.v0;  // log indices in rank order
    {
      const int64_t r0 = R * b / G, r1 = R * (b + 1) / G;
      unsigned long long sacc = 0;
      for (int64_t i = r0 + t; i < r1; i += NT) {
        const int32_t r = ld_(P.rlog + ld_(order + i));
        P.rank_of_root[r] = (int32_t)i;
        const uint64_t rows = (uint64_t)ld_(P.crows + r);
        const uint64_t cols = (uint64_t)ld_(P.csize + r) - rows;
        const uint64_t tr = (rows << 32) | cols;
        P.tri[i] = tr;
        sacc += tr;
      }
      sacc = block_sum(sacc, sm);
      if (t == 0) P.blk[4 * b + 3] = (int64_t)sacc;
      grid.sync();
      unsigned long long carry = 0;
      for (int c = t; c < b; c += NT) carry += (unsigned long long)ld_(P.blk + 4 * c + 3);
      carry = block_sum(carry, sm);
      comp_offsets(P, r0, r1, carry, 0, 0, 0, sm);  // the global scan already includes lo_t / lo_f
    }
    node_keys(P, gtid, Nn, gsz);
    grid.sync();
    const int cur2 = radix_sort<true>(grid, P, Nn, R > 1 ? key_bits(R - 1) : 0, sm);
    emit_nodes(P, cur2 ? P.k1 : P.k0, cur2 ? P.v1 : P.v0, gtid, Nn, gsz, 0, 0);
    nspans = R;
  }
  if (P.prof && gtid == 0) P.prof[10] += gtimer() - tlast;
  // terminal giant component: the middle ids, ascending (reorder.py:271-275)
  const int64_t rem = cnt_t + cnt_f;
  for (int64_t i = gtid; i < rem; i += gsz) {
    const int32_t v = ld_(act + i);
    if (i < cnt_t)
      P.row_fwd[v] = lo_t + i;
    else
      P.col_fwd[v - m] = lo_f + (i - cnt_t);
  }
  if (gtid == 0) {
    ctl->out[0] = lo_t;
    ctl->out[1] = lo_f;
    ctl->out[2] = iters;
    ctl->out[3] = nspans;
    ctl->out[4] = ngcc;
    ctl->out[5] = e_sum;
    ctl->out[6] = v_sum;
  }
}

__global__ void k_rp_expand_edges(int64_t m, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                  uint64_t* __restrict__ edges) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < m; r += nwarps) {
    const int64_t b0 = indptr[r], e = indptr[r + 1];
    for (int64_t p = b0 + lane; p < e; p += 32) edges[p] = ((uint64_t)r << 32) | (uint32_t)indices[p];
  }
}

__global__ void k_rp_init_nodes(int64_t V, uint8_t* __restrict__ state, int32_t* __restrict__ deg,
                                int32_t* __restrict__ parent, int32_t* __restrict__ csize, int32_t* __restrict__ crows,
                                int32_t* __restrict__ act) {
  FPI_GRID_STRIDE(i, V) {
    state[i] = 1;
    deg[i] = 0;
    parent[i] = (int32_t)i;
    csize[i] = 0;
    crows[i] = 0;
    act[i] = (int32_t)i;
  }
}

}  // namespace

bool run_reorder_persistent(fpi_context* h, int64_t m, int64_t n, int64_t nnz, const int64_t* d_indptr,
                            const int32_t* d_indices, double k, int64_t* d_row_fwd, int64_t* d_col_fwd,
                            ReorderOut& out) {
  FPI_REQUIRE(k > 0.0 && k < 1.0, FPI_EDOMAIN, "hub selection ratio k must be in (0, 1)");
  FPI_REQUIRE(m > 0 && n > 0, FPI_EDOMAIN, "graph has an empty node side");
  FPI_REQUIRE(m + n < (int64_t)INT32_MAX, FPI_ECAPACITY, "m + n exceeds the int32 node-id range");
  FPI_REQUIRE(nnz < (int64_t)INT32_MAX, FPI_ECAPACITY, "nnz exceeds the int32 edge-count range");
  const int64_t V = m + n;
  // static limits of the kernel: hub lists (the quota only shrinks after iteration 1)
  if ((int64_t)std::ceil(k * (double)m) > HUB_CAP || (int64_t)std::ceil(k * (double)n) > HUB_CAP) return false;
  int occ = 0;
  FPI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_reorder_persistent, NT, 0));
  if (occ < 1) return false;
  const int G = h->num_sms * (occ > RP_CTAS_PER_SM ? RP_CTAS_PER_SM : occ);
  if (V / G >= (1 << 20)) return false;  // per-tile counters are packed in 21-bit fields (tile <= NT anyway)

  cudaStream_t s = h->stream;
  if (h->spans_cap < V) {
    if (h->d_spans) cudaFree(h->d_spans);
    FPI_CUDA(cudaMalloc((void**)&h->d_spans, sizeof(int64_t) * 4 * (V + 1)));
    h->spans_cap = V;
  }
  h->n_spans = 0;
  h->gcc_sizes.clear();

  Scratch<uint64_t> e0(nnz > 0 ? nnz : 1, s), e1(nnz > 0 ? nnz : 1, s);
  Scratch<uint8_t> state(V, s);
  Scratch<int32_t> deg(V, s), parent(V, s), csize(V, s), crows(V, s), act0(V, s), act1(V, s), cand(V, s),
      rank_of_root(V, s), v0(V, s), v1(V, s), rlog(V, s), riter(V, s);
  Scratch<uint32_t> k0(V, s), k1(V, s);
  Scratch<uint64_t> tri(V, s), toff(V, s), hubkeys(2 * HUB_CAP, s);
  Scratch<int64_t> gcc(V + 2, s), blk(4 * G, s);
  Scratch<int32_t> hist(3 * 2 * HB, s), dig(256 * G + 256, s);
  Scratch<Ctl> ctl(1, s);
  FPI_CUDA(cudaMemsetAsync(hist.get(), 0, sizeof(int32_t) * 3 * 2 * HB, s));
  FPI_CUDA(cudaMemsetAsync(ctl.get(), 0, sizeof(Ctl), s));
  if (nnz) k_rp_expand_edges<<<h->num_sms * 8, 256, 0, s>>>(m, d_indptr, d_indices, e0);
  k_rp_init_nodes<<<grid_for(V, 256, h->num_sms * 8), 256, 0, s>>>(V, state, deg, parent, csize, crows, act0);
  FPI_LAUNCH_CHECK();

  Params P;
  P.m = (int32_t)m;
  P.n = (int32_t)n;
  P.k = k;
  P.levels = (bits_for((uint64_t)(m > n ? m : n)) + HBITS - 1) / HBITS;
  P.ne0 = (int)nnz;
  {
    const char* e = getenv("FPI_REORDER_HK");
    P.hk = e ? atoi(e) : 1;
    const char* e2 = getenv("FPI_REORDER_SHORT");
    P.hshort = e2 ? atoi(e2) : 1;
  }
  P.e0 = e0;
  P.e1 = e1;
  P.state = state;
  P.deg = deg;
  P.parent = parent;
  P.csize = csize;
  P.crows = crows;
  P.act0 = act0;
  P.act1 = act1;
  P.cand = cand;
  P.k0 = k0;
  P.k1 = k1;
  P.v0 = v0;
  P.v1 = v1;
  P.rank_of_root = rank_of_root;
  P.rlog = rlog;
  P.riter = riter;
  P.tri = tri;
  P.toff = toff;
  P.row_fwd = d_row_fwd;
  P.col_fwd = d_col_fwd;
  P.spans = h->d_spans;
  P.gcc_sizes = gcc;
  P.hist = hist;
  P.dig = dig;
  P.blk = blk;
  P.hubkeys = hubkeys;
  P.ctl = ctl;
  const bool prof_on = getenv("FPI_REORDER_PROFILE") != nullptr;
  Scratch<unsigned long long> prof(prof_on ? 16 : 1, s);
  P.prof = prof_on ? prof.get() : nullptr;
  if (prof_on) FPI_CUDA(cudaMemsetAsync(prof.get(), 0, sizeof(unsigned long long) * 16, s));
  void* args[] = {&P};
  FPI_CUDA(cudaLaunchCooperativeKernel((void*)k_reorder_persistent, dim3(G), dim3(NT), args, 0, s));
  FPI_LAUNCH_CHECK();
  note_launch(h, 3);

  const Ctl c = host_read(ctl.get(), s);
  const int64_t lo_t = c.out[0], lo_f = c.out[1];
  h->n_spans = c.out[3];
  h->gcc_sizes.resize((size_t)c.out[4]);
  if (c.out[4])
    FPI_CUDA(cudaMemcpyAsync(h->gcc_sizes.data(), gcc.get(), sizeof(int64_t) * c.out[4], cudaMemcpyDeviceToHost, s));
  FPI_CUDA(cudaStreamSynchronize(s));
  if (prof_on) {
    unsigned long long hp[16];
    FPI_CUDA(cudaMemcpy(hp, prof.get(), sizeof(hp), cudaMemcpyDeviceToHost));
    static const char* names[] = {"degree", "hub-select", "hub-collect", "hub-rank", "hook", "label", "pick",
                                  "part-count", "part-write", "compact"};
    fprintf(stderr, "[reorder persistent G=%d T=%lld]", G, (long long)c.out[2]);
    for (int i = 0; i < 10; ++i) fprintf(stderr, " %s %.3f", names[i], hp[i] * 1e-6);
    fprintf(stderr, " | spoke layout (after the loop) %.3f | hook it1-5: %.3f %.3f %.3f %.3f %.3f", hp[10] * 1e-6,
            hp[11] * 1e-6, hp[12] * 1e-6, hp[13] * 1e-6, hp[14] * 1e-6, hp[15] * 1e-6);
    fprintf(stderr, " ms\n");
  }
  out.m1 = lo_t;
  out.n1 = lo_f;
  out.m2 = m - lo_t;
  out.n2 = n - lo_f;
  out.T = c.out[2];
  out.e_sum = c.out[5];
  out.v_sum = c.out[6];
  return true;
}

}  // namespace fpi
