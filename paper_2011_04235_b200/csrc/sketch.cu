// Bit-exact numpy Gaussian sketch on the GPU:
//   X = np.random.default_rng(seed).standard_normal((rows, cols))  (svd.py:131-132)
//
// numpy draws from PCG64 (128-bit LCG, XSL-RR output) through a 256-layer
// ziggurat.  Every sample consumes one 64-bit draw in ~98.5% of cases and a
// variable number otherwise (wedge / tail rejections), so sample i does not
// sit at a fixed stream offset.  The kernel splits the raw-draw stream into
// chunks of CH draws:
//   pass 1  each chunk (one thread, LCG jump-ahead to its first draw) lists
//           its irregular positions (consumed > 1 draw) and, for each of the
//           E possible entry offsets, the number of samples that start inside
//           the chunk and the exit offset into the next chunk;
//   pass 2  those E-entry transfer maps are composed chunk by chunk
//           (per-block then across blocks) from entry 0 of chunk 0 to get
//           every chunk's true entry offset and first sample index;
//   pass 3  each chunk regenerates its draws and writes its samples.
// Regular samples need one draw; irregular ones replay numpy's sampler on a
// cloned generator.  The tail branch uses log1p_ieee (glibc-exact).
#include "common.cuh"
#include "capi_guard.cuh"
#include "log1p_ieee.cuh"
#include "generated/ziggurat_tables.h"
#include "instrument.cuh"

namespace fpi {
namespace {

typedef unsigned __int128 u128;

constexpr int CH = 256;       // raw draws per chunk
constexpr int E = 32;         // entry offsets tracked per chunk (max draws per sample)
constexpr int MAXIRR = 48;    // irregular positions recorded per chunk
constexpr int CPB = 128;      // chunks per block in the composition pass
constexpr double ZIG_R = 3.6541528853610088;        // ziggurat_nor_r
constexpr double ZIG_INV_R = 0.27366123732975828;   // ziggurat_nor_inv_r

__host__ __device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

struct Pcg {
  u128 state, inc;
  __device__ __forceinline__ uint64_t next() {
    state = state * pcg_mult() + inc;
    uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    unsigned rot = (unsigned)(state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
};

// state advanced by delta steps of x -> a x + c (O(log delta) square-and-multiply)
__host__ __device__ __forceinline__ u128 lcg_advance(u128 state, uint64_t delta, u128 mult, u128 plus) {
  u128 acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1) {
      acc_mult *= mult;
      acc_plus = acc_plus * mult + plus;
    }
    plus = (mult + 1) * plus;
    mult *= mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

struct ZigTables {
  uint64_t ki[256];
  double wi[256];
  double fi[256];
};
__constant__ ZigTables c_zig;

__device__ __forceinline__ double next_double(Pcg& g) {
  return (double)(g.next() >> 11) * (1.0 / 9007199254740992.0);
}

// One numpy random_standard_normal call whose first draw is r0 (already
// consumed); g continues the stream.  Returns the sample; *used counts draws.
__device__ double normal_slow(uint64_t r0, Pcg g, const ZigTables& z, int* used) {
  int n = 1;
  uint64_t r = r0;
  for (;;) {
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn((double)rabs, z.wi[idx]);
    if (sign) x = -x;
    if (rabs < z.ki[idx]) {
      *used = n;
      return x;
    }
    if (idx == 0) {
      for (;;) {
        double u1 = next_double(g);
        double u2 = next_double(g);
        n += 2;
        double xx = __dmul_rn(-ZIG_INV_R, log1p_ieee(-u1));
        double yy = -log1p_ieee(-u2);
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          *used = n;
          return ((rabs >> 8) & 1) ? -__dadd_rn(ZIG_R, xx) : __dadd_rn(ZIG_R, xx);
        }
      }
    } else {
      double u = next_double(g);
      n += 1;
      double lhs = __dadd_rn(__dmul_rn(__dsub_rn(z.fi[idx - 1], z.fi[idx]), u), z.fi[idx]);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
        *used = n;
        return x;
      }
    }
    r = g.next();
    n += 1;
  }
}

__device__ __forceinline__ bool fast_normal(uint64_t r, const ZigTables& z, double* out) {
  int idx = (int)(r & 0xff);
  r >>= 8;
  uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
  if (rabs >= z.ki[idx]) return false;
  double x = __dmul_rn((double)rabs, z.wi[idx]);
  *out = (r & 1) ? -x : x;
  return true;
}

__device__ __forceinline__ Pcg chunk_start(u128 st0, u128 inc, int64_t chunk) {
  Pcg g;
  g.inc = inc;
  g.state = lcg_advance(st0, (uint64_t)chunk * CH, pcg_mult(), inc);
  return g;
}

// pass 1: per chunk, E-entry transfer maps (count << 8 | exit).
__global__ void k_chunk_maps(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t nchunks,
                             uint32_t* __restrict__ maps, int* __restrict__ overflow) {
  __shared__ ZigTables z;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    z.ki[i] = c_zig.ki[i];
    z.wi[i] = c_zig.wi[i];
    z.fi[i] = c_zig.fi[i];
  }
  __syncthreads();
  const u128 st0 = ((u128)st_hi << 64) | st_lo, inc = ((u128)inc_hi << 64) | inc_lo;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
    Pcg g = chunk_start(st0, inc, c);
    int irr_pos[MAXIRR];
    int irr_len[MAXIRR];
    int nirr = 0;
    for (int p = 0; p < CH; ++p) {
      uint64_t r = g.next();
      double v;
      if (!fast_normal(r, z, &v)) {
        int used;
        normal_slow(r, g, z, &used);
        if (nirr < MAXIRR && used <= E) {
          irr_pos[nirr] = p;
          irr_len[nirr] = used;
          ++nirr;
        } else {
          atomicExch(overflow, 1);
        }
      }
    }
    for (int e = 0; e < E; ++e) {
      int pos = e, cnt = 0;
      for (int j = 0; j < nirr; ++j) {
        int ip = irr_pos[j];
        if (ip < pos) continue;
        if (ip >= CH) break;
        cnt += ip - pos + 1;
        pos = ip + irr_len[j];
      }
      int exitv = 0;
      if (pos < CH) {
        cnt += CH - pos;
      } else {
        exitv = pos - CH;
      }
      if (pos > CH + E - 1 || exitv >= E) atomicExch(overflow, 1);
      maps[c * E + e] = ((uint32_t)cnt << 8) | (uint32_t)exitv;
    }
  }
}

// The composition passes below are pointer chases (entry -> exit offset, chunk after chunk).  One
// warp per chain with lane = entry offset: the E = 32 maps of the next WB chunks / blocks are loaded
// as independent coalesced loads, then the chain advances through them by shuffles.
constexpr int WB = 32;

// pass 2a: per block of CPB chunks, the composed map for each entry offset (warp per block).
__global__ void k_block_maps(const uint32_t* __restrict__ maps, int64_t nchunks, int64_t nblocks,
                             uint64_t* __restrict__ bmaps) {
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= nblocks) return;
  const int64_t c0 = b * CPB, c1 = c0 + CPB < nchunks ? c0 + CPB : nchunks;
  uint64_t cnt = 0;
  int cur = lane;  // this lane follows entry offset `lane`
  for (int64_t cb = c0; cb < c1; cb += WB) {
    uint32_t mm[WB];
#pragma unroll
    for (int j = 0; j < WB; ++j) mm[j] = cb + j < c1 ? maps[(cb + j) * E + lane] : 0u;
#pragma unroll
    for (int j = 0; j < WB; ++j) {
      if (cb + j >= c1) break;
      const uint32_t m = __shfl_sync(0xffffffffu, mm[j], cur);
      cnt += m >> 8;
      cur = (int)(m & 0xff);
    }
  }
  bmaps[b * E + lane] = (cnt << 8) | (uint64_t)cur;
}

// pass 2b: one warp walks the blocks from entry 0.
__global__ void k_walk_blocks(const uint64_t* __restrict__ bmaps, int64_t nblocks, int32_t* __restrict__ bentry,
                              int64_t* __restrict__ bbase, int64_t* __restrict__ total) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int cur = 0;
  int64_t acc = 0;
  for (int64_t bb = 0; bb < nblocks; bb += WB) {
    uint64_t mm[WB];
#pragma unroll
    for (int j = 0; j < WB; ++j) mm[j] = bb + j < nblocks ? bmaps[(bb + j) * E + lane] : 0ull;
#pragma unroll
    for (int j = 0; j < WB; ++j) {
      if (bb + j >= nblocks) break;
      if (lane == 0) {
        bentry[bb + j] = cur;
        bbase[bb + j] = acc;
      }
      const uint64_t m = __shfl_sync(0xffffffffu, mm[j], cur);
      acc += (int64_t)(m >> 8);
      cur = (int)(m & 0xff);
    }
  }
  if (lane == 0) *total = acc;
}

// pass 2c: per block (one warp), walk its chunks from the block entry.
__global__ void k_walk_chunks(const uint32_t* __restrict__ maps, int64_t nchunks, int64_t nblocks,
                              const int32_t* __restrict__ bentry, const int64_t* __restrict__ bbase,
                              uint8_t* __restrict__ centry, int64_t* __restrict__ cbase) {
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= nblocks) return;
  int cur = bentry[b];
  int64_t acc = bbase[b];
  const int64_t c0 = b * CPB, c1 = c0 + CPB < nchunks ? c0 + CPB : nchunks;
  for (int64_t cb = c0; cb < c1; cb += WB) {
    uint32_t mm[WB];
#pragma unroll
    for (int j = 0; j < WB; ++j) mm[j] = cb + j < c1 ? maps[(cb + j) * E + lane] : 0u;
#pragma unroll
    for (int j = 0; j < WB; ++j) {
      if (cb + j >= c1) break;
      if (lane == j) {
        centry[cb + j] = (uint8_t)cur;
        cbase[cb + j] = acc;
      }
      const uint32_t m = __shfl_sync(0xffffffffu, mm[j], cur);
      acc += m >> 8;
      cur = (int)(m & 0xff);
    }
  }
}

// pass 3: emit samples.
__global__ void k_emit(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t nchunks,
                       const uint8_t* __restrict__ centry, const int64_t* __restrict__ cbase, int64_t nsamples,
                       int64_t cols, int64_t ld, double* __restrict__ out) {
  __shared__ ZigTables z;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    z.ki[i] = c_zig.ki[i];
    z.wi[i] = c_zig.wi[i];
    z.fi[i] = c_zig.fi[i];
  }
  __syncthreads();
  const u128 st0 = ((u128)st_hi << 64) | st_lo, inc = ((u128)inc_hi << 64) | inc_lo;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx = cbase[c];
    if (idx >= nsamples) continue;
    Pcg g = chunk_start(st0, inc, c);
    int entry = centry[c];
    for (int p = 0; p < entry; ++p) g.next();
    int pos = entry;
    int64_t row = idx / cols, col = idx - row * cols;
    while (pos < CH && idx < nsamples) {
      uint64_t r = g.next();
      double v;
      int used = 1;
      if (!fast_normal(r, z, &v)) {
        v = normal_slow(r, g, z, &used);
        for (int j = 1; j < used; ++j) g.next();
      }
      out[row * ld + col] = v;
      ++idx;
      if (++col == cols) {
        col = 0;
        ++row;
      }
      pos += used;
    }
  }
}

bool g_tables_loaded = false;

void load_tables() {
  if (g_tables_loaded) return;
  ZigTables t;
  for (int i = 0; i < 256; ++i) {
    t.ki[i] = zig::KI[i];
    memcpy(&t.wi[i], &zig::WI_BITS[i], 8);
    memcpy(&t.fi[i], &zig::FI_BITS[i], 8);
  }
  FPI_CUDA(cudaMemcpyToSymbol(c_zig, &t, sizeof(t)));
  g_tables_loaded = true;
}

}  // namespace

// ---- numpy SeedSequence(seed) -> PCG64 initial state (host) --------------
namespace seedseq {
const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
const uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;
const int XSHIFT = 16, POOL = 4;

inline uint32_t hashmix(uint32_t value, uint32_t& hc) {
  value ^= hc;
  hc *= MULT_A;
  value *= hc;
  value ^= value >> XSHIFT;
  return value;
}
inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
  r ^= r >> XSHIFT;
  return r;
}

// returns state_hi, state_lo, inc_hi, inc_lo after PCG64 seeding
void pcg64_state(uint64_t seed, uint64_t out[4]) {
  std::vector<uint32_t> ent;
  if (seed == 0) ent.push_back(0);
  while (seed) {
    ent.push_back((uint32_t)(seed & 0xffffffffu));
    seed >>= 32;
  }
  uint32_t pool[POOL];
  uint32_t hc = INIT_A;
  for (int i = 0; i < POOL; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u, hc);
  for (int s = 0; s < POOL; ++s)
    for (int d = 0; d < POOL; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
  for (size_t s = POOL; s < ent.size(); ++s)
    for (int d = 0; d < POOL; ++d) pool[d] = mix(pool[d], hashmix(ent[s], hc));
  // generate_state(4, uint64): 8 uint32 words, little-endian pairs
  uint32_t w[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % POOL];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> XSHIFT;
    w[i] = v;
  }
  uint64_t val[4];
  for (int i = 0; i < 4; ++i) val[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  // pcg64_set_seed: initstate = (val0 << 64) | val1, initseq = (val2 << 64) | val3
  u128 initstate = ((u128)val[0] << 64) | val[1];
  u128 initseq = ((u128)val[2] << 64) | val[3];
  u128 inc = (initseq << 1) | 1;
  u128 st = 0;
  st = st * pcg_mult() + inc;
  st += initstate;
  st = st * pcg_mult() + inc;
  out[0] = (uint64_t)(st >> 64);
  out[1] = (uint64_t)st;
  out[2] = (uint64_t)(inc >> 64);
  out[3] = (uint64_t)inc;
}
}  // namespace seedseq

void sketch_normal(fpi_context* h, int64_t seed, int64_t rows, int64_t cols, double* d_out, int64_t ld) {
  FPI_REQUIRE(seed >= 0, FPI_EDOMAIN, "seed must be non-negative");
  FPI_REQUIRE(rows >= 0 && cols >= 0 && ld >= cols, FPI_EDOMAIN, "bad sketch shape");
  const int64_t N = rows * cols;
  if (N == 0) return;
  load_tables();
  cudaStream_t s = h->stream;
  uint64_t st[4];
  seedseq::pcg64_state((uint64_t)seed, st);
  // raw draws needed ~ 1.0167 N; over-provision and extend if short
  int64_t nchunks = (int64_t)((double)N * 1.03 / CH) + 64;
  for (int attempt = 0; attempt < 4; ++attempt) {
    const int64_t nblocks = (nchunks + CPB - 1) / CPB;
    Scratch<uint32_t> maps(nchunks * E, s);
    Scratch<uint64_t> bmaps(nblocks * E, s);
    Scratch<int32_t> bentry(nblocks, s);
    Scratch<int64_t> bbase(nblocks + 1, s), total(1, s);
    Scratch<uint8_t> centry(nchunks, s);
    Scratch<int64_t> cbase(nchunks, s);
    Scratch<int> overflow(1, s);
    FPI_CUDA(cudaMemsetAsync(overflow.get(), 0, sizeof(int), s));
    const int T = 128;
    unsigned g1 = grid_for(nchunks, T, (int64_t)h->num_sms * 64);
    k_chunk_maps<<<g1, T, 0, s>>>(st[0], st[1], st[2], st[3], nchunks, maps, overflow);
    k_block_maps<<<grid_for(nblocks * 32, 256, 1 << 30), 256, 0, s>>>(maps, nchunks, nblocks, bmaps);
    k_walk_blocks<<<1, 32, 0, s>>>(bmaps, nblocks, bentry, bbase, total);
    k_walk_chunks<<<grid_for(nblocks * 32, 256, 1 << 30), 256, 0, s>>>(maps, nchunks, nblocks, bentry, bbase, centry,
                                                                       cbase);
    FPI_LAUNCH_CHECK();
    note_launch(h, 4);
    int64_t have = host_read(total.get(), s);
    int ovf = host_read(overflow.get(), s);
    FPI_REQUIRE(!ovf, FPI_ENUMERIC, "sketch: a ziggurat rejection chain exceeded the per-chunk window");
    if (have < N) {
      nchunks = (int64_t)((double)nchunks * 1.25) + 64;
      continue;
    }
    KTimer kt(h, "sketch_pcg64_ziggurat_emit", 0.0, 8.0 * (double)N);
    k_emit<<<g1, T, 0, s>>>(st[0], st[1], st[2], st[3], nchunks, centry, cbase, N, cols, ld, d_out);
    FPI_LAUNCH_CHECK();
    note_launch(h, 1);
    return;
  }
  throw Error(FPI_ENUMERIC, "sketch: could not provision enough raw draws");
}

}  // namespace fpi

extern "C" int fpi_sketch_normal(fpi_handle h, int64_t seed, int64_t rows, int64_t cols, double* d_out, int64_t ld) {
  FPI_API_BEGIN(h)
  fpi::sketch_normal(h, seed, rows, cols, d_out, ld);
  FPI_API_END(h)
}

extern "C" int fpi_pcg64_seed(int64_t seed, uint64_t* out) {
  if (!out || seed < 0) return FPI_EDOMAIN;
  fpi::seedseq::pcg64_state((uint64_t)seed, out);
  return FPI_OK;
}
