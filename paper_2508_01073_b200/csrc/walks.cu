// Walk-corpus kernels: uniform random walks (one walker per lane), the
// fixed-width -> flat compaction, duplicate-free filtering per root group,
// entity/property projections, token histogram and min_count filtering.
//
// Reference (pkg/src/walkvec/walks.py):
//   random_walks      :144-204  work list = repeat(roots, walk_number) (:166),
//                               8192-item shards, one numpy stream per shard
//                               seeded SeedSequence([seed, 0, shard]) (:168-173)
//   _walk_shard       :117-141  per hop: deg = off[cur+1]-off[cur]; alive &= deg>0;
//                               draw = rng.random(n) (one per row, alive or not);
//                               pick = min(int(draw*deg), deg-1) in float64
//   duplicate_free    :186-202  keep first occurrence per root group
//   project_corpus    :323-341
// The draw for (shard s, hop h, row i) is stream element k = h*n_s + i, so a
// walker addresses it directly: PCG64 by affine jump-ahead, Philox by counter.
#include "common.cuh"
#include "primitives.cuh"
#include "../../include/walkvec_b200.h"

namespace wv {

constexpr int kShard = 8192;  // walks.py:34 SHARD_SIZE
constexpr int kWalkThreads = 256;

// PCG64 jump table: entry b advances 2^b steps (multiplier-only, so shared).
__constant__ PcgJump c_pcg_pow2[64];
static uint64_t g_pcg_table_ready = 0;  // bit per device

static cudaError_t ensure_pcg_table() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64 && (g_pcg_table_ready >> dev) & 1) return cudaSuccess;
  PcgJump tab[64];
  pcg_jump_table(tab, 64);
  e = cudaMemcpyToSymbol(c_pcg_pow2, tab, sizeof(tab));
  if (e == cudaSuccess && dev < 64) g_pcg_table_ready |= (1ull << dev);
  return e;
}

__device__ __forceinline__ PcgJump pcg_jump_dev(uint64_t n) {
  PcgJump r{u128{1, 0}, u128{0, 0}};
  for (int b = 0; n; ++b, n >>= 1)
    if (n & 1) r = jump_compose(r, c_pcg_pow2[b]);
  return r;
}

struct WalkParams {
  const int64_t* row_offsets;
  const uint64_t* edges;
  const uint4* adj;  // optional walk adjacency: per edge {pred, dst, first edge of dst, out-degree of dst}
  const int64_t* roots;
  int64_t walk_number;
  double inv_walk_number;
  int64_t work_begin;  // global index of the first walker of this launch
  int64_t work_count;  // walkers in this launch
  int64_t last_shard;  // global shard index of the final (possibly partial) shard
  int64_t n_last;      // its row count
  int depth;
  int width;
  int n_prefix;
  uint32_t prefix[13];
  PcgJump stride_full;  // 8192 steps
  PcgJump stride_last;  // n_last steps
  int32_t* corpus;
  int32_t* lengths;
};

// Per-device table of the affine PCG64 jumps of n = 1..kShard steps: walker
// row i of a shard starts from jump(i + 1) of the shard's seeded state (one
// coalesced 32-byte load instead of a 13-step square-and-multiply per lane).
static PcgJump* g_jump_rows[16] = {nullptr};

__global__ void fill_jump_rows(PcgJump* tab) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n < kShard) tab[n] = pcg_jump_dev((uint64_t)n + 1);
}

static cudaError_t ensure_jump_rows(PcgJump** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
  if (g_jump_rows[dev] == nullptr) {
    PcgJump* t = nullptr;
    e = cudaMalloc(&t, sizeof(PcgJump) * kShard);
    if (e != cudaSuccess) return e;
    fill_jump_rows<<<kShard / 256, 256>>>(t);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return e;
    g_jump_rows[dev] = t;
  }
  *out = g_jump_rows[dev];
  return cudaSuccess;
}

// Generator state of one walker in flight.
struct Walker {
  u128 x;      // PCG64 state before its next draw
  u128 cstep;  // inc * S of the per-hop stride
  uint64_t i;  // row within the shard (Philox counter)
  int64_t cur;
  int len;
  bool last;   // in the final (short) shard
  bool alive;
};

// Random walks, WPT walkers per thread.  Walker w of the root-major work list
// is row i = w mod 8192 of shard s = w / 8192; its draw for hop h is element
// h * n_s + i of the shard's stream (walks.py:117-141, 166-173).  Two lanes
// per CTA seed the (at most two) shards the CTA's walkers fall in
// (SeedSequence -> PCG64 / Philox key, shared memory); each walker then jumps
// to its row with one table load.  The
// hop loop interleaves the thread's walkers so their dependent CSR reads
// (offsets -> packed edge) overlap.  Rows are staged in shared memory and
// written with 16-byte stores.
// Per-shard generator seeds (SeedSequence([seed, 0, s]) -> PCG64 state + inc, or
// the Philox key), computed once per shard of the launch instead of once per CTA:
// a shard spans 16 CTAs of 512 walkers, and the hashing is a serial chain the
// CTA's other warps wait on.
#ifndef WV_WALK_SEED_TABLE
#define WV_WALK_SEED_TABLE 1
#endif
template <int RNG>
__global__ void seed_shards(WalkParams P, int64_t s_first, int64_t n, uint64_t* __restrict__ tab) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint32_t pool[4];
  ss_pool(P.prefix, P.n_prefix, (uint64_t)(s_first + t), pool);
  uint64_t* o = tab + 4 * t;
  if (RNG == WV_RNG_PCG64) {
    const Pcg64 g = pcg_seed(pool);
    o[0] = g.state.lo;
    o[1] = g.state.hi;
    o[2] = g.inc.lo;
    o[3] = g.inc.hi;
  } else {
    uint64_t key[2];
    ss_generate_u64(pool, 2, key);
    o[0] = key[0];
    o[1] = key[1];
    o[2] = o[3] = 0;
  }
}

#ifndef WV_WALK_MINB
#define WV_WALK_MINB 4
#endif
template <int RNG, int WPT>
__global__ void __launch_bounds__(kWalkThreads, RNG == WV_RNG_PCG64 ? WV_WALK_MINB : 1) random_walk_kernel(WalkParams P,
                                                                              const PcgJump* __restrict__ jrows,
                                                                              const uint64_t* __restrict__ seeds,
                                                                              int64_t s_first, int64_t n_seeds) {
  extern __shared__ int32_t stage[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int width = P.width;
  const int64_t blk0 = blockIdx.x * (int64_t)kWalkThreads * WPT;
  // the CTA's walkers span at most two shards (kWalkThreads * WPT <= kShard):
  // lanes 0/1 of warp 0 seed them once for the whole CTA
  __shared__ uint64_t sh_seed[2][4];  // PCG64: state.lo, state.hi, inc.lo, inc.hi; Philox: key
  const int64_t s0 = (P.work_begin + blk0) / kShard;
  if (seeds != nullptr) {
    if (threadIdx.x < 8) {  // two shards x four words from the launch's seed table
      const int64_t t = s0 + (threadIdx.x >> 2) - s_first;
      if (t < n_seeds) sh_seed[threadIdx.x >> 2][threadIdx.x & 3] = seeds[4 * t + (threadIdx.x & 3)];
    }
  } else if (warp == 0 && lane < 2) {
    uint32_t pool[4];
    ss_pool(P.prefix, P.n_prefix, (uint64_t)(s0 + lane), pool);
    if (RNG == WV_RNG_PCG64) {
      const Pcg64 g = pcg_seed(pool);
      sh_seed[lane][0] = g.state.lo;
      sh_seed[lane][1] = g.state.hi;
      sh_seed[lane][2] = g.inc.lo;
      sh_seed[lane][3] = g.inc.hi;
    } else {
      uint64_t key[2];
      ss_generate_u64(pool, 2, key);
      sh_seed[lane][0] = key[0];
      sh_seed[lane][1] = key[1];
    }
  }
  Walker W[WPT];
  uint64_t k0[WPT], k1[WPT];
  const PcgJump* jr[WPT];
#pragma unroll
  for (int q = 0; q < WPT; ++q) {
    // walker q of this thread: sub-block q, so each warp's 32 walkers are consecutive
    const int64_t wl = blk0 + (int64_t)q * kWalkThreads + threadIdx.x;
    int32_t* my = stage + ((q * kWalkThreads) + warp * 32 + lane) * width;
    W[q].alive = wl < P.work_count;
    W[q].len = 0;
    W[q].cur = 0;
    const int64_t w = P.work_begin + (W[q].alive ? wl : 0);
    const int64_t s = w / kShard;
    W[q].i = (uint64_t)(w - s * kShard);
    W[q].last = (s == P.last_shard);
    jr[q] = jrows + W[q].i;  // i + 1 steps
    if (W[q].alive) {
      // root index w / walk_number via a float64 reciprocal and a one-step correction
      // (a 64-bit integer division costs ~70 instructions per walker)
      int64_t ri = (int64_t)((double)w * P.inv_walk_number);
      if (ri * P.walk_number > w) --ri;
      else if ((ri + 1) * P.walk_number <= w) ++ri;
      W[q].cur = P.roots[ri];
      my[0] = (int32_t)W[q].cur;
      W[q].len = 1;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < WPT; ++q) {
    const int64_t wl = blk0 + (int64_t)q * kWalkThreads + threadIdx.x;
    const int src = W[q].alive ? (int)((P.work_begin + wl) / kShard - s0) : 0;
    const uint64_t* sd = sh_seed[src];
    if (RNG == WV_RNG_PCG64) {
      const u128 state{sd[0], sd[1]}, inc{sd[2], sd[3]};
      const PcgJump j = *jr[q];
      W[q].x = add128(mul128(j.A, state), mul128(inc, j.S));
      W[q].cstep = mul128(inc, W[q].last ? P.stride_last.S : P.stride_full.S);
    } else {
      k0[q] = sd[0];
      k1[q] = sd[1];
    }
  }
  const int64_t* __restrict__ off = P.row_offsets;
  const uint64_t* __restrict__ edges = P.edges;
  if (P.adj != nullptr) {
    // one dependent 16-byte load per hop: the chosen edge carries the next vertex's
    // row start and degree (the CSR offsets are read once, for the root)
    const uint4* __restrict__ adj = P.adj;
    uint32_t start[WPT], deg[WPT];
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      start[q] = deg[q] = 0;
      if (W[q].alive) {
        const int64_t lo = __ldg(off + W[q].cur), hi = __ldg(off + W[q].cur + 1);
        start[q] = (uint32_t)lo;
        deg[q] = (uint32_t)(hi - lo);
      }
    }
    for (int h = 0; h < P.depth; ++h) {
      uint4 e[WPT];
#pragma unroll
      for (int q = 0; q < WPT; ++q) {
        if (W[q].alive && deg[q] == 0) W[q].alive = false;
        uint64_t u = 0;
        if (RNG == WV_RNG_PCG64) {
          u = pcg_output(W[q].x);
          W[q].x = add128(mul128(W[q].last ? P.stride_last.A : P.stride_full.A, W[q].x), W[q].cstep);
        } else if (W[q].alive) {
          const uint64_t n_s = W[q].last ? (uint64_t)P.n_last : (uint64_t)kShard;
          u = philox_numpy_u64(k0[q], k1[q], (uint64_t)h * n_s + W[q].i);
        }
        const int64_t dg = (int64_t)deg[q];
        int64_t pick = __double2ll_rz(__dmul_rn(u64_to_double(u), (double)dg));
        if (pick > dg - 1) pick = dg - 1;
        e[q] = W[q].alive ? __ldg(adj + (int64_t)start[q] + pick) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int q = 0; q < WPT; ++q) {
        if (W[q].alive) {
          int32_t* my = stage + ((q * kWalkThreads) + warp * 32 + lane) * width;
          my[2 * h + 1] = (int32_t)e[q].x;
          my[2 * h + 2] = (int32_t)e[q].y;
          W[q].cur = (int64_t)e[q].y;
          start[q] = e[q].z;
          deg[q] = e[q].w;
          W[q].len += 2;
        }
      }
      bool any = false;
#pragma unroll
      for (int q = 0; q < WPT; ++q) any |= W[q].alive;
      if (!any) break;
    }
  }
  for (int h = 0; h < (P.adj != nullptr ? 0 : P.depth); ++h) {
    int64_t lo[WPT], hi[WPT];
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      lo[q] = hi[q] = 0;
      if (W[q].alive) {
        lo[q] = __ldg(off + W[q].cur);
        hi[q] = __ldg(off + W[q].cur + 1);
      }
    }
    uint64_t e[WPT];
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      if (W[q].alive && hi[q] == lo[q]) W[q].alive = false;
      uint64_t u = 0;
      if (RNG == WV_RNG_PCG64) {
        u = pcg_output(W[q].x);
        W[q].x = add128(mul128(W[q].last ? P.stride_last.A : P.stride_full.A, W[q].x), W[q].cstep);
      } else if (W[q].alive) {
        const uint64_t n_s = W[q].last ? (uint64_t)P.n_last : (uint64_t)kShard;
        u = philox_numpy_u64(k0[q], k1[q], (uint64_t)h * n_s + W[q].i);
      }
      const int64_t deg = hi[q] - lo[q];
      int64_t pick = __double2ll_rz(__dmul_rn(u64_to_double(u), (double)deg));
      if (pick > deg - 1) pick = deg - 1;
      e[q] = W[q].alive ? __ldg(edges + lo[q] + pick) : 0ull;
    }
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      if (W[q].alive) {
        int32_t* my = stage + ((q * kWalkThreads) + warp * 32 + lane) * width;
        my[2 * h + 1] = (int32_t)(e[q] >> 32);
        my[2 * h + 2] = (int32_t)(uint32_t)e[q];
        W[q].cur = (int64_t)(uint32_t)e[q];
        W[q].len += 2;
      }
    }
    bool any = false;
#pragma unroll
    for (int q = 0; q < WPT; ++q) any |= W[q].alive;
    if (!any) break;
  }
#pragma unroll
  for (int q = 0; q < WPT; ++q) {
    const int64_t wl = blk0 + (int64_t)q * kWalkThreads + threadIdx.x;
    if (wl < P.work_count) P.lengths[wl] = W[q].len;
    // pad the staged row past the walk's end (-1, the reference's PAD)
    int32_t* my = stage + ((q * kWalkThreads) + warp * 32 + lane) * width;
    for (int j = W[q].len; j < width; ++j) my[j] = -1;
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < WPT; ++q) {
    const int64_t wl0 = blk0 + (int64_t)q * kWalkThreads + warp * 32;
    if (wl0 >= P.work_count) continue;
    const int64_t nvalid = min((int64_t)32, P.work_count - wl0);
    const int32_t* srcr = stage + ((q * kWalkThreads) + warp * 32) * width;
    int32_t* dst = P.corpus + wl0 * width;
    const int total = (int)nvalid * width;
    if (nvalid == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
      const int4* s4 = reinterpret_cast<const int4*>(srcr);
      int4* d4 = reinterpret_cast<int4*>(dst);
      for (int j = lane; j < total / 4; j += 32) d4[j] = s4[j];
    } else {
      for (int j = lane; j < total; j += 32) dst[j] = srcr[j];
    }
  }
}

// walk adjacency (wv_walk_adjacency_build): per edge e of the packed CSR,
// {pred, dst, row start of dst, out-degree of dst}; E < 2^32 (row starts fit u32)
__global__ void walk_adj_build(const int64_t* __restrict__ off, const uint64_t* __restrict__ edges, int64_t E,
                               uint4* __restrict__ adj) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t pe = edges[e];
    const uint32_t dst = (uint32_t)pe;
    const int64_t lo = off[dst], hi = off[dst + 1];
    adj[e] = make_uint4((uint32_t)(pe >> 32), dst, (uint32_t)lo, (uint32_t)(hi - lo));
  }
}

// ---------------------------------------------------------- compaction ----
template <typename TokOut>
__global__ void compact_rows(const int32_t* __restrict__ corpus, const int32_t* __restrict__ lengths,
                             int64_t n_walks, int width, const int64_t* __restrict__ offsets,
                             TokOut* __restrict__ tokens) {
  const int64_t total = n_walks * width;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = idx / width;
    const int j = (int)(idx - w * width);
    if (j < lengths[w]) tokens[offsets[w] + j] = (TokOut)corpus[idx];
  }
}

__global__ void set_last_offset(int64_t* offsets, int64_t n, const int64_t* total) { offsets[n] = *total; }

// ----------------------------------------------------- duplicate-free ----
__global__ void row_hash(const int32_t* __restrict__ corpus, const int32_t* __restrict__ lengths, int64_t n_walks,
                         int width, uint64_t* __restrict__ hash) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    const int L = lengths[w];
    uint64_t h = splitmix64((uint64_t)L);
    for (int j = 0; j < L; ++j) h = splitmix64(h ^ (uint64_t)(uint32_t)corpus[w * width + j]);
    hash[w] = h;
  }
}

__global__ void first_occurrence(const int32_t* __restrict__ corpus, const int32_t* __restrict__ lengths,
                                 int64_t n_walks, int width, int64_t group, const uint64_t* __restrict__ hash,
                                 uint8_t* __restrict__ keep) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g0 = (w / group) * group;
    const uint64_t h = hash[w];
    const int L = lengths[w];
    bool first = true;
    for (int64_t q = g0; q < w && first; ++q) {
      if (hash[q] != h || lengths[q] != L) continue;
      bool same = true;
      for (int j = 0; j < L && same; ++j) same = corpus[q * width + j] == corpus[w * width + j];
      if (same) first = false;
    }
    keep[w] = first ? 1 : 0;
  }
}

__global__ void masked_lengths(const int32_t* __restrict__ lengths, const uint8_t* __restrict__ keep,
                               int64_t n, int32_t* __restrict__ out) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n; w += (int64_t)gridDim.x * blockDim.x)
    out[w] = keep[w] ? lengths[w] : 0;
}

__global__ void gather_kept_rows(const int32_t* __restrict__ corpus, const int32_t* __restrict__ lengths,
                                 const uint8_t* __restrict__ keep, const int64_t* __restrict__ new_index,
                                 int64_t n_walks, int width, int32_t* __restrict__ out_corpus,
                                 int32_t* __restrict__ out_lengths) {
  const int64_t total = n_walks * width;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = idx / width;
    if (!keep[w]) continue;
    const int j = (int)(idx - w * width);
    const int64_t nw = new_index[w];
    out_corpus[nw * width + j] = corpus[idx];
    if (j == 0) out_lengths[nw] = lengths[w];
  }
}

// ------------------------------------------------ flat-corpus filtering ----
// mode: WV_KEEP_ENTITY (even positions), WV_KEEP_PROPERTY (0 + odd positions),
//       WV_KEEP_TOKENS (token mask, min_count filter; w2v.py:146-158)
__device__ __forceinline__ bool keep_pos(int mode, int64_t pos, int32_t tok, const uint8_t* mask) {
  if (mode == WV_KEEP_ENTITY) return (pos & 1) == 0;
  if (mode == WV_KEEP_PROPERTY) return pos == 0 || (pos & 1) == 1;
  return mask[tok] != 0;
}

__global__ void filter_count(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets, int64_t n_walks,
                             int mode, const uint8_t* __restrict__ mask, int64_t* __restrict__ kept) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    for (int64_t p = offsets[w]; p < offsets[w + 1]; ++p) c += keep_pos(mode, p - offsets[w], tokens[p], mask);
    kept[w] = c;
  }
}

__global__ void filter_scatter(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets, int64_t n_walks,
                               int mode, const uint8_t* __restrict__ mask, const int64_t* __restrict__ new_offsets,
                               int32_t* __restrict__ out) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = new_offsets[w];
    for (int64_t p = offsets[w]; p < offsets[w + 1]; ++p) {
      const int32_t t = tokens[p];
      if (keep_pos(mode, p - offsets[w], t, mask)) out[o++] = t;
    }
  }
}

// ------------------------------------------------------------ histogram ----
// Warp-aggregated: lanes holding the same token (hot predicate rows) merge
// into one atomic.
__global__ void token_hist(const int32_t* __restrict__ tokens, int64_t n, unsigned long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    const int32_t t = i < n ? tokens[i] : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, t);
    if (t >= 0 && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&counts[t], (unsigned long long)__popc(peers));
  }
}

static inline unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (unsigned)g;
}

static inline int64_t al256(int64_t b) { return (b + 255) & ~(int64_t)255; }

}  // namespace wv

extern "C" {

int wv_walk_adjacency_build(const int64_t* row_offsets, const uint64_t* packed_edges, int64_t vertex_count,
                            int64_t edge_count, void* walk_adj, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(edge_count >= 0 && edge_count < (1ll << 32), "walk adjacency needs fewer than 2^32 edges");
  WV_CHECK_ARG(vertex_count < (1ll << 32), "walk adjacency needs fewer than 2^32 vertices");
  if (edge_count == 0) return 0;
  const int64_t g = (edge_count + 255) / 256;
  walk_adj_build<<<(unsigned)(g < 148 * 32 ? g : 148 * 32), 256, 0, (cudaStream_t)stream>>>(
      row_offsets, packed_edges, edge_count, (uint4*)walk_adj);
  WV_LAUNCH_CHECK();
  return 0;
}

int64_t wv_random_walks_workspace_bytes(int64_t work_begin, int64_t work_count) {
  using namespace wv;
  if (work_count <= 0) return 256;
  const int64_t n_seeds = (work_begin + work_count - 1) / kShard - work_begin / kShard + 1;
  return n_seeds * 32 + 256;
}

int wv_random_walks(const int64_t* row_offsets, const uint64_t* packed_edges, const void* walk_adj,
                    int64_t vertex_count,
                    const int64_t* roots, int64_t n_roots, int64_t walk_number, int walk_depth,
                    int64_t work_begin, int64_t work_count, const uint32_t* seed_prefix, int n_prefix, int rng_kind,
                    int32_t* corpus, int32_t* lengths, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(walk_depth >= 1, "walk_depth must be >= 1");
  WV_CHECK_ARG(walk_number >= 1, "walk_number must be >= 1");
  WV_CHECK_ARG(n_roots >= 1, "start_vertices must be non-empty");
  WV_CHECK_ARG(vertex_count >= 1, "empty graph");
  WV_CHECK_ARG(n_prefix >= 0 && n_prefix <= 13, "seed prefix too long");
  WV_CHECK_ARG(rng_kind == WV_RNG_PCG64 || rng_kind == WV_RNG_PHILOX, "unknown rng kind %d", rng_kind);
  const int64_t total = n_roots * walk_number;
  WV_CHECK_ARG(work_begin >= 0 && work_count >= 0 && work_begin + work_count <= total, "work range out of bounds");
  const int width = 2 * walk_depth + 1;
  WV_CHECK_ARG((int64_t)kWalkThreads * width * 4 <= 227 * 1024, "walk_depth %d exceeds the staged-row limit (110)",
               walk_depth);
  if (work_count == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  WV_CUDA(ensure_pcg_table());
  WalkParams P;
  P.row_offsets = row_offsets;
  P.edges = packed_edges;
  P.adj = (const uint4*)walk_adj;
  P.roots = roots;
  P.walk_number = walk_number;
  P.inv_walk_number = 1.0 / (double)walk_number;
  P.work_begin = work_begin;
  P.work_count = work_count;
  P.last_shard = (total - 1) / kShard;
  P.n_last = total - P.last_shard * kShard;
  P.depth = walk_depth;
  P.width = width;
  P.n_prefix = n_prefix;
  for (int i = 0; i < n_prefix; ++i) P.prefix[i] = seed_prefix[i];
  PcgJump tab[64];
  pcg_jump_table(tab, 64);
  P.stride_full = pcg_jump_n(tab, kShard);
  P.stride_last = pcg_jump_n(tab, (uint64_t)P.n_last);
  P.corpus = corpus;
  P.lengths = lengths;
  PcgJump* jrows = nullptr;
  WV_CUDA(ensure_jump_rows(&jrows));
  // two walkers per thread while their staged rows fit in shared memory
  const bool two = (size_t)2 * kWalkThreads * width * sizeof(int32_t) <= 96 * 1024;
  const int wpt = two ? 2 : 1;
  const size_t smem = (size_t)wpt * kWalkThreads * width * sizeof(int32_t);
  const int64_t per_block = (int64_t)kWalkThreads * wpt;
  const int64_t blocks = (work_count + per_block - 1) / per_block;
  WV_CHECK_ARG(blocks < (1ll << 31), "too many walkers for one launch");
  uint64_t* seeds = nullptr;
  const int64_t s_first = work_begin / kShard;
  const int64_t n_seeds = work_count > 0 ? (work_begin + work_count - 1) / kShard - s_first + 1 : 0;
  if (WV_WALK_SEED_TABLE && n_seeds > 0 && ws != nullptr) {
    WV_CHECK_ARG(ws_bytes >= wv_random_walks_workspace_bytes(work_begin, work_count), "workspace too small");
    seeds = (uint64_t*)ws;  // per-shard seeds in the caller's workspace (ws = NULL: seeded per CTA)
    if (rng_kind == WV_RNG_PCG64)
      seed_shards<WV_RNG_PCG64><<<(unsigned)((n_seeds + 127) / 128), 128, 0, st>>>(P, s_first, n_seeds, seeds);
    else
      seed_shards<WV_RNG_PHILOX><<<(unsigned)((n_seeds + 127) / 128), 128, 0, st>>>(P, s_first, n_seeds, seeds);
    WV_LAUNCH_CHECK();
  }
  auto launch = [&](auto kern) -> int {
    if (smem > 48 * 1024)
      WV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)blocks, kWalkThreads, smem, st>>>(P, jrows, seeds, s_first, n_seeds);
    return 0;
  };
  int rc;
  if (rng_kind == WV_RNG_PCG64)
    rc = two ? launch(random_walk_kernel<WV_RNG_PCG64, 2>) : launch(random_walk_kernel<WV_RNG_PCG64, 1>);
  else
    rc = two ? launch(random_walk_kernel<WV_RNG_PHILOX, 2>) : launch(random_walk_kernel<WV_RNG_PHILOX, 1>);
  if (rc) return rc;
  WV_LAUNCH_CHECK();
  return 0;
}

int64_t wv_compact_workspace_bytes(int64_t n_walks) {
  using namespace wv;
  return al256(scan_tiles(n_walks + 1) * 8) + al256(8) + 256;
}

int wv_corpus_compact(const int32_t* corpus, const int32_t* lengths, int64_t n_walks, int width,
                      int64_t* offsets, void* tokens, int token_bytes, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(token_bytes == 4 || token_bytes == 8, "token_bytes must be 4 or 8");
  WV_CHECK_ARG(ws_bytes >= wv_compact_workspace_bytes(n_walks), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  int64_t* scan_ws = (int64_t*)w;
  w += al256(scan_tiles(n_walks + 1) * 8);
  int64_t* total = (int64_t*)w;
  WV_CUDA((excl_scan<int32_t, int64_t>(lengths, n_walks, offsets, total, scan_ws, st)));
  set_last_offset<<<1, 1, 0, st>>>(offsets, n_walks, total);
  WV_LAUNCH_CHECK();
  if (n_walks == 0) return 0;
  const int64_t cells = n_walks * width;
  if (token_bytes == 4)
    compact_rows<int32_t><<<grid_for(cells, 256), 256, 0, st>>>(corpus, lengths, n_walks, width, offsets,
                                                                 (int32_t*)tokens);
  else
    compact_rows<int64_t><<<grid_for(cells, 256), 256, 0, st>>>(corpus, lengths, n_walks, width, offsets,
                                                                 (int64_t*)tokens);
  WV_LAUNCH_CHECK();
  return 0;
}

int64_t wv_dedup_workspace_bytes(int64_t n_walks) {
  using namespace wv;
  return al256(n_walks * 8) * 2 + al256(n_walks) + al256(scan_tiles(n_walks) * 8) + al256(8) + 256;
}

// Duplicate-free (walks.py:186-202): within each group of `group` consecutive
// walks keep the first occurrence of each distinct token sequence.  Writes
// the kept rows (in order) to out_corpus/out_lengths and their count to
// *n_kept (device int64).
int wv_duplicate_free(const int32_t* corpus, const int32_t* lengths, int64_t n_walks, int width, int64_t group,
                      int32_t* out_corpus, int32_t* out_lengths, int64_t* n_kept, void* ws, int64_t ws_bytes,
                      void* stream) {
  using namespace wv;
  WV_CHECK_ARG(group >= 1, "group must be >= 1");
  WV_CHECK_ARG(ws_bytes >= wv_dedup_workspace_bytes(n_walks), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (n_walks == 0) {
    WV_CUDA(cudaMemsetAsync(n_kept, 0, 8, st));
    return 0;
  }
  char* w = (char*)ws;
  uint64_t* hash = (uint64_t*)w;
  w += al256(n_walks * 8);
  int64_t* new_index = (int64_t*)w;
  w += al256(n_walks * 8);
  uint8_t* keep = (uint8_t*)w;
  w += al256(n_walks);
  int64_t* scan_ws = (int64_t*)w;
  row_hash<<<grid_for(n_walks, 256), 256, 0, st>>>(corpus, lengths, n_walks, width, hash);
  first_occurrence<<<grid_for(n_walks, 128), 128, 0, st>>>(corpus, lengths, n_walks, width, group, hash, keep);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<uint8_t, int64_t>(keep, n_walks, new_index, n_kept, scan_ws, st)));
  gather_kept_rows<<<grid_for(n_walks * width, 256), 256, 0, st>>>(corpus, lengths, keep, new_index, n_walks, width,
                                                                     out_corpus, out_lengths);
  WV_LAUNCH_CHECK();
  return 0;
}

int64_t wv_filter_workspace_bytes(int64_t n_walks) {
  using namespace wv;
  return al256((n_walks + 1) * 8) + al256(scan_tiles(n_walks + 1) * 8) + al256(8) + 256;
}

// Flat corpus filter: per-walk keep predicate -> new offsets (n_walks+1) and
// tokens.  Walk count is preserved (empty walks stay, as in the reference).
int wv_corpus_filter(const int32_t* tokens, const int64_t* offsets, int64_t n_walks, int mode,
                     const uint8_t* token_mask, int64_t* new_offsets, int32_t* new_tokens, void* ws, int64_t ws_bytes,
                     void* stream) {
  using namespace wv;
  WV_CHECK_ARG(mode == WV_KEEP_ENTITY || mode == WV_KEEP_PROPERTY || mode == WV_KEEP_TOKENS, "bad filter mode");
  WV_CHECK_ARG(mode != WV_KEEP_TOKENS || token_mask != nullptr, "token mask required");
  WV_CHECK_ARG(ws_bytes >= wv_filter_workspace_bytes(n_walks), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  int64_t* kept = (int64_t*)w;
  w += al256((n_walks + 1) * 8);
  int64_t* scan_ws = (int64_t*)w;
  w += al256(scan_tiles(n_walks + 1) * 8);
  int64_t* total = (int64_t*)w;
  if (n_walks > 0) {
    filter_count<<<grid_for(n_walks, 256), 256, 0, st>>>(tokens, offsets, n_walks, mode, token_mask, kept);
    WV_LAUNCH_CHECK();
  }
  WV_CUDA((excl_scan<int64_t, int64_t>(kept, n_walks, new_offsets, total, scan_ws, st)));
  set_last_offset<<<1, 1, 0, st>>>(new_offsets, n_walks, total);
  if (n_walks > 0)
    filter_scatter<<<grid_for(n_walks, 256), 256, 0, st>>>(tokens, offsets, n_walks, mode, token_mask, new_offsets,
                                                           new_tokens);
  WV_LAUNCH_CHECK();
  return 0;
}

int wv_token_histogram(const int32_t* tokens, int64_t n_tokens, int64_t vocab_size, int64_t* counts, int zero_first,
                       void* stream) {
  using namespace wv;
  cudaStream_t st = (cudaStream_t)stream;
  if (zero_first) WV_CUDA(cudaMemsetAsync(counts, 0, vocab_size * 8, st));
  if (n_tokens == 0) return 0;
  token_hist<<<grid_for(n_tokens, 256), 256, 0, st>>>(tokens, n_tokens, (unsigned long long*)counts);
  WV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
