// SGNS training kernels (skip-gram, negative sampling, per-row Adam).
//
// Reference semantics (pkg/src/walkvec/w2v.py):
//   init_embeddings     :123-131  U(-1/d, 1/d) float64 from SeedSequence([seed,1,0]),
//                                 input matrix then output matrix
//   generate_pairs      :161-191  shift-major (s=1..W) blocks (t[i],t[i+s]) then (t[i+s],t[i])
//   _train_single       :547-576  permutation per epoch, contiguous batches, fresh
//                                 negatives per batch, non-finite loss -> TrainingDiverged
//   _sgns_forward /
//   sgns_batch_grads    :247-299  gradients of the batch-mean BCE loss
//   _coalesce           :407-416  duplicate rows summed in slot order
//   RowAdam.update      :384-404  per-row step counts (sparse) / global step (dense)
//
// B200 design: one warp per pair gathers the (2+k) rows with 16-byte loads,
// reduces the (1+k) dots with shuffles and emits the per-pair coefficients
// plus two [B,d] rows (the centre row u and its gradient).  A stable radix
// sort groups every contribution by destination row in the reference's slot
// order; one warp per unique row then sums its contributions and applies
// Adam in place.  No float atomics: results are deterministic run to run.
#include <cfloat>
#include <cstdlib>
#include <cmath>

#include "common.cuh"
#include "primitives.cuh"
#include "../../include/walkvec_b200.h"

namespace wv {

constexpr int kPairThreads = 256;
constexpr int kPairWarps = kPairThreads / 32;
constexpr int kOwnerThreads = 256;
#ifndef WV_FP64_RCP
// float64 RowAdam with the per-row reciprocals of the bias corrections: m * (1 / bc1) and
// v * (1 / bc2) instead of numpy's two divisions (each within an ulp; the fp64 parity bound
// stays 1e-12).  Two fewer correctly rounded divides per element: single-row owner
// 279 -> 271 us, step +2.0 % (profiles/r02/abn_r02x_fp64.txt); 0 keeps numpy's divisions.
#define WV_FP64_RCP 1
#endif
#ifndef WV_SINGLES
#define WV_SINGLES 2  // single-contribution rows through sgns_owner_single_kernel: 0 never, 1 always, 2 float64
                      // (fp64 +1.1 %; fp32 -13 %: its heavy pieces no longer hide behind the light rows)
#endif
#ifndef WV_SINGLES_SERIAL
#define WV_SINGLES_SERIAL 0  // heavy pieces then multi-contribution rows serially (0: concurrently)
#endif
#ifndef WV_SINGLES_CONCURRENT
// 1: the single-contribution rows run beside the heavy pieces and multi-contribution rows
// (which go to the high-priority stream ss->h) instead of after them; the singles kernel is
// then launched as short-lived tiles (WV_SINGLE_TILE) so the latency-bound heavy / multi
// CTAs take SM slots as soon as any free up and the singles fill the rest of the bandwidth
// (fp64: +1.6 % over singles-after, tiles of 8 / 12 / 16 items per thread alike, 2: -8 %,
// 32: -4 %; the heavy stream at low priority: -9 %; profiles/r02/abn_r02a[ab]_*.txt)
#define WV_SINGLES_CONCURRENT 1
#endif
#ifndef WV_SINGLE_TILE
#define WV_SINGLE_TILE 12  // (row, chunk) items per thread of one singles CTA in the concurrent schedule
#endif
#ifndef WV_MULTI_PER_SM
#define WV_MULTI_PER_SM 0  // CTAs per SM of the multi-contribution light rows (0: all resident)
#endif
#ifndef WV_SINGLE_MINB
#define WV_SINGLE_MINB 4  // 64 registers (5: 48 with a 32-byte stack, -5 %)
#endif
#ifndef WV_OWNER_GROUP
#define WV_OWNER_GROUP 2
#endif
#ifndef WV_OWNER_MINB
#define WV_OWNER_MINB 4
#endif
constexpr int kOwnerGroup = WV_OWNER_GROUP;  // contributions loaded together per light row

// ---------------------------------------------------- precise arithmetic --
// Explicit rounding so the update mirrors numpy's operation order (no FMA
// contraction) in the float64 path.
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float exp_t(float a) { return expf(a); }
// a*b + c: one FMA for float32; float64 keeps numpy's separate rounding
__device__ __forceinline__ float mad_t(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double mad_t(double a, double b, double c) { return __dadd_rn(__dmul_rn(a, b), c); }
__device__ __forceinline__ double exp_t(double a) { return exp(a); }

// ------------------------------------------------------ vector row I/O ----
// Aligned to its own size (4/8/16 B): every chunk sits at a multiple of EPC
// elements from an aligned row base, and the alignment lets shared-memory chunk
// reads compile to one LDS.64/128 instead of EPC conflicting 4-byte LDS.
template <typename T, int EPC>
struct alignas(sizeof(T) * EPC) Chunk {
  T v[EPC];
};

template <typename T, int EPC>
__device__ __forceinline__ Chunk<T, EPC> ld_chunk(const T* p) {
  Chunk<T, EPC> c;
  if constexpr (EPC * sizeof(T) == 16) {
    if constexpr (sizeof(T) == 4) {
      float4 f = __ldg(reinterpret_cast<const float4*>(p));
      c.v[0] = f.x; c.v[1] = f.y; c.v[2] = f.z; c.v[3] = f.w;
    } else {
      double2 f = __ldg(reinterpret_cast<const double2*>(p));
      c.v[0] = f.x; c.v[1] = f.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < EPC; ++e) c.v[e] = __ldg(p + e);
  }
  return c;
}

// Coherent load (rows being updated inside the same kernel family).
template <typename T, int EPC>
__device__ __forceinline__ Chunk<T, EPC> ld_chunk_rw(const T* p) {
  Chunk<T, EPC> c;
  if constexpr (EPC * sizeof(T) == 16) {
    if constexpr (sizeof(T) == 4) {
      float4 f = *reinterpret_cast<const float4*>(p);
      c.v[0] = f.x; c.v[1] = f.y; c.v[2] = f.z; c.v[3] = f.w;
    } else {
      double2 f = *reinterpret_cast<const double2*>(p);
      c.v[0] = f.x; c.v[1] = f.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < EPC; ++e) c.v[e] = p[e];
  }
  return c;
}

template <typename T, int EPC>
__device__ __forceinline__ void st_chunk(T* p, const Chunk<T, EPC>& c) {
  if constexpr (EPC * sizeof(T) == 16) {
    if constexpr (sizeof(T) == 4) {
      *reinterpret_cast<float4*>(p) = make_float4(c.v[0], c.v[1], c.v[2], c.v[3]);
    } else {
      *reinterpret_cast<double2*>(p) = make_double2(c.v[0], c.v[1]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < EPC; ++e) p[e] = c.v[e];
  }
}

// Streaming (evict-first) 16-byte row I/O for the optimizer moments: they are
// touched once per batch, so they should not push the parameter rows the
// gather just read out of L2.
#ifndef WV_OWNER_MV_STREAM
#define WV_OWNER_MV_STREAM 0  // loads and stores; measured slower (owner 151 -> 161 us)
#endif
#ifndef WV_OWNER_MV_STCS
#define WV_OWNER_MV_STCS 0  // stores only (fp64, with or without WV_OWNER_P_STCS: -1.2 %, r02ag)
#endif
#ifndef WV_OWNER_P_STCS
#define WV_OWNER_P_STCS 0
#endif
template <typename T, int EPC>
__device__ __forceinline__ Chunk<T, EPC> ld_chunk_mv(const T* p) {
  if constexpr (WV_OWNER_MV_STREAM && EPC * sizeof(T) == 16 && sizeof(T) == 4) {
    const float4 f = __ldcs(reinterpret_cast<const float4*>(p));
    Chunk<T, EPC> c;
    c.v[0] = f.x; c.v[1] = f.y; c.v[2] = f.z; c.v[3] = f.w;
    return c;
  } else {
    return ld_chunk_rw<T, EPC>(p);
  }
}
template <typename T, int EPC>
__device__ __forceinline__ void st_chunk_mv(T* p, const Chunk<T, EPC>& c) {
  if constexpr ((WV_OWNER_MV_STREAM || WV_OWNER_MV_STCS) && EPC * sizeof(T) == 16 && sizeof(T) == 4) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(c.v[0], c.v[1], c.v[2], c.v[3]));
  } else if constexpr (WV_OWNER_MV_STCS && EPC * sizeof(T) == 16 && sizeof(T) == 8) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(c.v[0], c.v[1]));
  } else {
    st_chunk<T, EPC>(p, c);
  }
}
// Parameter-row load in the owner.  WV_OWNER_P_DEMOTE = 1 / 2: read with an L2
// evict-first / evict-normal policy, so lines the gather marked evict-last do
// not stay pinned once their batch has consumed them.
#ifndef WV_OWNER_P_DEMOTE
#define WV_OWNER_P_DEMOTE 0
#endif
#ifndef WV_OWNER_P_APPLY
#define WV_OWNER_P_APPLY 0
#endif
template <typename T, int EPC>
__device__ __forceinline__ Chunk<T, EPC> ld_chunk_p(const T* p) {
  if constexpr (WV_OWNER_P_DEMOTE != 0 && EPC * sizeof(T) == 16 && sizeof(T) == 4) {
    uint64_t pol;
    if (WV_OWNER_P_DEMOTE == 1)
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    Chunk<T, EPC> c;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(c.v[0]), "=f"(c.v[1]), "=f"(c.v[2]), "=f"(c.v[3])
                 : "l"(p), "l"(pol));
    return c;
  } else {
    return ld_chunk_rw<T, EPC>(p);
  }
}
template <typename T, int EPC>
__device__ __forceinline__ void st_chunk_p(T* p, const Chunk<T, EPC>& c) {
  if constexpr (WV_OWNER_P_STCS && EPC * sizeof(T) == 16 && sizeof(T) == 4) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(c.v[0], c.v[1], c.v[2], c.v[3]));
  } else if constexpr (WV_OWNER_P_STCS && EPC * sizeof(T) == 16 && sizeof(T) == 8) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(c.v[0], c.v[1]));
  } else {
    st_chunk<T, EPC>(p, c);
  }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Eight warp sums at once: a transposed butterfly (offsets 16, 8, 4 halve the
// value set, 2 and 1 finish) -- 9 shuffles instead of 40, and every value sees
// exactly the pairwise-add tree of warp_sum.  Lane l returns value (l >> 2) & 7.
template <typename T>
__device__ __forceinline__ T warp_sum8(const T (&p)[8]) {
  const int lane = threadIdx.x & 31;
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
  T a[4], b2[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const T keep = h16 ? p[4 + i] : p[i];
    const T send = h16 ? p[i] : p[4 + i];
    a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const T keep = h8 ? a[2 + i] : a[i];
    const T send = h8 ? a[i] : a[2 + i];
    b2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  T c;
  {
    const T keep = h4 ? b2[1] : b2[0];
    const T send = h4 ? b2[0] : b2[1];
    c = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  c += __shfl_xor_sync(0xffffffffu, c, 2);
  c += __shfl_xor_sync(0xffffffffu, c, 1);
  return c;
}

// numpy logaddexp(0, x)
__device__ __forceinline__ double log1pexp(double x) { return x > 0 ? x + log1p(exp(-x)) : log1p(exp(x)); }

// ------------------------------------------------------------- Feistel ----
struct Feistel {
  int half_bits;
  uint64_t mask;
  uint64_t keys[4];
};

__device__ __forceinline__ Feistel make_feistel(uint64_t seed, uint64_t epoch, int64_t n) {
  Feistel f;
  int bits = 0;
  while (bits < 62 && ((uint64_t)(n - 1) >> bits)) ++bits;
  f.half_bits = (bits + 1) / 2;
  if (f.half_bits < 1) f.half_bits = 1;
  f.mask = (1ull << f.half_bits) - 1;
  uint64_t s = splitmix64(seed * 0x9E3779B97F4A7C15ull + 0x5851F42D4C957F2Dull * (epoch + 1));
  for (int r = 0; r < 4; ++r) {
    s = splitmix64(s + r);
    f.keys[r] = s;
  }
  return f;
}

__device__ __forceinline__ uint64_t feistel_once(const Feistel& f, uint64_t x) {
  uint64_t L = x >> f.half_bits, R = x & f.mask;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    uint64_t nl = R;
    R = L ^ (splitmix64(R ^ f.keys[r]) & f.mask);
    L = nl;
  }
  return (L << f.half_bits) | R;
}

// bijection on [0, n) by cycle walking
__device__ __forceinline__ uint64_t feistel_perm(const Feistel& f, uint64_t pos, int64_t n) {
  uint64_t x = feistel_once(f, pos);
  while (x >= (uint64_t)n) x = feistel_once(f, x);
  return x;
}

// pairs of one walk of length L with window W: 2 * sum_{s=1..min(W,L-1)} (L - s)
__host__ __device__ __forceinline__ int64_t walk_pairs(int64_t L, int W) {
  int64_t t = 0;
  for (int s = 1; s <= W && s < L; ++s) t += 2 * (L - s);
  return t;
}

// local pair q of a length-L walk -> (centre pos, context pos), reference order:
// for s: block A (i, i+s) for i in [0, L-s), then block B (i+s, i).
__device__ __forceinline__ void walk_pair_pos(int64_t L, int W, int64_t q, int64_t& cpos, int64_t& xpos) {
  for (int s = 1; s <= W && s < L; ++s) {
    const int64_t blk = L - s;
    if (q < blk) {
      cpos = q;
      xpos = q + s;
      return;
    }
    q -= blk;
    if (q < blk) {
      cpos = q + s;
      xpos = q;
      return;
    }
    q -= blk;
  }
  cpos = xpos = 0;
}

// ------------------------------------------------------------ the batch ---
// The corpus side of a batch (pair source, negatives).  It lives in device
// memory (the workspace) so a captured CUDA graph of batches stays valid when
// the session moves on to the next corpus: wv_sgns_bind rewrites it.
struct CorpusDesc {
  int mode;  // WV_PAIRS_NATIVE or WV_PAIRS_EXPLICIT
  int window;
  int n_classes;
  int model;  // WV_MODEL_SKIPGRAM or WV_MODEL_CBOW
  int64_t N;  // pairs per epoch
  uint64_t seed;
  // native corpus index
  const int32_t* tokens;
  const int64_t* offsets;
  const int64_t* class_len;
  const int64_t* class_pair_start;  // n_classes + 1
  const int64_t* class_walk_start;
  const int32_t* walks_by_class;
  const int32_t* candidates;  // null => identity over [0, n_candidates)
  int64_t n_candidates;
  // explicit replay
  const int32_t* pairs;      // [N,2]
  const int64_t* perm;       // [N] epoch permutation
  const int32_t* negatives;  // [N,k] per permuted position
  // CBOW instance table [N, 2W + 1] (context columns then the target)
  const int32_t* inst;
};

struct PairArgs {
  int64_t V;
  int d;
  int k;
  int R;   // rows per item: 2 + k (skip-gram) or 2W + 1 + k (CBOW)
  int cw;  // CBOW window W (0: skip-gram)
  int64_t B;  // rows in this batch
  const CorpusDesc* desc;
  // outputs
  void* U;
  void* G;
  void* coef;
  uint32_t* cnt;   // [2V] per-row item count / list cursor; all zero between batches
  uint32_t* uniq;  // [items] unique row keys of the batch
  uint32_t* gctr;  // grouping counters (GC_*)
  int32_t* idx;    // [B, 2+k] centre, context, negatives
  double* partials;
  WvSgnsDevState* state;
  int64_t Bn;     // gradient normaliser (rows of the global batch; 0: B)
  int nshard;     // row-sharded mode: this rank claims rows r with r % nshard == shard
  int shard;
  int64_t Vl;     // local rows per matrix (key space of the claims: [0, 2 Vl))
  uint32_t* rank; // [items] an item's position among its row's items (from the claim)
  uint8_t* flag;  // [2V] row keys the batch touches (the split owner of the previous batch reads them)
};

// ------------------------------------------------------------ grouping ---
// Contributions are grouped by destination row without a sort.  A row key is
// the input-matrix row r (key r) or the output-matrix row r (key V + r); an
// item's slot is its position in the reference's gradient stacking order:
// centre b -> b, context b -> B + b, negative j of pair b -> 2B + bk + j
// (the order np.add.at applies them, w2v.py:287-295, 407-416).
//   decode : cnt[key] += 1 per item; the first item of a key claims a unique id
//   group_segments : per unique key, reserve cnt[key] list slots (cnt[key]
//            becomes the list cursor), advance the row's RowAdam step, split
//            light / heavy rows
//   group_place : each item appends its slot to its row's list
// The list order inside a row is arbitrary; the owner kernels restore slot
// order (warp ranking / CTA radix sort) before summing, so results are
// deterministic, and reset cnt[key] to 0 for the next batch.
enum { GC_UNIQUE = 0, GC_TOTAL = 1, GC_LIGHT = 2, GC_HEAVY = 3, GC_PIECES = 4, GC_NA = 5, GC_NB = 6,
       GC_SINGLE = 7 };

// global row key (row, or V + row) -> local key of this rank, false if another rank owns it
__device__ __forceinline__ bool owned_key(uint32_t key, int64_t V, int nshard, int shard, int64_t Vl, uint32_t& lk) {
  if (nshard <= 1) {
    lk = key;
    return true;
  }
  const bool side = key >= (uint32_t)V;
  const uint32_t row = side ? key - (uint32_t)V : key;
  if ((int)(row % (uint32_t)nshard) != shard) return false;
  lk = row / (uint32_t)nshard + (side ? (uint32_t)Vl : 0u);
  return true;
}

// count the item on its row (the returned count is the item's rank in the
// row's list, so placement needs no second atomic); the first claims the row
__device__ __forceinline__ void group_claim(const PairArgs& A, uint32_t key, int64_t item) {
  const uint32_t active = __activemask();
  uint32_t lk = key;
  const bool owned = A.nshard <= 1 || owned_key(key, A.V, A.nshard, A.shard, A.Vl, lk);
  bool first = false;
  if (owned) {
    const uint32_t r = atomicAdd(A.cnt + lk, 1u);
    A.rank[item] = r;
    first = r == 0u;
    if (first && A.flag) A.flag[lk] = 1;
  }
  // new rows take unique ids with one atomic per warp (GC_UNIQUE is one address)
  const uint32_t fm = __ballot_sync(active, first);
  if (fm == 0u) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(fm) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(A.gctr + GC_UNIQUE, (uint32_t)__popc(fm));
  base = __shfl_sync(active, base, leader);
  if (first) A.uniq[base + __popc(fm & ((1u << lane) - 1u))] = lk;
}

// Phase 1a, thread per item: the batch's row indices (centre, context, k
// negatives) and the row claims for grouping.  Item j = 0 decodes the pair
// (Feistel position -> length class -> walk -> window slot: a chain of
// dependent L2 reads) and writes centre and context; items j >= 2 draw one
// negative each.  Thread-per-item spreads the latency chains over all SMs.
// one negative: Philox4x32 counter (position, epoch, j/2), two draws per call,
// uniform over the candidates; or the replayed numpy stream
__device__ __forceinline__ int32_t draw_negative(const CorpusDesc& D, int64_t pos, uint64_t epoch, int j, int k) {
  if (D.mode == WV_PAIRS_NATIVE) {
    uint32_t rnd[4] = {(uint32_t)pos, (uint32_t)((uint64_t)pos >> 32), (uint32_t)epoch, (uint32_t)(j >> 1)};
    philox4x32_10(rnd, (uint32_t)D.seed ^ 0xA5A5F00Du, (uint32_t)(D.seed >> 32) ^ 0x3C6EF372u);
    const uint64_t r64 = ((uint64_t)rnd[2 * (j & 1) + 1] << 32) | rnd[2 * (j & 1)];
    const int64_t ci = (int64_t)mulhi64(r64, (uint64_t)D.n_candidates);
    return D.candidates ? D.candidates[ci] : (int32_t)ci;
  }
  return D.negatives[pos * k + j];
}

// permuted position -> (centre, context): native mode walks Feistel position ->
// length class -> walk -> window slot (the reference's shift-major pair order,
// w2v.py:177-190); explicit mode reads pairs[perm[pos]].  ``q`` = the pair index.
__device__ __forceinline__ int64_t decode_pair(const CorpusDesc& D, const Feistel& fs, int64_t pos, int32_t& center,
                                               int32_t& context) {
  if (D.mode == WV_PAIRS_NATIVE) {
    const int64_t q = (int64_t)feistel_perm(fs, (uint64_t)pos, D.N);
    int lo_c = 0, hi_c = D.n_classes;  // last class with start <= q
    while (hi_c - lo_c > 1) {
      int mid = (lo_c + hi_c) >> 1;
      if (D.class_pair_start[mid] <= q) lo_c = mid; else hi_c = mid;
    }
    const int64_t L = D.class_len[lo_c];
    const int64_t np = walk_pairs(L, D.window);
    const int64_t r = q - D.class_pair_start[lo_c];
    const int64_t wslot = r / np;
    const int64_t local = r - wslot * np;
    const int64_t walk = D.walks_by_class[D.class_walk_start[lo_c] + wslot];
    int64_t cpos, xpos;
    walk_pair_pos(L, D.window, local, cpos, xpos);
    const int64_t base = D.offsets[walk];
    center = D.tokens[base + cpos];
    context = D.tokens[base + xpos];
    return q;
  }
  const int64_t pi = D.perm[pos];
  center = D.pairs[2 * pi];
  context = D.pairs[2 * pi + 1];
  return pi;
}

// test/inspection entry (wv_sgns_decode): positions [pos0, pos0 + n) of one
// epoch -> rows [n, 2 + k] (centre, context, negatives) and the pair index q
__global__ void sgns_decode_positions(CorpusDesc D, int k, int64_t epoch, int64_t pos0, int64_t n,
                                      int32_t* __restrict__ rows, int64_t* __restrict__ qout) {
  Feistel fs;
  if (D.mode == WV_PAIRS_NATIVE) fs = make_feistel(D.seed, (uint64_t)epoch, D.N);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = pos0 + i;
    int32_t c, x;
    const int64_t q = decode_pair(D, fs, pos, c, x);
    int32_t* row = rows + i * (2 + k);
    row[0] = c;
    row[1] = x;
    for (int j = 0; j < k; ++j) row[2 + j] = draw_negative(D, pos, (uint64_t)epoch, j, k);
    if (qout) qout[i] = q;
  }
}

__global__ void __launch_bounds__(128) sgns_decode_kernel(PairArgs A) {
  __shared__ CorpusDesc D;
  if (threadIdx.x == 0) D = *A.desc;
  __syncthreads();
  const int k = A.k;
  const int R = 2 + k;
  const int64_t B = A.B;
  // work items: [0, B) decode pair b (centre + context); [B, B + Bk) draw
  // negative j of pair b.  The two kinds never share a warp except at the one
  // boundary, so the long pair-decode chains do not hold the negatives' lanes.
  const int64_t items = B * (1 + k);
  const int64_t lo = A.state->lo;
  const uint64_t epoch = (uint64_t)A.state->epoch;
  Feistel fs;
  if (D.mode == WV_PAIRS_NATIVE) fs = make_feistel(D.seed, epoch, D.N);
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    if (it < B) {
      const int64_t b = it;
      const int64_t pos = lo + b;
      int32_t* row = A.idx + b * R;
      int32_t center, context;
      decode_pair(D, fs, pos, center, context);
      row[0] = center;
      row[1] = context;
      group_claim(A, (uint32_t)center, b * R);
      group_claim(A, (uint32_t)(context + A.V), b * R + 1);
    } else {
      const int64_t t = it - B;
      const int64_t b = t / k;
      const int j = (int)(t - b * k);
      const int64_t pos = lo + b;
      const int32_t neg = draw_negative(D, pos, epoch, j, k);
      A.idx[b * R + 2 + j] = neg;
      group_claim(A, (uint32_t)(neg + A.V), b * R + 2 + j);
    }
  }
}

// CBOW decode, thread per item: items 0..2W-1 are the instance's context rows
// (input side, -1 outside the walk), 2W the target and 2W+1.. the negatives
// (output side); the instance is instances[perm(position)].
__global__ void __launch_bounds__(128) cbow_decode_kernel(PairArgs A) {
  __shared__ CorpusDesc D;
  if (threadIdx.x == 0) D = *A.desc;
  __syncthreads();
  const int k = A.k;
  const int R = A.R;
  const int ctxw = 2 * A.cw;
  const int64_t items = A.B * R;
  const int64_t lo = A.state->lo;
  const uint64_t epoch = (uint64_t)A.state->epoch;
  Feistel fs;
  if (D.mode == WV_PAIRS_NATIVE) fs = make_feistel(D.seed, epoch, D.N);
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = it / R;
    const int jj = (int)(it - b * R);
    const int64_t pos = lo + b;
    int32_t* row = A.idx + b * R;
    if (jj <= ctxw) {
      const int64_t q = D.mode == WV_PAIRS_NATIVE ? (int64_t)feistel_perm(fs, (uint64_t)pos, D.N) : D.perm[pos];
      const int32_t t = D.inst[q * (ctxw + 1) + jj];
      row[jj] = t;
      if (t >= 0) group_claim(A, (uint32_t)t + (jj == ctxw ? (uint32_t)A.V : 0u), it);
    } else {
      const int32_t neg = draw_negative(D, pos, epoch, jj - ctxw - 1, k);
      row[jj] = neg;
      group_claim(A, (uint32_t)(neg + A.V), it);
    }
  }
}

// ------------------------------------------------ bulk-copy (TMA) gather --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// one row, global -> shared, completion counted on `bar` (cp.async.bulk -> UBLKCP)
__device__ __forceinline__ void bulk_row_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
#ifndef WV_GATHER_EVICT_LAST
#define WV_GATHER_EVICT_LAST 1  // owner 151.6 -> 143.0 us, gather 44.2 -> 48.2 us, step +2.8 %
#endif
#ifndef WV_GATHER_KEEP_FRAC
#define WV_GATHER_KEEP_FRAC 1.0  // fraction of the copied lines marked evict-last
#endif
#define WV_STR2(x) #x
#define WV_STR(x) WV_STR2(x)
// Same copy with an L2 evict-last policy: the parameter rows a batch gathers are
// read again by that batch's RowAdam owner.
__device__ __forceinline__ void bulk_row_g2s_keep(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, " WV_STR(WV_GATHER_KEEP_FRAC) ";" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <typename T>
__device__ __forceinline__ T log1pexp_t(T x);
template <>
__device__ __forceinline__ double log1pexp_t<double>(double x) { return log1pexp(x); }
template <>
__device__ __forceinline__ float log1pexp_t<float>(float x) { return x > 0.f ? x + log1pf(__expf(-x)) : log1pf(__expf(x)); }

#ifndef WV_SHARED_EXP
#define WV_SHARED_EXP 1
#endif
// Loss term log(1 + e^x) of one dot (x = -dot for the positive, +dot for a
// negative; w2v.py:262-273) and sigmoid(dot) (w2v.py:242-244).  float64 shares
// one exp(-|dot|) between them: the loss term is bit-identical to log1pexp, and
// the sigmoid is 1 / (1 + e) for dot >= 0 (bit-identical to the reference's
// 1 / (1 + exp(-dot))) and e / (1 + e) below (within an ulp of it).
template <typename T>
__device__ __forceinline__ T loss_sigmoid(T dot, bool positive, double& loss) {
  if constexpr (sizeof(T) == 8 && WV_SHARED_EXP) {
    const double e = exp(-fabs(dot));
    const double x = positive ? -dot : dot;
    loss += (x > 0 ? x : 0.0) + log1p(e);
    return dot >= 0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
  } else {
    loss += (double)log1pexp_t<T>(positive ? -dot : dot);
    return T(1) / (T(1) + exp_t(-dot));
  }
}

// Batch loss of one block -> partials; the last block to finish folds the
// partials in block order (deterministic) into the device state.
__device__ __forceinline__ void finish_batch_loss(const PairArgs& A, double block_sum) {
  __shared__ bool is_last;
  if (threadIdx.x == 0) {
    A.partials[blockIdx.x] = block_sum;
    __threadfence();
    const unsigned done = atomicAdd(&A.state->block_counter, 1u);
    is_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) {
    __threadfence();
    double s = 0;
    for (unsigned i = 0; i < gridDim.x; ++i) s += ((volatile double*)A.partials)[i];
    WvSgnsDevState* st = A.state;
    st->block_counter = 0;
    const double batch_loss = s / (double)A.B;
    if (!isfinite(batch_loss) && st->diverged_batch < 0) {
      st->diverged_batch = st->batch;
      st->diverged_epoch = st->epoch;
    }
    st->epoch_loss_sum += batch_loss * (double)A.B;
    st->epoch_count += A.B;
    st->last_batch_loss = batch_loss;
  }
}

#ifndef WV_GATHER_WARPS
#define WV_GATHER_WARPS 8
#endif
#ifndef WV_GATHER_WARPS_WIDE
// wide rows (fp64 d 200): 10 warps x 2 stages = 224 KB ring.  The gather is bound by the
// latency of its dependent float64 chains (dots, butterfly, exp, divide), so warps beat
// stages: ncu alone 76 -> 50 us (4.9 TB/s) vs 5 x 3, step +0.9 % (r02x); 4 x 3: 88 us
#define WV_GATHER_WARPS_WIDE 10
#endif
#ifndef WV_GATHER_WARPS_WIDE2
#define WV_GATHER_WARPS_WIDE2 5  // fallback ring when 10 x 2 does not fit (larger k or d): 5 x 3
#endif
#ifndef WV_GATHER_PREFETCH
#define WV_GATHER_PREFETCH 0  // pairs (per warp, in ring steps) whose rows are L2-prefetched ahead of their copies
#endif
#ifndef WV_GATHER_STAGES
#define WV_GATHER_STAGES 3  // 3 x 8 warps: one 134 KB CTA per SM leaves room for the side stream (+2.7 % vs 2 x 8)
#endif
constexpr int kBulkWarps = WV_GATHER_WARPS;
constexpr int kBulkWarpsWide = WV_GATHER_WARPS_WIDE;
#ifndef WV_GATHER_STAGES_WIDE
#define WV_GATHER_STAGES_WIDE 2
#endif
constexpr int kBulkStagesWide = WV_GATHER_STAGES_WIDE;
constexpr int kBulkWarpsWide2 = WV_GATHER_WARPS_WIDE2;
constexpr int kBulkStagesWide2 = 3;
constexpr int kBulkStages = WV_GATHER_STAGES;  // pairs in flight per warp

// Phase 1b (default path): warp per pair with the 2+k rows fetched by
// cp.async.bulk into a per-warp two-stage shared-memory ring.  Lane j issues
// row j's copy, so the whole pair (7 x 800 B at d=200) is in flight at once
// and the next pair's rows land while this pair computes; no row data is held
// in registers across the wait, which keeps occupancy up.  Lanes 0..k each
// evaluate one loss term (the reference's float64 logaddexp, w2v.py:262-273).
// CB = CBOW (w2v.py:302-361): the item is an instance whose up-to-2W context
// rows are averaged into u = c (the masked mean), its target row takes the
// positive logit, and the input-side gradient is grad_c / len.
// KC > 0: the negative count is a compile-time constant (KC + 1 <= 8 dots):
// the 1 + KC output rows are loaded from shared memory once into registers
// and reused by the dots and the gradient row.
template <typename T, int EPC, int MAXC, bool CB, int NW, int KC, int ST>
__global__ void __launch_bounds__(NW * 32) sgns_gather_bulk_kernel(PairArgs A, const T* __restrict__ in,
                                                                    const T* __restrict__ out) {
  constexpr int kBulkWarps = NW;
  constexpr int kBulkStages = ST;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = A.d, k = A.k;
  const int R = CB ? A.R : 2 + k;
  const int ctxw = CB ? 2 * A.cw : 1;  // input-side rows per item; the positive output row follows them
  const int C = d / EPC;
  const int64_t B = A.B;
  const uint32_t row_bytes = (uint32_t)(d * sizeof(T));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);  // [warps][kBulkStages]
  T* ring = reinterpret_cast<T*>(smem_raw + 16 * kBulkWarps * kBulkStages) + (size_t)warp * kBulkStages * R * d;
  uint64_t* mybar = bars + kBulkStages * warp;
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < kBulkStages; ++st) mbar_init(mybar + st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  T* U = (T*)A.U;
  T* G = (T*)A.G;
  T* coef = (T*)A.coef;
  const T invB = (T)1 / (T)(A.Bn > 0 ? A.Bn : B);
  const int64_t stride = (int64_t)gridDim.x * kBulkWarps;
  int64_t b = blockIdx.x * (int64_t)kBulkWarps + warp;
  auto row_of = [&](int64_t pb) -> int32_t { return (lane < R && pb < B) ? __ldg(A.idx + pb * R + lane) : -1; };
  auto issue = [&](int64_t pb, int stage, int32_t r) {
    T* dst = ring + (size_t)stage * R * d;
    const uint32_t valid = __ballot_sync(0xffffffffu, lane < R && r >= 0);  // CBOW: masked context columns
    if (lane == 0) mbar_arrive_expect_tx(mybar + stage, row_bytes * (uint32_t)__popc(valid));
    __syncwarp();
    if ((valid >> lane) & 1u) {
      const T* src = (lane < ctxw ? in : out) + (int64_t)r * d;
      if (WV_GATHER_EVICT_LAST)
        bulk_row_g2s_keep(dst + (size_t)lane * d, src, row_bytes, mybar + stage);
      else
        bulk_row_g2s(dst + (size_t)lane * d, src, row_bytes, mybar + stage);
    }
  };
  // prologue: the first kBulkStages - 1 pairs
#pragma unroll
  for (int st = 0; st < kBulkStages - 1; ++st)
    if (b + st * stride < B) issue(b + st * stride, st, row_of(b + st * stride));
  double loss_acc = 0.0;
  uint32_t phase = 0u;  // bit per stage
  // row indices of the next pair to issue, loaded one iteration ahead so the
  // copies are issued without waiting on the index load
  int32_t r_next = row_of(b + (int64_t)(kBulkStages - 1) * stride);
  for (int it = 0; b < B; ++it, b += stride) {
    const int stage = it % kBulkStages;
    const int64_t nb = b + (int64_t)(kBulkStages - 1) * stride;
    if (nb < B) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(nb, (it + kBulkStages - 1) % kBulkStages, r_next);
    }
    r_next = row_of(nb + stride);
    if constexpr (WV_GATHER_PREFETCH > 0) {
      // L2 prefetch of a pair further ahead: more bytes in flight than the ring's shared memory holds
      const int64_t pf = nb + (int64_t)WV_GATHER_PREFETCH * stride;
      const int32_t rp = row_of(pf);
      if (rp >= 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((lane < ctxw ? in : out) + (int64_t)rp * d),
                     "r"(row_bytes)
                     : "memory");
    }
    while (!mbar_try_wait(mybar + stage, (phase >> stage) & 1u)) {
    }
    phase ^= 1u << stage;
    const T* rows = ring + (size_t)stage * R * d;
    Chunk<T, EPC> u[MAXC];
    T len_t = 1;
    if constexpr (CB) {
      // c = masked mean of the context rows, summed in column order (w2v.py:308)
      const int32_t t = lane < ctxw ? __ldg(A.idx + b * R + lane) : -1;
      const uint32_t cm = __ballot_sync(0xffffffffu, t >= 0);
      const T len = (T)__popc(cm);
      len_t = len;
#pragma unroll
      for (int q = 0; q < MAXC; ++q) {
        const int c = lane + 32 * q;
#pragma unroll
        for (int e = 0; e < EPC; ++e) u[q].v[e] = 0;
        if (c < C) {
          for (int j = 0; j < ctxw; ++j)
            if ((cm >> j) & 1u) {
              const Chunk<T, EPC> x = *reinterpret_cast<const Chunk<T, EPC>*>(rows + (size_t)j * d + c * EPC);
#pragma unroll
              for (int e = 0; e < EPC; ++e) u[q].v[e] = add_rn(u[q].v[e], x.v[e]);
            }
#pragma unroll
          for (int e = 0; e < EPC; ++e) u[q].v[e] = div_rn(u[q].v[e], len);
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < MAXC; ++q) {
        const int c = lane + 32 * q;
        if (c < C) u[q] = *reinterpret_cast<const Chunk<T, EPC>*>(rows + c * EPC);
      }
    }
    if constexpr (KC > 0) {
      Chunk<T, EPC> x[KC + 1][MAXC];
#pragma unroll
      for (int t = 0; t <= KC; ++t)
#pragma unroll
        for (int q = 0; q < MAXC; ++q) {
          const int c = lane + 32 * q;
          if (c < C) x[t][q] = *reinterpret_cast<const Chunk<T, EPC>*>(rows + (size_t)(ctxw + t) * d + c * EPC);
        }
      T part[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        part[t] = 0;
        if (t <= KC) {
#pragma unroll
          for (int q = 0; q < MAXC; ++q) {
            const int c = lane + 32 * q;
            if (c < C) {
#pragma unroll
              for (int e = 0; e < EPC; ++e) part[t] += u[q].v[e] * x[t][q].v[e];
            }
          }
        }
      }
      const T red = warp_sum8(part);  // dot ((lane >> 2) & 7)
      const T mydot = __shfl_sync(0xffffffffu, red, (lane & 7) << 2);
      T mycoef = 0;
      if (lane <= KC) {
        const T sg = loss_sigmoid<T>(mydot, lane == 0, loss_acc);
        mycoef = (lane == 0 ? sg - T(1) : sg) * invB;
        coef[b * (KC + 1) + lane] = mycoef;
      }
      T cf[KC + 1];
#pragma unroll
      for (int j = 0; j <= KC; ++j) cf[j] = __shfl_sync(0xffffffffu, mycoef, j);
#pragma unroll
      for (int q = 0; q < MAXC; ++q) {
        const int c = lane + 32 * q;
        if (c < C) {
          Chunk<T, EPC> gg;
#pragma unroll
          for (int e = 0; e < EPC; ++e) {
            T acc = 0;
#pragma unroll
            for (int j = 1; j <= KC; ++j) acc = mad_t(cf[j], x[j][q].v[e], acc);
            gg.v[e] = mad_t(cf[0], x[0][q].v[e], acc);
          }
          st_chunk<T, EPC>(G + b * d + c * EPC, gg);
          st_chunk<T, EPC>(U + b * d + c * EPC, u[q]);
        }
      }
      __syncwarp();
      continue;
    }
    // dot j = <u, row ctxw+j> (j = 0: context / target, j >= 1: negative j-1),
    // eight at a time through one transposed butterfly; lane j ends up holding dot j
    T mydot = 0;
    for (int j0 = 0; j0 <= k; j0 += 8) {
      T part[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        part[t] = 0;
        if (j0 + t <= k) {
          const T* rj = rows + (size_t)(ctxw + j0 + t) * d;
#pragma unroll
          for (int q = 0; q < MAXC; ++q) {
            const int c = lane + 32 * q;
            if (c < C) {
              const Chunk<T, EPC> x = *reinterpret_cast<const Chunk<T, EPC>*>(rj + c * EPC);
#pragma unroll
              for (int e = 0; e < EPC; ++e) part[t] += u[q].v[e] * x.v[e];
            }
          }
        }
      }
      const T red = warp_sum8(part);  // dot j0 + ((lane >> 2) & 7)
      const T got = __shfl_sync(0xffffffffu, red, (lane & 7) << 2);
      if (lane >= j0 && lane < j0 + 8) mydot = got;
    }
    // lane j: loss term and coefficient of dot j
    T mycoef = 0;
    if (lane <= k) {
      const T sg = loss_sigmoid<T>(mydot, lane == 0, loss_acc);
      mycoef = (lane == 0 ? sg - T(1) : sg) * invB;
      coef[b * (k + 1) + lane] = mycoef;
    }
    const T gpos = __shfl_sync(0xffffffffu, mycoef, 0);
#pragma unroll
    for (int q = 0; q < MAXC; ++q) {
      const int c = lane + 32 * q;
      Chunk<T, EPC> acc;
#pragma unroll
      for (int e = 0; e < EPC; ++e) acc.v[e] = 0;
      for (int j = 1; j <= k; ++j) {
        const T gneg = __shfl_sync(0xffffffffu, mycoef, j);
        if (c < C) {
          const Chunk<T, EPC> x =
              *reinterpret_cast<const Chunk<T, EPC>*>(rows + (size_t)(ctxw + j) * d + c * EPC);
#pragma unroll
          for (int e = 0; e < EPC; ++e) acc.v[e] = mad_t(gneg, x.v[e], acc.v[e]);
        }
      }
      if (c < C) {
        const Chunk<T, EPC> v = *reinterpret_cast<const Chunk<T, EPC>*>(rows + (size_t)ctxw * d + c * EPC);
        Chunk<T, EPC> gg;
#pragma unroll
        for (int e = 0; e < EPC; ++e) gg.v[e] = mad_t(gpos, v.v[e], acc.v[e]);
        if constexpr (CB) {
          // per-context-token share grad_c / len (w2v.py:356)
#pragma unroll
          for (int e = 0; e < EPC; ++e) gg.v[e] = div_rn(gg.v[e], len_t);
        }
        st_chunk<T, EPC>(G + b * d + c * EPC, gg);
        st_chunk<T, EPC>(U + b * d + c * EPC, u[q]);
      }
    }
    __syncwarp();
  }
  // block loss: lanes -> warp -> block (fixed order)
  loss_acc = warp_sum(loss_acc);
  __shared__ double wl[kBulkWarps];
  if (lane == 0) wl[warp] = loss_acc;
  __syncthreads();
  double blk = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kBulkWarps; ++w) blk += wl[w];
  finish_batch_loss(A, blk);
}

// Phase 1b, warp per pair: gather the 2+k rows with 16-byte loads -- every
// load of a negative group is issued before the first dot product so each
// lane keeps several independent row chunks in flight -- then the (1+k) dots
// (warp shuffles), the loss, the per-pair coefficients and two [B,d] rows:
// the centre row u and its gradient g_u = gpos v + sum_j gneg_j n_j.
template <typename T, int EPC, int MAXC, int NG>
__global__ void __launch_bounds__(kPairThreads) sgns_gather_kernel(PairArgs A, const T* __restrict__ in,
                                                                     const T* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = A.d, k = A.k;
  const int C = d / EPC;
  const int64_t B = A.B;
  T* U = (T*)A.U;
  T* G = (T*)A.G;
  T* coef = (T*)A.coef;
  const T invB = (T)1 / (T)B;
  double loss_acc = 0.0;
  for (int64_t b = blockIdx.x * (int64_t)kPairWarps + warp; b < B; b += (int64_t)gridDim.x * kPairWarps) {
    const int32_t my = lane < 2 + k ? __ldg(A.idx + b * (2 + k) + lane) : 0;
    const int32_t center = __shfl_sync(0xffffffffu, my, 0);
    const int32_t context = __shfl_sync(0xffffffffu, my, 1);
    const T* urow = in + (int64_t)center * d;
    const T* vrow = out + (int64_t)context * d;
    Chunk<T, EPC> u[MAXC], g[MAXC], nv[NG][MAXC];
    const int g0 = k < NG ? k : NG;
#pragma unroll
    for (int q = 0; q < MAXC; ++q) {
      const int c = lane + 32 * q;
      if (c < C) {
        u[q] = ld_chunk<T, EPC>(urow + c * EPC);
        g[q] = ld_chunk<T, EPC>(vrow + c * EPC);
      }
    }
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const int32_t nj = __shfl_sync(0xffffffffu, my, 2 + j);
      if (j < g0) {
        const T* nrow = out + (int64_t)nj * d;
#pragma unroll
        for (int q = 0; q < MAXC; ++q) {
          const int c = lane + 32 * q;
          if (c < C) nv[j][q] = ld_chunk<T, EPC>(nrow + c * EPC);
        }
      }
    }
    T dot = 0;
#pragma unroll
    for (int q = 0; q < MAXC; ++q) {
      const int c = lane + 32 * q;
      if (c < C) {
#pragma unroll
        for (int e = 0; e < EPC; ++e) dot += u[q].v[e] * g[q].v[e];
      }
    }
    const T pos_logit = warp_sum(dot);
    double l = log1pexp(-(double)pos_logit);
    const T gpos = (T(1) / (T(1) + exp_t(-pos_logit)) - T(1)) * invB;
    if (lane == 0) coef[b * (k + 1)] = gpos;
#pragma unroll
    for (int q = 0; q < MAXC; ++q) {
      const int c = lane + 32 * q;
      if (c < C) {
#pragma unroll
        for (int e = 0; e < EPC; ++e) g[q].v[e] = mul_rn(gpos, g[q].v[e]);
      }
    }
    Chunk<T, EPC> acc[MAXC];
#pragma unroll
    for (int q = 0; q < MAXC; ++q)
#pragma unroll
      for (int e = 0; e < EPC; ++e) acc[q].v[e] = 0;
    for (int j0 = 0; j0 < k; j0 += NG) {
      const int gn = k - j0 < NG ? k - j0 : NG;
      if (j0 > 0) {  // later negative groups (k > NG): issue the whole group, then reduce
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          const int32_t nj = __shfl_sync(0xffffffffu, my, 2 + ((j0 + j) < k ? j0 + j : 0));
          if (j < gn) {
            const T* nrow = out + (int64_t)nj * d;
#pragma unroll
            for (int q = 0; q < MAXC; ++q) {
              const int c = lane + 32 * q;
              if (c < C) nv[j][q] = ld_chunk<T, EPC>(nrow + c * EPC);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        if (j < gn) {
          T nd = 0;
#pragma unroll
          for (int q = 0; q < MAXC; ++q) {
            const int c = lane + 32 * q;
            if (c < C) {
#pragma unroll
              for (int e = 0; e < EPC; ++e) nd += u[q].v[e] * nv[j][q].v[e];
            }
          }
          const T neg_logit = warp_sum(nd);
          l += log1pexp((double)neg_logit);
          const T gneg = (T(1) / (T(1) + exp_t(-neg_logit))) * invB;
#pragma unroll
          for (int q = 0; q < MAXC; ++q) {
            const int c = lane + 32 * q;
            if (c < C) {
#pragma unroll
              for (int e = 0; e < EPC; ++e) acc[q].v[e] = add_rn(acc[q].v[e], mul_rn(gneg, nv[j][q].v[e]));
            }
          }
          if (lane == 0) coef[b * (k + 1) + 1 + j0 + j] = gneg;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < MAXC; ++q) {
      const int c = lane + 32 * q;
      if (c < C) {
        Chunk<T, EPC> gg;
#pragma unroll
        for (int e = 0; e < EPC; ++e) gg.v[e] = add_rn(g[q].v[e], acc[q].v[e]);
        st_chunk<T, EPC>(G + b * d + c * EPC, gg);
        st_chunk<T, EPC>(U + b * d + c * EPC, u[q]);
      }
    }
    loss_acc += l;  // identical on all lanes
  }

  // deterministic batch-loss reduction: per-block partial, last block sums
  __shared__ double wl[kPairWarps];
  __shared__ bool is_last;
  if (lane == 0) wl[warp] = loss_acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int w = 0; w < kPairWarps; ++w) s += wl[w];
    A.partials[blockIdx.x] = s;
    __threadfence();
    unsigned done = atomicAdd(&A.state->block_counter, 1u);
    is_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) {
    __threadfence();
    double s = 0;
    for (unsigned i = 0; i < gridDim.x; ++i) s += ((volatile double*)A.partials)[i];
    WvSgnsDevState* st = A.state;
    st->block_counter = 0;
    const double batch_loss = s / (double)B;
    if (!isfinite(batch_loss) && st->diverged_batch < 0) {
      st->diverged_batch = st->batch;
      st->diverged_epoch = st->epoch;
    }
    st->epoch_loss_sum += batch_loss * (double)B;
    st->epoch_count += B;
    st->last_batch_loss = batch_loss;
  }
}

// Rows with more than kLightMax contributions in a batch (predicates, hub
// entities) go to the CTA-per-row kernel; the rest to the warp-per-row one.
#ifndef WV_LIGHT_MAX
#define WV_LIGHT_MAX 16  // contributions of a light row; more go through the heavy pieces
#endif
constexpr int kLightMax = WV_LIGHT_MAX;
constexpr int kHeavyThreads = 256;
constexpr int kHeavyGroup = 8;            // rows loaded together per warp in the heavy kernel
constexpr int64_t kBitmapMaxWords = 12288;  // slot bitmap in shared memory: batches up to 393,216 items
__host__ __device__ __forceinline__ uint32_t heavy_bitmap_words(int64_t items) {
  const int64_t w = (items + 31) / 32;
  return w <= kBitmapMaxWords ? (uint32_t)w : 0u;
}

// One record per unique (matrix, row) of the batch, built by group_segments.
struct Segment {
  uint32_t start;  // first entry of the row's slot list
  uint32_t len;    // contributions
  uint32_t key;    // row key (input row r, or V + output row r)
  uint32_t pad;
  double bc1;      // Adam bias corrections 1 - b1^t, 1 - b2^t with the row's new step t
  double bc2;      // (their reciprocals under WV_FP64_RCP: bias_corr)
};

// RowAdam bias corrections 1 - b1^t, 1 - b2^t for t < kBcTable, computed once
// per device with the same pow as the fallback (a table load replaces two
// float64 pow calls per unique row)
constexpr int kBcTable = 1 << 16;
// 1 - b^t (w2v.py:386-387), or its reciprocal under WV_FP64_RCP (see AdamBC)
__device__ __forceinline__ double bias_corr(double b, int t) {
  const double c = 1.0 - pow(b, (double)t);
  return WV_FP64_RCP ? 1.0 / c : c;
}
__global__ void fill_bc_table(double2* tab) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < kBcTable) tab[t] = make_double2(bias_corr(0.9, t), bias_corr(0.999, t));
}

__global__ void group_segments(const uint32_t* __restrict__ uniq, uint32_t* __restrict__ cnt, uint32_t* gctr,
                               int64_t V, int sparse, int32_t* __restrict__ steps_in, int32_t* __restrict__ steps_out,
                               Segment* __restrict__ segs, Segment* __restrict__ heavy, int64_t max_unique,
                               WvSgnsDevState* state, int64_t B, const double2* __restrict__ bc_table,
                               Segment* __restrict__ singles) {
  const int lane = threadIdx.x & 31;
  // the batch's pairs are decoded: advance the decode cursor for the next batch
  if (blockIdx.x == 0 && threadIdx.x == 0) state->lo += B;
  const uint32_t nu = *(volatile uint32_t*)(gctr + GC_UNIQUE);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < nu && base < max_unique; base += stride) {
    const int64_t u = base + threadIdx.x;
    const bool ok = u < nu;
    const uint32_t key = ok ? uniq[u] : 0u;
    const uint32_t len = ok ? cnt[key] : 0u;
    // block-aggregated reservations: one atomic per block and counter (the
    // three counters are single addresses every block contends on)
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += n;
    }
    const bool is_heavy = ok && len > (uint32_t)kLightMax;
    const bool is_single = singles != nullptr && ok && len == 1u;  // the lean single-contribution owner
    const uint32_t ml = __ballot_sync(0xffffffffu, ok && !is_heavy && !is_single);
    const uint32_t mh = __ballot_sync(0xffffffffu, is_heavy);
    const uint32_t ms = __ballot_sync(0xffffffffu, is_single);
    __shared__ uint32_t wsum[4][32];
    __shared__ uint32_t bbase[4];
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    if (lane == 31) {
      wsum[0][warp] = incl;
      wsum[1][warp] = __popc(ml);
      wsum[2][warp] = __popc(mh);
      wsum[3][warp] = __popc(ms);
    }
    __syncthreads();
    if (threadIdx.x < 4) {
      uint32_t run = 0;
      for (int w = 0; w < nwarps; ++w) {
        const uint32_t v = wsum[threadIdx.x][w];
        wsum[threadIdx.x][w] = run;
        run += v;
      }
      const int ctr = threadIdx.x == 0 ? GC_TOTAL : threadIdx.x == 1 ? GC_LIGHT : threadIdx.x == 2 ? GC_HEAVY
                                                                                                   : GC_SINGLE;
      bbase[threadIdx.x] = run ? atomicAdd(gctr + ctr, run) : 0u;
    }
    __syncthreads();
    const uint32_t start = bbase[0] + wsum[0][warp] + incl - len;
    const uint32_t lb = bbase[1] + wsum[1][warp];
    const uint32_t hb = bbase[2] + wsum[2][warp];
    const uint32_t sb = bbase[3] + wsum[3][warp];
    __syncthreads();  // wsum / bbase are rewritten by the next iteration
    if (ok) {
      cnt[key] = start;  // becomes the placement cursor
      Segment sg;
      sg.start = start;
      sg.len = len;
      sg.key = key;
      sg.pad = 0;
      sg.bc1 = sg.bc2 = 1.0;
      if (sparse) {
        const bool side_out = key >= (uint32_t)V;
        int32_t* steps = side_out ? steps_out : steps_in;
        const int64_t row = side_out ? (int64_t)key - V : (int64_t)key;
        const int t = steps[row] + 1;
        steps[row] = t;
        if (t < kBcTable) {
          const double2 bc = bc_table[t];
          sg.bc1 = bc.x;
          sg.bc2 = bc.y;
        } else {
          sg.bc1 = bias_corr(0.9, t);
          sg.bc2 = bias_corr(0.999, t);
        }
      }
      const uint32_t below = (1u << lane) - 1u;
      if (is_heavy)
        heavy[hb + __popc(mh & below)] = sg;
      else if (is_single)
        singles[sb + __popc(ms & below)] = sg;
      else
        segs[lb + __popc(ml & below)] = sg;
    }
  }
}

// every item appends its slot to its row's list
// Slots (the order np.add.at applies contributions, w2v.py:407-416):
//   skip-gram: centre b -> b; context b -> B + b; negative j -> 2B + bk + j
//   CBOW     : context column c of instance b -> b*2W + c (input side);
//              target b -> b; negative j -> B + bk + j (output side)
// so an output slot minus out_base (B for skip-gram, 0 for CBOW) is < B for
// the positive row and B + bk + j for negative j in both models.
__global__ void group_place(const int32_t* __restrict__ idx, int64_t B, int k, int R, int cw, int64_t V,
                            uint32_t* __restrict__ cnt, uint32_t* __restrict__ list) {
  const int64_t items = B * R;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < items; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / R;
    const int j = (int)(i - b * R);
    const int32_t t = idx[i];
    uint32_t key, slot;
    if (cw == 0) {
      key = (uint32_t)t + (j == 0 ? 0u : (uint32_t)V);
      slot = (uint32_t)(j == 0 ? b : (j == 1 ? B + b : 2 * B + b * k + (j - 2)));
    } else {
      if (t < 0) continue;  // context column outside the walk
      const int ctxw = 2 * cw;
      key = (uint32_t)t + (j < ctxw ? 0u : (uint32_t)V);
      slot = (uint32_t)(j < ctxw ? b * ctxw + j : (j == ctxw ? b : B + b * k + (j - ctxw - 1)));
    }
    list[atomicAdd(cnt + key, 1u)] = slot;
  }
}

// group_place with the atomics of equal keys inside a warp merged (hot rows:
// predicates and hubs take ~100 contributions per batch): one atomic per
// distinct key per warp, lanes take consecutive list positions
__global__ void group_place_agg(const int32_t* __restrict__ idx, int64_t B, int k, int R, int cw, int64_t V,
                                uint32_t* __restrict__ cnt, uint32_t* __restrict__ list, int nshard, int shard,
                                int64_t Vl) {
  const int64_t items = B * R;
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < items; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    uint32_t key = 0xffffffffu, slot = 0;
    if (i < items) {
      const int64_t b = i / R;
      const int j = (int)(i - b * R);
      const int32_t t = idx[i];
      if (cw == 0) {
        key = (uint32_t)t + (j == 0 ? 0u : (uint32_t)V);
        slot = (uint32_t)(j == 0 ? b : (j == 1 ? B + b : 2 * B + b * k + (j - 2)));
      } else if (t >= 0) {
        const int ctxw = 2 * cw;
        key = (uint32_t)t + (j < ctxw ? 0u : (uint32_t)V);
        slot = (uint32_t)(j < ctxw ? b * ctxw + j : (j == ctxw ? b : B + b * k + (j - ctxw - 1)));
      }
    }
    if (key != 0xffffffffu && nshard > 1) {
      uint32_t lk;
      key = owned_key(key, V, nshard, shard, Vl, lk) ? lk : 0xffffffffu;
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    uint32_t pos = 0;
    if (lane == leader && key != 0xffffffffu) pos = atomicAdd(cnt + key, (uint32_t)__popc(peers));
    pos = __shfl_sync(0xffffffffu, pos, leader);
    if (key != 0xffffffffu) list[pos + rank] = slot;
  }
}

// every claimed item writes its slot at (row's list start + its claim rank):
// no atomics (group_segments turned cnt[key] into the list start)
__global__ void group_place_rank(const int32_t* __restrict__ idx, const uint32_t* __restrict__ rank, int64_t B, int k,
                                 int R, int cw, int64_t V, const uint32_t* __restrict__ cnt,
                                 uint32_t* __restrict__ list, int nshard, int shard, int64_t Vl) {
  const int64_t items = B * R;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < items; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / R;
    const int j = (int)(i - b * R);
    const int32_t t = idx[i];
    uint32_t key, slot;
    if (cw == 0) {
      key = (uint32_t)t + (j == 0 ? 0u : (uint32_t)V);
      slot = (uint32_t)(j == 0 ? b : (j == 1 ? B + b : 2 * B + b * k + (j - 2)));
    } else {
      if (t < 0) continue;
      const int ctxw = 2 * cw;
      key = (uint32_t)t + (j < ctxw ? 0u : (uint32_t)V);
      slot = (uint32_t)(j < ctxw ? b * ctxw + j : (j == ctxw ? b : B + b * k + (j - ctxw - 1)));
    }
    if (nshard > 1) {
      uint32_t lk;
      if (!owned_key(key, V, nshard, shard, Vl, lk)) continue;
      key = lk;
    }
    list[cnt[key] + rank[i]] = slot;
  }
}

// Slot-to-source mapping parameters (skip-gram / CBOW).
struct SlotMap {
  uint32_t out_base;  // B (skip-gram) or 0 (CBOW)
  uint32_t in_div;    // input slot -> G row: slot / in_div (1 or 2W)
  uint32_t in_mag;    // ~2^32 / in_div
  uint32_t kmag;      // ~2^32 / k
};

__device__ __forceinline__ uint32_t div_mag(uint32_t t, uint32_t dv, uint32_t mag, int32_t& rem) {
  uint32_t q = __umulhi(t, mag);
  int32_t r = (int32_t)(t - q * dv);
  if (r < 0) {
    --q;
    r += (int32_t)dv;
  } else if (r >= (int32_t)dv) {
    ++q;
    r -= (int32_t)dv;
  }
  rem = r;
  return q;
}

static inline uint32_t host_mag(uint32_t dv) { return dv > 1 ? (uint32_t)(0xFFFFFFFFull / dv + 1ull) : 0xFFFFFFFFu; }

// Contribution slot -> (source U/G row, coefficient index); ci = 0xffffffff
// marks an input-side contribution (G row, coefficient 1).
__device__ __forceinline__ uint2 slot_entry(uint32_t v, bool side_out, int64_t B, int k, const SlotMap& sm) {
  int32_t r;
  if (!side_out) return make_uint2(sm.in_div == 1 ? v : div_mag(v, sm.in_div, sm.in_mag, r), 0xffffffffu);
  const uint32_t sv = v - sm.out_base;
  uint32_t pp, j;
  if (sv < (uint32_t)B) {
    pp = sv;
    j = 0;
  } else {
    pp = div_mag(sv - (uint32_t)B, (uint32_t)k, sm.kmag, r);
    j = 1 + (uint32_t)r;
  }
  return make_uint2(pp, pp * (uint32_t)(k + 1) + j);
}

// Light rows only: restore slot order inside each row's list (<= kLightMax
// entries, insertion sort in registers) and resolve every slot to its source
// (U/G row, coefficient index), so the owner's per-element threads walk a
// ready list.  Runs on the side stream with the grouping (off the critical
// path once batches are pipelined).  ci = 0xffffffff marks an input-side
// contribution (G row, coefficient 1).
__global__ void group_order(Segment* __restrict__ segs, const uint32_t* __restrict__ gctr,
                            const uint32_t* __restrict__ list, uint2* __restrict__ ents, int64_t V, int64_t B, int k,
                            SlotMap sm, Segment* __restrict__ singles) {
  if (singles != nullptr) {  // single-contribution rows: their one entry rides in the record
    const uint32_t ns = *(volatile const uint32_t*)(gctr + GC_SINGLE);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
      const Segment sg = singles[i];
      const uint2 e = slot_entry(list[sg.start], sg.key >= (uint32_t)V, B, k, sm);
      singles[i].start = e.x;
      singles[i].pad = e.y;
    }
  }
  const uint32_t nl = *(volatile const uint32_t*)(gctr + GC_LIGHT);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += gridDim.x * blockDim.x) {
    const Segment sg = segs[i];
    const bool side_out = sg.key >= (uint32_t)V;
    if (sg.len == 1) {  // the common case: the entry rides in the segment record (start, pad)
      const uint2 e = slot_entry(list[sg.start], side_out, B, k, sm);
      segs[i].start = e.x;
      segs[i].pad = e.y;
      continue;
    }
    uint32_t sl[kLightMax];
#pragma unroll
    for (int q = 0; q < kLightMax; ++q) sl[q] = q < (int)sg.len ? list[sg.start + q] : 0xffffffffu;
    // insertion sort (sentinels sort last)
#pragma unroll
    for (int q = 1; q < kLightMax; ++q) {
#pragma unroll
      for (int j = q; j > 0; --j) {
        const uint32_t a = sl[j - 1], b = sl[j];
        sl[j - 1] = min(a, b);
        sl[j] = max(a, b);
      }
    }
#pragma unroll
    for (int q = 0; q < kLightMax; ++q) {
      if (q >= (int)sg.len) break;
      ents[sg.start + q] = slot_entry(sl[q], side_out, B, k, sm);
    }
  }
}

struct OwnerArgs {
  int64_t V;
  int d;
  int k;
  int64_t B;
  int64_t n_items;
  const uint32_t* list;  // per-row slot lists (arbitrary order inside a row)
  uint32_t* list_tmp;    // scratch for the heavy rows' slot sort
  uint32_t* cnt;         // reset to 0 per row once consumed
  int slot_bits;         // bits of the largest slot (2B + Bk - 1)
  SlotMap sm;            // slot -> (source row, coefficient) mapping of the model
  uint32_t cmag;         // ~2^32 / (d / EPC) for the flat owner's (row, chunk) split
  const uint2* ents;     // slot-ordered (source row, coefficient index), from group_order / heavy_order
  const uint2* pieces;   // heavy-row pieces (row, piece index) from heavy_order
  void* partial;         // [pieces, d] piece partial sums
  uint32_t* rowdone;     // per heavy row: pieces finished (zeroed per batch)
  const uint32_t* gctr;  // grouping counters (GC_PIECES: piece count)
  const Segment* segs;
  const Segment* heavy;
  const Segment* singles;  // single-contribution light rows (count gctr[GC_SINGLE])
  const uint32_t* seg_count;  // [0] light segments, [1] heavy segments
  const uint32_t* seg_base;   // split owner: the launch's segments start at segs + *seg_base (null: 0)
  uint32_t piece;             // heavy-row piece size (contributions)
  int bookkeep;               // 1: this launch advances the batch counters (one launch per batch)
  uint8_t* flag;              // row-key membership flags of this batch, cleared per row (null: none)
  const void* U;
  const void* G;
  const void* coef;
  void* in;
  void* out;
  void* m_in;
  void* v_in;
  void* m_out;
  void* v_out;
  uint8_t* touched_in;
  uint8_t* touched_out;
  uint8_t* modified_in;
  uint8_t* modified_out;
  double lr;
  void* gsum;          // [items, d] per-segment gradient rows (split mode): light i at i, heavy h at items-1-h
  int split;           // 1: the owner kernels write gsum and sgns_adam_kernel applies RowAdam
  int sparse;          // 1: RowAdam sparse mode; 0: write dense gradient rows
  void* dense_g_in;    // dense mode gradient staging [V,d]
  void* dense_g_out;
  WvSgnsDevState* state;
};

// RowAdam element update (w2v.py:384-395): m, v recurrences, bias-corrected
// step.  float64 keeps numpy's exact operation order (correctly rounded
// divisions); the float32 store multiplies by the per-row reciprocals of the
// bias corrections and uses a fast divide (a few ulp; the fp32 store is
// tolerance-checked against the reference, not bit-checked).
// Per-row bias corrections in the form the element update consumes.  A row's
// segment record carries them as the grouping computed them once per unique
// row: with WV_FP64_RCP the reciprocals 1 / (1 - b^t) (multiplied by), else
// 1 - b^t (divided by, numpy's order).  float32 always multiplies.
template <typename T>
struct AdamBC {
#if WV_FP64_RCP
  double r1, r2;
  __device__ __forceinline__ AdamBC(double a, double b) : r1(a), r2(b) {}
#else
  double bc1, bc2;
  __device__ __forceinline__ AdamBC(double a, double b) : bc1(a), bc2(b) {}
#endif
};
template <>
struct AdamBC<float> {
  float r1, r2;
  __device__ __forceinline__ AdamBC(double a, double b) {
#ifdef __CUDA_ARCH__
#if WV_FP64_RCP
    r1 = (float)a;
    r2 = (float)b;
#else
    r1 = __frcp_rn((float)a);
    r2 = __frcp_rn((float)b);
#endif
#endif
  }
};

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// RowAdam element update (w2v.py:384-395): m, v recurrences, bias-corrected
// step.  float64 keeps numpy's operation order with correctly rounded
// operations and no FMA contraction; under WV_FP64_RCP the two bias-correction
// divisions become multiplications by per-row reciprocals (within an ulp each).  The float32 store uses FMAs, the per-row
// reciprocals of the bias corrections and approximate sqrt / divide (a few
// ulp; the fp32 store is tolerance-checked against the reference).
template <typename T>
__device__ __forceinline__ T adam_elem(T& p, T& m, T& v, T g, const AdamBC<T>& bc, T lr) {
  const T b1 = (T)0.9, b2 = (T)0.999, omb1 = (T)(1.0 - 0.9), omb2 = (T)(1.0 - 0.999), eps = (T)1e-8;
  T upd;
  if constexpr (sizeof(T) == 8) {
    m = add_rn(mul_rn(b1, m), mul_rn(omb1, g));
    v = add_rn(mul_rn(b2, v), mul_rn(mul_rn(omb2, g), g));
#if WV_FP64_RCP
    // reciprocal bias corrections (within an ulp of numpy's divisions; fewer registers)
    upd = div_rn(mul_rn(lr, mul_rn(m, (T)bc.r1)), add_rn(sqrt_rn(mul_rn(v, (T)bc.r2)), eps));
#else
    upd = div_rn(mul_rn(lr, div_rn(m, (T)bc.bc1)), add_rn(sqrt_rn(div_rn(v, (T)bc.bc2)), eps));
#endif
  } else {
    m = fmaf(b1, m, omb1 * g);
    v = fmaf(b2, v, (omb2 * g) * g);
    upd = __fdividef(lr * (m * bc.r1), sqrt_approx(v * bc.r2) + eps);
  }
  const T np_ = p - upd;
  const T old = p;
  p = np_;
  return (np_ != old) || (np_ != np_) ? T(1) : T(0);
}

// Contribution slot v -> (source row index, coefficient): input-matrix rows
// take the pair's centre gradient row G[b] (coefficient 1); output-matrix rows
// take coef * U[b] (the context's gpos or negative j's gneg).
template <typename T>
__device__ __forceinline__ uint32_t contribution(uint32_t v, bool side_out, int64_t B, int k, const SlotMap& sm,
                                                 const T* coef, T& c) {
  const uint2 e = slot_entry(v, side_out, B, k, sm);
  c = side_out ? __ldg(coef + e.y) : T(1);
  return e.x;  // G row (input side) or U row (output side)
}

// Phase 3: one warp per (unique row, 32-chunk slice of the row): sum the row's
// contributions in slot order (the order np.add.at applies them, w2v.py:415)
// and apply RowAdam in place.  One 16-byte chunk per lane keeps registers low
// so many warps are resident; the optimizer-state loads are issued before the
// contribution walk so their DRAM latency overlaps it.
template <typename T, int EPC, int MAXC>
__global__ void __launch_bounds__(kOwnerThreads, WV_OWNER_MINB) sgns_owner_kernel(OwnerArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (kOwnerThreads / 32);
  const int64_t gw = blockIdx.x * (int64_t)(kOwnerThreads / 32) + (threadIdx.x >> 5);
  const int d = A.d, k = A.k;
  const int C = d / EPC;
  const int64_t B = A.B;
  const uint32_t nseg = *A.seg_count;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // the batch is consumed: advance the cursor (read by the next batch's decode)
    WvSgnsDevState* st = A.state;
    atomicAdd((unsigned long long*)&st->rows_updated, (unsigned long long)nseg);
    st->batch += 1;
    st->step += 1;
  }
  const T* U = (const T*)A.U;
  const T* G = (const T*)A.G;
  const T* coef = (const T*)A.coef;
  const T b1 = (T)0.9, b2 = (T)0.999, omb1 = (T)(1.0 - 0.9), omb2 = (T)(1.0 - 0.999), eps = (T)1e-8;
  const T lr = (T)A.lr;
  const int64_t slots = (int64_t)nseg * MAXC;
  // Per-row metadata (segment record -> slot list -> coefficients) is a chain
  // of dependent L2 reads; the next row's chain is resolved while this row's
  // optimizer-state loads are in flight (software pipelining across rows).
  struct Meta {
    uint32_t start, len, key;
    double bc1, bc2;
    uint32_t myslot, my_ri;
    T my_c;
  };
  auto load_meta = [&](int64_t sl, Meta& mt) {
    const Segment sg = A.segs[sl / MAXC];
    mt.start = sg.start;
    mt.len = sg.len;
    mt.key = sg.key;
    mt.bc1 = sg.bc1;
    mt.bc2 = sg.bc2;
    mt.myslot = lane < (int)sg.len ? A.list[sg.start + lane] : 0xffffffffu;
    mt.my_c = 0;
    mt.my_ri = 0;
    if (lane < (int)sg.len) mt.my_ri = contribution<T>(mt.myslot, sg.key >= (uint32_t)A.V, B, k, A.sm, coef, mt.my_c);
  };
  Meta nxt;
  if (gw < slots) load_meta(gw, nxt);
  for (int64_t slot = gw; slot < slots; slot += warps_total) {
    const Meta cur = nxt;
    const int cc = (int)(slot % MAXC) * 32 + lane;
    Segment sg;
    sg.start = cur.start;
    sg.len = cur.len;
    sg.bc1 = cur.bc1;
    sg.bc2 = cur.bc2;
    const uint32_t key = cur.key;
    const bool side_out = key >= (uint32_t)A.V;
    const int64_t row = side_out ? (int64_t)key - A.V : (int64_t)key;
    const bool active = cc < C;
    const uint32_t myslot = cur.myslot;
    const T my_c = cur.my_c;
    const uint32_t my_ri = cur.my_ri;
    T* P = (T*)(side_out ? A.out : A.in);
    T* M = (T*)(side_out ? A.m_out : A.m_in);
    T* Vv = (T*)(side_out ? A.v_out : A.v_in);
    const int64_t o = row * d + (int64_t)cc * EPC;
    Chunk<T, EPC> p, m, vv, g;
    if (A.sparse && !A.split && active) {
      p = ld_chunk_rw<T, EPC>(P + o);
      m = ld_chunk_rw<T, EPC>(M + o);
      vv = ld_chunk_rw<T, EPC>(Vv + o);
    }
    // next row's metadata while this row's state loads are in flight
    if (slot + warps_total < slots) load_meta(slot + warps_total, nxt);
    int myrank = 0;
    for (int j = 0; j < (int)sg.len; ++j) myrank += __shfl_sync(0xffffffffu, myslot, j) < myslot;
#pragma unroll
    for (int e = 0; e < EPC; ++e) g.v[e] = 0;
    // contributions in groups of kOwnerGroup: all loads of a group are issued before the
    // (slot-ordered) adds, so a row's walk costs len/kOwnerGroup dependent round trips
    for (uint32_t i0 = 0; i0 < sg.len; i0 += kOwnerGroup) {
      const int nq = (int)min((uint32_t)kOwnerGroup, sg.len - i0);
      uint32_t ri[kOwnerGroup];
      T c[kOwnerGroup];
#pragma unroll
      for (int q = 0; q < kOwnerGroup; ++q) {
        const uint32_t owner = __ballot_sync(0xffffffffu, myrank == (int)i0 + q && lane < (int)sg.len);
        const int src_lane = owner ? __ffs(owner) - 1 : 0;
        ri[q] = __shfl_sync(0xffffffffu, my_ri, src_lane);
        c[q] = __shfl_sync(0xffffffffu, my_c, src_lane);
      }
      const T* srcb = (side_out ? U : G) + cc * EPC;
      Chunk<T, EPC> x[kOwnerGroup];
      if (active) {
#pragma unroll
        for (int q = 0; q < kOwnerGroup; ++q)
          if (q < nq) x[q] = ld_chunk<T, EPC>(srcb + (size_t)ri[q] * d);
#pragma unroll
        for (int q = 0; q < kOwnerGroup; ++q)
          if (q < nq) {
#pragma unroll
            for (int e = 0; e < EPC; ++e) g.v[e] = add_rn(g.v[e], side_out ? mul_rn(c[q], x[q].v[e]) : x[q].v[e]);
          }
      }
    }
    if (!A.sparse || A.split) {
      if (!A.sparse) {
        T* D = (T*)(side_out ? A.dense_g_out : A.dense_g_in);
        if (active) st_chunk<T, EPC>(D + o, g);
      } else if (active) {
        st_chunk<T, EPC>((T*)A.gsum + (slot / MAXC) * d + (int64_t)cc * EPC, g);
      }
      if (lane == 0 && cc == 0) {
        (side_out ? A.touched_out : A.touched_in)[row] = 1;
        A.cnt[key] = 0;
      }
      continue;
    }
    const AdamBC<T> bc(sg.bc1, sg.bc2);
    bool changed = false;
    if (active) {
#pragma unroll
      for (int e = 0; e < EPC; ++e) changed |= adam_elem<T>(p.v[e], m.v[e], vv.v[e], g.v[e], bc, lr) != T(0);
      st_chunk<T, EPC>(P + o, p);
      st_chunk<T, EPC>(M + o, m);
      st_chunk<T, EPC>(Vv + o, vv);
    }
    changed = __any_sync(0xffffffffu, changed);
    if (lane == 0) {
      if (cc == 0) {
        (side_out ? A.touched_out : A.touched_in)[row] = 1;
        A.cnt[key] = 0;
      }
      if (changed) (side_out ? A.modified_out : A.modified_in)[row] = 1;
    }
  }
}

// Phase 3 (default for 16-byte-multiple rows): warp per light row with the
// row's optimizer state (p, m, v) fetched by cp.async.bulk into a per-warp
// two-stage shared-memory ring: while row i is summed and updated, row i+1's
// state is already in flight and row i+2's metadata chain is resolving, so
// each warp keeps a full row of DRAM reads outstanding without holding it in
// registers.  Updated rows are written straight back from registers.
constexpr int kOwnerBulkWarps = 8;
constexpr int kOwnerBulkX = 1;                 // contribution rows fetched with the state rows
constexpr int kOwnerBulkRows = 3 + kOwnerBulkX;  // p, m, v, x0, x1
template <typename T, int EPC, int MAXC>
__global__ void __launch_bounds__(kOwnerBulkWarps * 32, 4) sgns_owner_bulk_kernel(OwnerArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = A.d, k = A.k;
  const int C = d / EPC;
  const int64_t B = A.B;
  const uint32_t row_bytes = (uint32_t)(d * sizeof(T));
  uint64_t* mybar = reinterpret_cast<uint64_t*>(smem_raw) + 2 * warp;
  T* ring = reinterpret_cast<T*>(smem_raw + 128) + (size_t)warp * 2 * kOwnerBulkRows * d;
  const uint32_t nseg = *A.seg_count;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    WvSgnsDevState* st = A.state;
    atomicAdd((unsigned long long*)&st->rows_updated, (unsigned long long)nseg);
    st->batch += 1;
    st->step += 1;
  }
  if (lane == 0) {
    mbar_init(mybar, 1);
    mbar_init(mybar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const T* U = (const T*)A.U;
  const T* G = (const T*)A.G;
  const T* coef = (const T*)A.coef;
  const T lr = (T)A.lr;
  const int64_t warps_total = (int64_t)gridDim.x * kOwnerBulkWarps;
  // a row's metadata: lane j holds contribution j (slot-order rank, source row, coefficient)
  struct Meta {
    uint32_t len, key;
    double bc1, bc2;
    int myrank;
    uint32_t my_ri;
    T my_c;
  };
  auto load_meta = [&](int64_t sgi, Meta& mt) {
    const Segment sg = A.segs[sgi];
    mt.len = sg.len;
    mt.key = sg.key;
    mt.bc1 = sg.bc1;
    mt.bc2 = sg.bc2;
    const uint32_t myslot = lane < (int)sg.len ? A.list[sg.start + lane] : 0xffffffffu;
    mt.my_c = 0;
    mt.my_ri = 0;
    if (lane < (int)sg.len) mt.my_ri = contribution<T>(myslot, sg.key >= (uint32_t)A.V, B, k, A.sm, coef, mt.my_c);
    int r = 0;
    for (int j = 0; j < (int)sg.len; ++j) r += __shfl_sync(0xffffffffu, myslot, j) < myslot;
    mt.myrank = lane < (int)sg.len ? r : 64;
  };
  // contribution of rank q: (source row, coefficient)
  auto ranked = [&](const Meta& mt, int q, uint32_t& ri, T& c) {
    const uint32_t owner = __ballot_sync(0xffffffffu, mt.myrank == q);
    const int src_lane = owner ? __ffs(owner) - 1 : 0;
    ri = __shfl_sync(0xffffffffu, mt.my_ri, src_lane);
    c = __shfl_sync(0xffffffffu, mt.my_c, src_lane);
  };
  auto issue = [&](const Meta& mt, int stage) {
    const bool so = mt.key >= (uint32_t)A.V;
    const int64_t row = so ? (int64_t)mt.key - A.V : (int64_t)mt.key;
    const int nx = (int)min((uint32_t)kOwnerBulkX, mt.len);
    uint32_t rx[kOwnerBulkX];
#pragma unroll
    for (int q = 0; q < kOwnerBulkX; ++q) {
      T cq;
      ranked(mt, q, rx[q], cq);
    }
    if (lane == 0) mbar_arrive_expect_tx(mybar + stage, (uint32_t)(3 + nx) * row_bytes);
    __syncwarp();
    T* dst = ring + (size_t)stage * kOwnerBulkRows * d;
    if (lane < 3) {
      const T* base = (const T*)(lane == 0 ? (so ? A.out : A.in) : lane == 1 ? (so ? A.m_out : A.m_in)
                                                                             : (so ? A.v_out : A.v_in));
      bulk_row_g2s(dst + (size_t)lane * d, base + row * d, row_bytes, mybar + stage);
    } else if (lane < 3 + nx) {
      const int q = lane - 3;
      uint32_t r = rx[0];
#pragma unroll
      for (int t = 1; t < kOwnerBulkX; ++t)
        if (q == t) r = rx[t];
      bulk_row_g2s(dst + (size_t)lane * d, (so ? U : G) + (size_t)r * d, row_bytes, mybar + stage);
    }
  };
  int64_t sgi = blockIdx.x * (int64_t)kOwnerBulkWarps + warp;
  Meta cur, nxt;
  uint32_t phase[2] = {0u, 0u};
  if (sgi < nseg) {
    load_meta(sgi, cur);
    issue(cur, 0);
    if (sgi + warps_total < nseg) load_meta(sgi + warps_total, nxt);
  }
  for (int it = 0; sgi < nseg; ++it, sgi += warps_total) {
    const int stage = it & 1;
    const bool have_next = sgi + warps_total < nseg;
    if (have_next) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(nxt, stage ^ 1);
    }
    const Meta m0 = cur;
    if (have_next) {
      cur = nxt;
      if (sgi + 2 * warps_total < nseg) load_meta(sgi + 2 * warps_total, nxt);
    }
    const bool side_out = m0.key >= (uint32_t)A.V;
    const int64_t row = side_out ? (int64_t)m0.key - A.V : (int64_t)m0.key;
    const int nx = (int)min((uint32_t)kOwnerBulkX, m0.len);
    T cx[kOwnerBulkX];
#pragma unroll
    for (int q = 0; q < kOwnerBulkX; ++q) {
      uint32_t rq;
      ranked(m0, q, rq, cx[q]);
    }
    while (!mbar_try_wait(mybar + stage, phase[stage])) {
    }
    phase[stage] ^= 1u;
    const T* sp = ring + (size_t)stage * kOwnerBulkRows * d;
    Chunk<T, EPC> g[MAXC];
#pragma unroll
    for (int qq = 0; qq < MAXC; ++qq) {
      const int cc = lane + 32 * qq;
#pragma unroll
      for (int e = 0; e < EPC; ++e) g[qq].v[e] = 0;
      if (cc < C) {
#pragma unroll
        for (int q = 0; q < kOwnerBulkX; ++q)
          if (q < nx) {
            const Chunk<T, EPC> x = *reinterpret_cast<const Chunk<T, EPC>*>(sp + (size_t)(3 + q) * d + cc * EPC);
#pragma unroll
            for (int e = 0; e < EPC; ++e) g[qq].v[e] = add_rn(g[qq].v[e], side_out ? mul_rn(cx[q], x.v[e]) : x.v[e]);
          }
      }
    }
    // contributions past the first kOwnerBulkX (rare for light rows): plain loads, slot order
    const T* srcb = side_out ? U : G;
    for (int q = kOwnerBulkX; q < (int)m0.len; ++q) {
      uint32_t rq;
      T cq;
      ranked(m0, q, rq, cq);
#pragma unroll
      for (int qq = 0; qq < MAXC; ++qq) {
        const int cc = lane + 32 * qq;
        if (cc < C) {
          const Chunk<T, EPC> x = ld_chunk<T, EPC>(srcb + (size_t)rq * d + cc * EPC);
#pragma unroll
          for (int e = 0; e < EPC; ++e) g[qq].v[e] = add_rn(g[qq].v[e], side_out ? mul_rn(cq, x.v[e]) : x.v[e]);
        }
      }
    }
    T* P = (T*)(side_out ? A.out : A.in);
    T* M = (T*)(side_out ? A.m_out : A.m_in);
    T* Vv = (T*)(side_out ? A.v_out : A.v_in);
    const AdamBC<T> bc(m0.bc1, m0.bc2);
    bool changed = false;
#pragma unroll
    for (int qq = 0; qq < MAXC; ++qq) {
      const int cc = lane + 32 * qq;
      if (cc < C) {
        Chunk<T, EPC> p = *reinterpret_cast<const Chunk<T, EPC>*>(sp + cc * EPC);
        Chunk<T, EPC> m = *reinterpret_cast<const Chunk<T, EPC>*>(sp + d + cc * EPC);
        Chunk<T, EPC> vv = *reinterpret_cast<const Chunk<T, EPC>*>(sp + 2 * d + cc * EPC);
#pragma unroll
        for (int e = 0; e < EPC; ++e) changed |= adam_elem<T>(p.v[e], m.v[e], vv.v[e], g[qq].v[e], bc, lr) != T(0);
        const int64_t o = row * d + (int64_t)cc * EPC;
        st_chunk<T, EPC>(P + o, p);
        st_chunk<T, EPC>(M + o, m);
        st_chunk<T, EPC>(Vv + o, vv);
      }
    }
    changed = __any_sync(0xffffffffu, changed);
    if (lane == 0) {
      (side_out ? A.touched_out : A.touched_in)[row] = 1;
      A.cnt[m0.key] = 0;
      if (changed) (side_out ? A.modified_out : A.modified_in)[row] = 1;
    }
    __syncwarp();
  }
}

// Phase 3 (default, sparse RowAdam): one thread per kFlatU x (light row,
// 16-byte chunk) items in a flat grid-stride space, so no lane idles on a row's ragged
// chunk count and every thread's loads are independent (the access pattern
// measured closest to HBM bandwidth, profiles/micro/rows_bench.cu).  The
// row's optimizer state is loaded as soon as its segment record is known;
// contributions come from group_order's slot-ordered list and are summed in
// that order (w2v.py:415 np.add.at order), then RowAdam is applied in place.
#ifndef WV_FLAT_U
#define WV_FLAT_U 1
#endif
#ifndef WV_FLAT_MINB
#define WV_FLAT_MINB 4  // 64 registers, no spill stack (48 spilled 40 B): fp64 owner 297 -> 290 us
#endif
#ifndef WV_OWNER_FUSED_HEAVY
#define WV_OWNER_FUSED_HEAVY 0
#endif
#ifndef WV_PIECE_THREADS
#define WV_PIECE_THREADS 128
#endif
#ifndef WV_PIECE_GRID
#define WV_PIECE_GRID 148
#endif
#ifndef WV_FLAT_SEGPF
#define WV_FLAT_SEGPF 0  // load the next item's segment record one iteration ahead
#endif
#ifndef WV_FLAT_PREFETCH
#define WV_FLAT_PREFETCH 0
#endif
#ifndef WV_FLAT_ASYNC
#define WV_FLAT_ASYNC 0  // measured slower (smem carve-out shrinks L1; 205 vs 151 us)
#endif
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
constexpr int kFlatU = WV_FLAT_U;  // (row, chunk) items per thread in flight

template <typename T, int EPC, int MAXC>
__device__ __forceinline__ void heavy_piece_work(const OwnerArgs& A, uint32_t pc);
// Single-contribution light rows (92 % of a cfg2 batch's unique rows): the row's one
// contribution rides in its record (start = source U/G row, pad = coefficient), so a
// (row, 16-byte chunk) item is p, m, v, one contribution chunk and the RowAdam update,
// with no entry list -- fewer registers than the general light-row kernel, more CTAs.
// Same arithmetic as sgns_owner_flat_kernel (g = 0 + contribution, adam_elem).
template <typename T, int EPC>
__global__ void __launch_bounds__(256, WV_SINGLE_MINB) sgns_owner_single_kernel(OwnerArgs A, bool tiles) {
  const int d = A.d;
  const uint32_t C = (uint32_t)(d / EPC);
  const uint32_t total = *(volatile const uint32_t*)(A.gctr + GC_SINGLE) * C;
  const T* U = (const T*)A.U;
  const T* G = (const T*)A.G;
  const T* coef = (const T*)A.coef;
  const T lr = (T)A.lr;
  auto item = [&](uint32_t i) {
    uint32_t r = __umulhi(i, A.cmag);
    int32_t c = (int32_t)(i - r * C);
    if (c < 0) {
      --r;
      c += (int32_t)C;
    } else if (c >= (int32_t)C) {
      ++r;
      c -= (int32_t)C;
    }
    const Segment sg = A.singles[r];
    const bool side_out = sg.key >= (uint32_t)A.V;
    const int64_t row = side_out ? (int64_t)sg.key - A.V : (int64_t)sg.key;
    const int64_t o = row * d + (int64_t)c * EPC;
    T* P = (T*)(side_out ? A.out : A.in);
    T* M = (T*)(side_out ? A.m_out : A.m_in);
    T* Vv = (T*)(side_out ? A.v_out : A.v_in);
    Chunk<T, EPC> p = ld_chunk_p<T, EPC>(P + o);
    Chunk<T, EPC> m = ld_chunk_mv<T, EPC>(M + o);
    Chunk<T, EPC> vv = ld_chunk_mv<T, EPC>(Vv + o);
    const Chunk<T, EPC> x = ld_chunk<T, EPC>((side_out ? U : G) + (int64_t)sg.start * d + (int64_t)c * EPC);
    const T cf = side_out ? __ldg(coef + sg.pad) : T(1);
    const AdamBC<T> bc(sg.bc1, sg.bc2);
    bool changed = false;
#pragma unroll
    for (int e = 0; e < EPC; ++e) {
      const T g = add_rn(T(0), side_out ? mul_rn(cf, x.v[e]) : x.v[e]);
      changed |= adam_elem<T>(p.v[e], m.v[e], vv.v[e], g, bc, lr) != T(0);
    }
    st_chunk_p<T, EPC>(P + o, p);
    st_chunk_mv<T, EPC>(M + o, m);
    st_chunk_mv<T, EPC>(Vv + o, vv);
    if (changed) (side_out ? A.modified_out : A.modified_in)[row] = 1;
    if (c == 0) {
      (side_out ? A.touched_out : A.touched_in)[row] = 1;
      A.cnt[sg.key] = 0;
    }
  };
  if (tiles) {  // one short-lived tile of blockDim.x * WV_SINGLE_TILE items (concurrent schedule)
    const uint32_t base = blockIdx.x * blockDim.x * (uint32_t)WV_SINGLE_TILE + threadIdx.x;
#pragma unroll 1
    for (int j = 0; j < WV_SINGLE_TILE; ++j) {
      const uint32_t i = base + (uint32_t)j * blockDim.x;
      if (i >= total) break;
      item(i);
    }
  } else {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) item(i);
  }
}

template <typename T, int EPC, int MAXC>
__global__ void __launch_bounds__(256, WV_FLAT_MINB) sgns_owner_flat_kernel(OwnerArgs A) {
  const int d = A.d;
  const uint32_t C = (uint32_t)(d / EPC);
  const uint32_t nseg = *A.seg_count;
  const Segment* segs = A.segs + (A.seg_base ? *A.seg_base : 0u);
  if (A.bookkeep && blockIdx.x == 0 && threadIdx.x == 0) {
    WvSgnsDevState* st = A.state;
    atomicAdd((unsigned long long*)&st->rows_updated,
              (unsigned long long)(A.gctr[GC_LIGHT] + A.gctr[GC_HEAVY] + A.gctr[GC_SINGLE]));
    st->batch += 1;
    st->step += 1;
  }
  // heavy-row pieces first (warp per piece, spread over every SM), then the
  // light rows' (row, chunk) items
  if (WV_OWNER_FUSED_HEAVY) {
    const uint32_t np_total = *(volatile const uint32_t*)(A.gctr + GC_PIECES);
    const uint32_t warps = gridDim.x * (blockDim.x / 32);
    for (uint32_t pc = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); pc < np_total; pc += warps)
      heavy_piece_work<T, EPC, MAXC>(A, pc);
  }
  const T* U = (const T*)A.U;
  const T* G = (const T*)A.G;
  const T* coef = (const T*)A.coef;
  const T lr = (T)A.lr;
  const uint32_t total = nseg * C;
  const uint32_t stride = gridDim.x * blockDim.x * kFlatU;
  if constexpr (WV_FLAT_ASYNC && kFlatU == 1 && EPC * sizeof(T) == 16) {
    // Two-deep software pipeline: the next item's optimizer state (and its only
    // contribution row, for single-contribution rows) is copied HBM -> shared
    // with cp.async while this item is summed and updated, so each thread keeps
    // two items' loads in flight without holding them in registers.
    __shared__ __align__(16) uint4 abuf[2][4][256];
    __shared__ Segment sbuf[2][256];  // the in-flight items' segment records (off the register file)
    const int tid = threadIdx.x;
    auto chunk_of = [&](uint32_t i, uint32_t& r) {
      r = __umulhi(i, A.cmag);
      int32_t c = (int32_t)(i - r * C);
      if (c < 0) {
        --r;
        c += (int32_t)C;
      } else if (c >= (int32_t)C) {
        ++r;
        c -= (int32_t)C;
      }
      return c;
    };
    auto issue = [&](uint32_t i, int s) {
      uint32_t r;
      const int32_t c = chunk_of(i, r);
      const Segment sg = segs[r];
      sbuf[s][tid] = sg;
      const bool so = sg.key >= (uint32_t)A.V;
      const int64_t row = so ? (int64_t)sg.key - A.V : (int64_t)sg.key;
      const int64_t o = row * d + (int64_t)c * EPC;
      cp_async16(&abuf[s][0][tid], (const T*)(so ? A.out : A.in) + o);
      cp_async16(&abuf[s][1][tid], (const T*)(so ? A.m_out : A.m_in) + o);
      cp_async16(&abuf[s][2][tid], (const T*)(so ? A.v_out : A.v_in) + o);
      if (sg.len == 1) cp_async16(&abuf[s][3][tid], (so ? U : G) + (int64_t)sg.start * d + (int64_t)c * EPC);
      cp_async_commit();
    };
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    int s = 0;
    if (i < total) issue(i, 0);
    for (; i < total; i += stride) {
      const uint32_t inx = i + stride;
      if (inx < total)
        issue(inx, s ^ 1);
      else
        cp_async_commit();
      cp_async_wait<1>();
      uint32_t rr;
      const int32_t c = chunk_of(i, rr);
      const Segment sg = sbuf[s][tid];
      const bool side_out = sg.key >= (uint32_t)A.V;
      const int64_t row = side_out ? (int64_t)sg.key - A.V : (int64_t)sg.key;
      const int64_t o = row * d + (int64_t)c * EPC;
      Chunk<T, EPC> p = *reinterpret_cast<const Chunk<T, EPC>*>(&abuf[s][0][tid]);
      Chunk<T, EPC> m = *reinterpret_cast<const Chunk<T, EPC>*>(&abuf[s][1][tid]);
      Chunk<T, EPC> vv = *reinterpret_cast<const Chunk<T, EPC>*>(&abuf[s][2][tid]);
      Chunk<T, EPC> g;
#pragma unroll
      for (int e = 0; e < EPC; ++e) g.v[e] = 0;
      if (sg.len == 1) {
        const Chunk<T, EPC> x = *reinterpret_cast<const Chunk<T, EPC>*>(&abuf[s][3][tid]);
        const T cf = side_out ? __ldg(coef + sg.pad) : T(1);
#pragma unroll
        for (int e = 0; e < EPC; ++e) g.v[e] = add_rn(g.v[e], side_out ? mul_rn(cf, x.v[e]) : x.v[e]);
      } else {
        const T* srcb = (side_out ? U : G) + (int64_t)c * EPC;
        for (uint32_t q = 0; q < sg.len; ++q) {
          const uint2 en = __ldg(A.ents + sg.start + q);
          const Chunk<T, EPC> x = ld_chunk<T, EPC>(srcb + (int64_t)en.x * d);
          if (side_out) {
            const T cq = __ldg(coef + en.y);
#pragma unroll
            for (int e = 0; e < EPC; ++e) g.v[e] = add_rn(g.v[e], mul_rn(cq, x.v[e]));
          } else {
#pragma unroll
            for (int e = 0; e < EPC; ++e) g.v[e] = add_rn(g.v[e], x.v[e]);
          }
        }
      }
      const AdamBC<T> bc(sg.bc1, sg.bc2);
      bool changed = false;
#pragma unroll
      for (int e = 0; e < EPC; ++e) changed |= adam_elem<T>(p.v[e], m.v[e], vv.v[e], g.v[e], bc, lr) != T(0);
      st_chunk<T, EPC>((T*)(side_out ? A.out : A.in) + o, p);
      st_chunk<T, EPC>((T*)(side_out ? A.m_out : A.m_in) + o, m);
      st_chunk<T, EPC>((T*)(side_out ? A.v_out : A.v_in) + o, vv);
      if (changed) (side_out ? A.modified_out : A.modified_in)[row] = 1;
      if (c == 0) {
        (side_out ? A.touched_out : A.touched_in)[row] = 1;
        A.cnt[sg.key] = 0;
        if (A.flag) A.flag[sg.key] = 0;
      }
      s ^= 1;
    }
    cp_async_wait<0>();
    return;
  }
  // the next item's segment record is loaded one iteration ahead (its p/m/v addresses
  // are then known at the top of the iteration: one dependent load less per item)
  auto split_item = [&](uint32_t i, int32_t& c) -> uint32_t {
    uint32_t r = __umulhi(i, A.cmag);
    c = (int32_t)(i - r * C);
    if (c < 0) {
      --r;
      c += (int32_t)C;
    } else if (c >= (int32_t)C) {
      ++r;
      c -= (int32_t)C;
    }
    return r;
  };
  Segment sg_next;
  int32_t c_next = 0;
  if constexpr (WV_FLAT_SEGPF && kFlatU == 1) {
    const uint32_t i_first = blockIdx.x * blockDim.x + threadIdx.x;
    if (i_first < total) sg_next = segs[split_item(i_first, c_next)];
  }
  for (uint32_t i0 = blockIdx.x * blockDim.x * kFlatU + threadIdx.x; i0 < total; i0 += stride) {
    if (WV_FLAT_PREFETCH > 0) {
      // L2 prefetch of the optimizer-state rows this thread's item will touch
      // WV_FLAT_PREFETCH iterations ahead (one bulk prefetch per row and array,
      // issued by the thread holding the row's chunk 0 or the warp's first lane)
      const uint32_t i2 = i0 + (uint32_t)WV_FLAT_PREFETCH * stride;
      if (i2 < total) {
        uint32_t r2 = __umulhi(i2, A.cmag);
        int32_t c2 = (int32_t)(i2 - r2 * C);
        if (c2 < 0) {
          --r2;
          c2 += (int32_t)C;
        } else if (c2 >= (int32_t)C) {
          ++r2;
          c2 -= (int32_t)C;
        }
        if (c2 == 0 || (threadIdx.x & 31) == 0) {
          const uint32_t key = segs[r2].key;
          const bool so = key >= (uint32_t)A.V;
          const int64_t row = so ? (int64_t)key - A.V : (int64_t)key;
          const uint32_t bytes = (uint32_t)(d * sizeof(T));
          const T* rows3[3] = {(const T*)(so ? A.out : A.in), (const T*)(so ? A.m_out : A.m_in),
                               (const T*)(so ? A.v_out : A.v_in)};
#pragma unroll
          for (int a = 0; a < 3; ++a)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rows3[a] + row * d), "r"(bytes)
                         : "memory");
        }
      }
    }
    Segment sg[kFlatU];
    int32_t cr[kFlatU];
    bool ok[kFlatU];
    if constexpr (WV_FLAT_SEGPF && kFlatU == 1) {
      ok[0] = true;
      sg[0] = sg_next;
      cr[0] = c_next;
      const uint32_t in_ = i0 + stride;
      if (in_ < total) sg_next = segs[split_item(in_, c_next)];
    } else {
#pragma unroll
      for (int u = 0; u < kFlatU; ++u) {
        const uint32_t i = i0 + u * blockDim.x;
        ok[u] = i < total;
        int32_t c;
        const uint32_t r = split_item(i, c);
        cr[u] = c;
        if (ok[u]) sg[u] = segs[r];
      }
    }
    Chunk<T, EPC> p[kFlatU], m[kFlatU], vv[kFlatU], g[kFlatU];
#pragma unroll
    for (int u = 0; u < kFlatU; ++u) {
#pragma unroll
      for (int e = 0; e < EPC; ++e) g[u].v[e] = 0;
      if (!ok[u]) continue;
      const bool side_out = sg[u].key >= (uint32_t)A.V;
      const int64_t row = side_out ? (int64_t)sg[u].key - A.V : (int64_t)sg[u].key;
      const int64_t o = row * d + (int64_t)cr[u] * EPC;
      p[u] = ld_chunk_p<T, EPC>((const T*)(side_out ? A.out : A.in) + o);
      m[u] = ld_chunk_mv<T, EPC>((const T*)(side_out ? A.m_out : A.m_in) + o);
      vv[u] = ld_chunk_mv<T, EPC>((const T*)(side_out ? A.v_out : A.v_in) + o);
    }
#pragma unroll
    for (int u = 0; u < kFlatU; ++u) {
      if (!ok[u]) continue;
      const bool side_out = sg[u].key >= (uint32_t)A.V;
      const T* srcb = (side_out ? U : G) + (int64_t)cr[u] * EPC;
      for (uint32_t q = 0; q < sg[u].len; ++q) {
        // single-contribution rows carry their entry in the segment record (group_order)
        const uint2 en = sg[u].len == 1 ? make_uint2(sg[u].start, sg[u].pad) : __ldg(A.ents + sg[u].start + q);
        const Chunk<T, EPC> x = ld_chunk<T, EPC>(srcb + (int64_t)en.x * d);
        if (side_out) {
          const T c = __ldg(coef + en.y);
#pragma unroll
          for (int e = 0; e < EPC; ++e) g[u].v[e] = add_rn(g[u].v[e], mul_rn(c, x.v[e]));
        } else {
#pragma unroll
          for (int e = 0; e < EPC; ++e) g[u].v[e] = add_rn(g[u].v[e], x.v[e]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kFlatU; ++u) {
      if (!ok[u]) continue;
      const bool side_out = sg[u].key >= (uint32_t)A.V;
      const int64_t row = side_out ? (int64_t)sg[u].key - A.V : (int64_t)sg[u].key;
      const int64_t o = row * d + (int64_t)cr[u] * EPC;
      const AdamBC<T> bc(sg[u].bc1, sg[u].bc2);
      bool changed = false;
#pragma unroll
      for (int e = 0; e < EPC; ++e) changed |= adam_elem<T>(p[u].v[e], m[u].v[e], vv[u].v[e], g[u].v[e], bc, lr) != T(0);
      st_chunk_p<T, EPC>((T*)(side_out ? A.out : A.in) + o, p[u]);
      if (WV_OWNER_P_APPLY) {
        // hand the gather's evict-last line back to the normal pool once updated
        const uintptr_t ln = (uintptr_t)((T*)(side_out ? A.out : A.in) + o) & ~(uintptr_t)127;
        asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(ln) : "memory");
      }
      st_chunk_mv<T, EPC>((T*)(side_out ? A.m_out : A.m_in) + o, m[u]);
      st_chunk_mv<T, EPC>((T*)(side_out ? A.v_out : A.v_in) + o, vv[u]);
      if (changed) (side_out ? A.modified_out : A.modified_in)[row] = 1;
      if (cr[u] == 0) {
        (side_out ? A.touched_out : A.touched_in)[row] = 1;
        A.cnt[sg[u].key] = 0;
        if (A.flag) A.flag[sg[u].key] = 0;
      }
    }
  }
}

// Stable LSD radix sort (8-bit digits) of n slots by one CTA of kHeavyThreads
// threads: a ping-pongs with tmp; returns the buffer holding the result.  Per
// tile of kHeavyThreads items each warp ranks equal digits with match_any and
// the per-(warp, digit) counts are prefixed in warp order, so ties keep input
// order (slots are distinct anyway; stability keeps it a pure permutation).
__device__ uint32_t* cta_sort_slots(uint32_t* a, uint32_t* tmp, uint32_t n, int bits,
                                    uint32_t (*cnt)[256]) {
  constexpr int NW = kHeavyThreads / 32;
  __shared__ uint32_t base[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int shift = 0; shift < bits; shift += 8) {
    // global digit histogram -> exclusive bases
    for (int t = threadIdx.x; t < 256; t += kHeavyThreads) base[t] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += kHeavyThreads) atomicAdd(&base[(a[i] >> shift) & 255u], 1u);
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t carry = 0;
      for (int c0 = 0; c0 < 256; c0 += 32) {
        const uint32_t v = base[c0 + lane];
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += x;
        }
        base[c0 + lane] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    __syncthreads();
    for (uint32_t t0 = 0; t0 < n; t0 += kHeavyThreads) {
      const uint32_t i = t0 + threadIdx.x;
      const bool ok = i < n;
      const uint32_t x = ok ? a[i] : 0u;
      const uint32_t dg = ok ? (x >> shift) & 255u : 256u + lane;  // unique dummy digit
      for (int t = threadIdx.x; t < NW * 256; t += kHeavyThreads) cnt[t / 256][t % 256] = 0;
      __syncthreads();
      const uint32_t peers = __match_any_sync(0xffffffffu, dg);
      const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
      if (ok && rank == 0) cnt[warp][dg] = __popc(peers);
      __syncthreads();
      for (int t = threadIdx.x; t < 256; t += kHeavyThreads) {
        uint32_t off = base[t];
        for (int w = 0; w < NW; ++w) {
          const uint32_t c = cnt[w][t];
          cnt[w][t] = off;
          off += c;
        }
        base[t] = off;
      }
      __syncthreads();
      if (ok) tmp[cnt[warp][dg] + rank] = x;
      __syncthreads();
    }
    uint32_t* sw = a;
    a = tmp;
    tmp = sw;
    __syncthreads();
  }
  return a;
}

// Phase 3b: one CTA per heavy row.  Warp w sums the w-th contiguous eighth of
// the row's contributions (slot order inside each part), the parts are added
// in part order through shared memory (a fixed two-level order, so the result
// is deterministic), then the threads apply RowAdam element-parallel.
template <typename T, int EPC, int MAXC>
#ifndef WV_HEAVY_MINB
#define WV_HEAVY_MINB 1
#endif
#ifndef WV_HEAVY_GRID
#define WV_HEAVY_GRID (148 * 4)
#endif
// float64: the heavy pieces run alone before the light rows (all of a piece group's loads in
// flight, a 592-CTA grid), and the light rows then take 4 CTAs per SM: +1.2 % over the concurrent
// schedule; float32 keeps the concurrent one (serial measured -3.2 %)
#ifndef WV_PIECE_ALL_LOADS
#define WV_PIECE_ALL_LOADS 2  // 0 never, 1 always, 2 float64 only
#endif
#ifndef WV_HEAVY_SERIAL
#define WV_HEAVY_SERIAL 2  // 0 never, 1 always, 2 float64 only
#endif
#ifndef WV_SERIAL_PIECE_GRID
#define WV_SERIAL_PIECE_GRID 592
#endif
#ifndef WV_SERIAL_OWNER_PER_SM
#define WV_SERIAL_OWNER_PER_SM 4
#endif
#ifndef WV_SPLIT_B_PER_SM
#define WV_SPLIT_B_PER_SM 2  // split owner: B-row CTAs per SM (they share the SMs with the next gather)
#endif
#ifndef WV_SPLIT_OWNER
#define WV_SPLIT_OWNER 0  // measured: the B rows starve the concurrent gather (97 -> 307 us), 60.4 -> 44.7 M pairs/s fp64
#endif
#ifndef WV_OWNER_PER_SM
#define WV_OWNER_PER_SM 3  // light-row owner CTAs per SM (room for the concurrent heavy pieces); 0: all resident
#endif
__global__ void __launch_bounds__(kHeavyThreads, WV_HEAVY_MINB) sgns_heavy_kernel(OwnerArgs A) {
  constexpr int W = kHeavyThreads / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* part = reinterpret_cast<T*>(smem_raw);  // [W][d]
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem_raw + (size_t)W * A.d * sizeof(T));
  const uint32_t bitmap_words = heavy_bitmap_words(A.n_items);
  __shared__ uint32_t sort_hist[kHeavyThreads / 32][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = A.d, k = A.k;
  const int C = d / EPC;
  const int64_t B = A.B;
  const uint32_t nh = A.seg_count[1];
  const T* U = (const T*)A.U;
  const T* G = (const T*)A.G;
  const T* coef = (const T*)A.coef;
  const T b1 = (T)0.9, b2 = (T)0.999, omb1 = (T)(1.0 - 0.9), omb2 = (T)(1.0 - 0.999), eps = (T)1e-8;
  const T lr = (T)A.lr;
  if (blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd((unsigned long long*)&A.state->rows_updated, (unsigned long long)nh);
  for (uint32_t h = blockIdx.x; h < nh; h += gridDim.x) {
    const Segment sg = A.heavy[h];
    const uint32_t key = sg.key;
    const bool side_out = key >= (uint32_t)A.V;
    const int64_t row = side_out ? (int64_t)key - A.V : (int64_t)key;
    // restore slot order of the row's list: a bitmap over the batch's slot
    // space (set bits, prefix popcounts, emit in order) when it fits in shared
    // memory, else a CTA radix sort; either way the result is in slot order
    const uint32_t* sorted;
    if (bitmap_words > 0) {
      for (uint32_t i = threadIdx.x; i < bitmap_words; i += kHeavyThreads) bitmap[i] = 0u;
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < sg.len; i += kHeavyThreads) {
        const uint32_t x = A.list[sg.start + i];
        atomicOr(&bitmap[x >> 5], 1u << (x & 31));
      }
      __syncthreads();
      const uint32_t per_t = (bitmap_words + kHeavyThreads - 1) / kHeavyThreads;
      const uint32_t w0 = min(bitmap_words, threadIdx.x * per_t), w1 = min(bitmap_words, w0 + per_t);
      uint32_t mine = 0;
      for (uint32_t w = w0; w < w1; ++w) mine += __popc(bitmap[w]);
      __shared__ uint32_t scan_total;
      uint32_t pos = block_excl_scan<uint32_t, kHeavyThreads>(mine, &scan_total);
      uint32_t* out_sorted = A.list_tmp + sg.start;
      for (uint32_t w = w0; w < w1; ++w) {
        uint32_t bits = bitmap[w];
        while (bits) {
          const int bt = __ffs(bits) - 1;
          out_sorted[pos++] = w * 32u + (uint32_t)bt;
          bits &= bits - 1u;
        }
      }
      __syncthreads();
      sorted = out_sorted;
    } else {
      sorted = cta_sort_slots(const_cast<uint32_t*>(A.list) + sg.start, A.list_tmp + sg.start, sg.len, A.slot_bits,
                              sort_hist);
    }
    // warp w sums the w-th contiguous part of the sorted list: 32 slots and
    // their coefficients are fetched per lane at once, then the rows are
    // loaded kHeavyGroup at a time and added in slot order
    const uint32_t per = (sg.len + W - 1) / W;
    const uint32_t lo = min(sg.len, per * warp), hi = min(sg.len, per * (warp + 1));
    const T* srcb = side_out ? U : G;
    Chunk<T, EPC> g[MAXC];
#pragma unroll
    for (int q = 0; q < MAXC; ++q)
#pragma unroll
      for (int e = 0; e < EPC; ++e) g[q].v[e] = 0;
    for (uint32_t i0 = lo; i0 < hi; i0 += 32) {
      const uint32_t n32 = min(32u, hi - i0);
      T my_c = 0;
      uint32_t my_ri = 0;
      if ((uint32_t)lane < n32) my_ri = contribution<T>(sorted[i0 + lane], side_out, B, k, A.sm, coef, my_c);
      for (uint32_t j0 = 0; j0 < n32; j0 += kHeavyGroup) {
        const int nq = (int)min((uint32_t)kHeavyGroup, n32 - j0);
        uint32_t ri[kHeavyGroup];
        T c[kHeavyGroup];
#pragma unroll
        for (int q = 0; q < kHeavyGroup; ++q) {
          ri[q] = __shfl_sync(0xffffffffu, my_ri, (j0 + q) & 31);
          c[q] = __shfl_sync(0xffffffffu, my_c, (j0 + q) & 31);
        }
#pragma unroll
        for (int qq = 0; qq < MAXC; ++qq) {
          const int cc = lane + 32 * qq;
          if (cc < C) {
            Chunk<T, EPC> x[kHeavyGroup];
#pragma unroll
            for (int q = 0; q < kHeavyGroup; ++q)
              if (q < nq) x[q] = ld_chunk<T, EPC>(srcb + (size_t)ri[q] * d + cc * EPC);
#pragma unroll
            for (int q = 0; q < kHeavyGroup; ++q)
              if (q < nq) {
#pragma unroll
                for (int e = 0; e < EPC; ++e)
                  g[qq].v[e] = add_rn(g[qq].v[e], side_out ? mul_rn(c[q], x[q].v[e]) : x[q].v[e]);
              }
          }
        }
      }
    }
#pragma unroll
    for (int qq = 0; qq < MAXC; ++qq) {
      const int cc = lane + 32 * qq;
      if (cc < C) {
#pragma unroll
        for (int e = 0; e < EPC; ++e) part[warp * d + cc * EPC + e] = g[qq].v[e];
      }
    }
    __syncthreads();
    T* P = (T*)(side_out ? A.out : A.in);
    T* M = (T*)(side_out ? A.m_out : A.m_in);
    T* Vv = (T*)(side_out ? A.v_out : A.v_in);
    const AdamBC<T> bc(sg.bc1, sg.bc2);
    bool changed = false;
    for (int e = threadIdx.x; e < d; e += kHeavyThreads) {
      T gr = part[e];
#pragma unroll
      for (int w = 1; w < W; ++w) gr = add_rn(gr, part[w * d + e]);
      const int64_t o = row * d + e;
      if (!A.sparse) {
        ((T*)(side_out ? A.dense_g_out : A.dense_g_in))[o] = gr;
        continue;
      }
      if (A.split) {
        ((T*)A.gsum)[(A.n_items - 1 - (int64_t)h) * d + e] = gr;
        continue;
      }
      T p = P[o], m = M[o], vv = Vv[o];
      changed |= adam_elem<T>(p, m, vv, gr, bc, lr) != T(0);
      P[o] = p;
      M[o] = m;
      Vv[o] = vv;
    }
    changed = __syncthreads_or(changed);
    if (threadIdx.x == 0) {
      (side_out ? A.touched_out : A.touched_in)[row] = 1;
      if (changed && A.sparse && !A.split) (side_out ? A.modified_out : A.modified_in)[row] = 1;
      A.cnt[key] = 0;
    }
    __syncthreads();  // shared buffers are reused by the next heavy row
  }
}

// ------------------------------------------------ heavy rows, split -----
// Heavy rows (predicates, hub entities: > kLightMax contributions, up to
// thousands) are spread over many warps instead of one CTA per row, so the
// hottest row no longer bounds the phase: heavy_order (side stream, off the
// critical path) sorts each heavy row's list into slot order, resolves the
// entries and cuts the row into pieces of kPiece contributions; heavy_piece
// (one warp per piece) sums its piece in slot order, and the warp finishing a
// row's last piece sums the piece partials in piece order and applies RowAdam.
// The association ((c0 + .. + c31) + (c32 + ..)) is fixed, so results are
// deterministic run to run.
#ifndef WV_PIECE
#define WV_PIECE 32
#endif
constexpr int kPiece = WV_PIECE;
static_assert(kPiece >= 1 && kPiece <= 32, "heavy pieces map one contribution per lane");

#ifndef WV_PIECE_FP64
#define WV_PIECE_FP64 32  // float64 piece size (16 measured -3 %; at most 32: a piece's entries live one per lane)
#endif
static_assert(WV_PIECE >= 1 && WV_PIECE <= 32 && WV_PIECE_FP64 >= 1 && WV_PIECE_FP64 <= 32,
              "heavy pieces hold one entry per lane: at most 32 contributions");
constexpr int kPieceMin = WV_PIECE_FP64 < kPiece ? WV_PIECE_FP64 : kPiece;
__host__ __device__ __forceinline__ int64_t max_pieces(int64_t items) {
  return items / kPieceMin + items / (kLightMax + 1) + 2;
}

__global__ void __launch_bounds__(kHeavyThreads) heavy_order(OwnerArgs A, uint32_t* gctr, uint2* pieces) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem_raw);
  const uint32_t bitmap_words = heavy_bitmap_words(A.n_items);
  __shared__ uint32_t sort_hist[kHeavyThreads / 32][256];
  __shared__ uint32_t s_pbase;
  const uint32_t nh = *(volatile uint32_t*)(gctr + GC_HEAVY);
  Segment* heavy = const_cast<Segment*>(A.heavy);
  uint2* ents = const_cast<uint2*>(A.ents);
  for (uint32_t h = blockIdx.x; h < nh; h += gridDim.x) {
    const Segment sg = heavy[h];
    const bool side_out = sg.key >= (uint32_t)A.V;
    const uint32_t* sorted;
    if (bitmap_words > 0) {
      for (uint32_t i = threadIdx.x; i < bitmap_words; i += kHeavyThreads) bitmap[i] = 0u;
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < sg.len; i += kHeavyThreads) {
        const uint32_t x = A.list[sg.start + i];
        atomicOr(&bitmap[x >> 5], 1u << (x & 31));
      }
      __syncthreads();
      const uint32_t per_t = (bitmap_words + kHeavyThreads - 1) / kHeavyThreads;
      const uint32_t w0 = min(bitmap_words, threadIdx.x * per_t), w1 = min(bitmap_words, w0 + per_t);
      uint32_t mine = 0;
      for (uint32_t w = w0; w < w1; ++w) mine += __popc(bitmap[w]);
      __shared__ uint32_t scan_total;
      uint32_t pos = block_excl_scan<uint32_t, kHeavyThreads>(mine, &scan_total);
      uint32_t* out_sorted = A.list_tmp + sg.start;
      for (uint32_t w = w0; w < w1; ++w) {
        uint32_t bits = bitmap[w];
        while (bits) {
          const int bt = __ffs(bits) - 1;
          out_sorted[pos++] = w * 32u + (uint32_t)bt;
          bits &= bits - 1u;
        }
      }
      __syncthreads();
      sorted = out_sorted;
    } else {
      sorted = cta_sort_slots(const_cast<uint32_t*>(A.list) + sg.start, A.list_tmp + sg.start, sg.len, A.slot_bits,
                              sort_hist);
    }
    for (uint32_t i = threadIdx.x; i < sg.len; i += kHeavyThreads)
      ents[sg.start + i] = slot_entry(sorted[i], side_out, A.B, A.k, A.sm);
    const uint32_t np = (sg.len + A.piece - 1) / A.piece;
    if (threadIdx.x == 0) {
      s_pbase = atomicAdd(gctr + GC_PIECES, np);
      heavy[h].pad = s_pbase;
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < np; j += kHeavyThreads) pieces[s_pbase + j] = make_uint2(h, j);
    __syncthreads();  // shared buffers are reused by the next heavy row
  }
}

constexpr int kPieceGroup = 4;  // contribution rows loaded together per warp

// One heavy-row piece, by one warp (called from the flat owner kernel).
template <typename T, int EPC, int MAXC>
__device__ __forceinline__ void heavy_piece_work(const OwnerArgs& A, uint32_t pc) {
  const int lane = threadIdx.x & 31;
  const int d = A.d;
  const int C = d / EPC;
  const T* U = (const T*)A.U;
  const T* G = (const T*)A.G;
  const T* coef = (const T*)A.coef;
  const T lr = (T)A.lr;
  T* partial = (T*)A.partial;
  {
    const uint2 pd = A.pieces[pc];
    const Segment sg = A.heavy[pd.x];
    const bool side_out = sg.key >= (uint32_t)A.V;
    const uint32_t np = (sg.len + A.piece - 1) / A.piece;
    const uint32_t q0 = pd.y * A.piece;
    const int n = (int)min(A.piece, sg.len - q0);
    uint2 my = make_uint2(0, 0);
    T my_c = 1;
    if (lane < n) {
      my = __ldg(A.ents + sg.start + q0 + lane);
      if (side_out) my_c = __ldg(coef + my.y);
    }
    const T* srcb = side_out ? U : G;
    Chunk<T, EPC> g[MAXC];
#pragma unroll
    for (int qq = 0; qq < MAXC; ++qq)
#pragma unroll
      for (int e = 0; e < EPC; ++e) g[qq].v[e] = 0;
    for (int j0 = 0; j0 < n; j0 += kPieceGroup) {
      uint32_t ri[kPieceGroup];
      T c[kPieceGroup];
#pragma unroll
      for (int q = 0; q < kPieceGroup; ++q) {
        ri[q] = __shfl_sync(0xffffffffu, my.x, (j0 + q) & 31);
        c[q] = __shfl_sync(0xffffffffu, my_c, (j0 + q) & 31);
      }
      if constexpr (WV_PIECE_ALL_LOADS == 1 || (WV_PIECE_ALL_LOADS == 2 && sizeof(T) == 8)) {
        // every chunk of the group's contributions in flight at once (more registers)
        Chunk<T, EPC> x[MAXC][kPieceGroup];
#pragma unroll
        for (int qq = 0; qq < MAXC; ++qq) {
          const int cc = lane + 32 * qq;
#pragma unroll
          for (int q = 0; q < kPieceGroup; ++q)
            if (cc < C && j0 + q < n) x[qq][q] = ld_chunk<T, EPC>(srcb + (size_t)ri[q] * d + cc * EPC);
        }
#pragma unroll
        for (int qq = 0; qq < MAXC; ++qq) {
          const int cc = lane + 32 * qq;
          if (cc < C) {
#pragma unroll
            for (int q = 0; q < kPieceGroup; ++q)
              if (j0 + q < n) {
#pragma unroll
                for (int e = 0; e < EPC; ++e)
                  g[qq].v[e] = add_rn(g[qq].v[e], side_out ? mul_rn(c[q], x[qq][q].v[e]) : x[qq][q].v[e]);
              }
          }
        }
        continue;
      }
#pragma unroll
      for (int qq = 0; qq < MAXC; ++qq) {
        const int cc = lane + 32 * qq;
        if (cc < C) {
          Chunk<T, EPC> x[kPieceGroup];
#pragma unroll
          for (int q = 0; q < kPieceGroup; ++q)
            if (j0 + q < n) x[q] = ld_chunk<T, EPC>(srcb + (size_t)ri[q] * d + cc * EPC);
#pragma unroll
          for (int q = 0; q < kPieceGroup; ++q)
            if (j0 + q < n) {
#pragma unroll
              for (int e = 0; e < EPC; ++e)
                g[qq].v[e] = add_rn(g[qq].v[e], side_out ? mul_rn(c[q], x[q].v[e]) : x[q].v[e]);
            }
        }
      }
    }
    if (np > 1) {
      // publish the piece partial; the warp finishing the row's last piece applies it
#pragma unroll
      for (int qq = 0; qq < MAXC; ++qq) {
        const int cc = lane + 32 * qq;
        if (cc < C) st_chunk<T, EPC>(partial + ((size_t)sg.pad + pd.y) * d + cc * EPC, g[qq]);
      }
      __threadfence();
      __syncwarp();
      uint32_t last = 0;
      if (lane == 0) last = atomicAdd(A.rowdone + pd.x, 1u) == np - 1 ? 1u : 0u;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (!last) return;
      __threadfence();
#pragma unroll
      for (int qq = 0; qq < MAXC; ++qq) {
        const int cc = lane + 32 * qq;
        if (cc < C) {
#pragma unroll
          for (int e = 0; e < EPC; ++e) g[qq].v[e] = 0;
          for (uint32_t t = 0; t < np; ++t) {
            const T* src = partial + ((size_t)sg.pad + t) * d + cc * EPC;
#pragma unroll
            for (int e = 0; e < EPC; ++e) g[qq].v[e] = add_rn(g[qq].v[e], __ldcg(src + e));
          }
        }
      }

    }
    const int64_t row = side_out ? (int64_t)sg.key - A.V : (int64_t)sg.key;
    T* P = (T*)(side_out ? A.out : A.in);
    T* M = (T*)(side_out ? A.m_out : A.m_in);
    T* Vv = (T*)(side_out ? A.v_out : A.v_in);
    const AdamBC<T> bc(sg.bc1, sg.bc2);
    bool changed = false;
#pragma unroll
    for (int qq = 0; qq < MAXC; ++qq) {
      const int cc = lane + 32 * qq;
      if (cc < C) {
        const int64_t o = row * d + (int64_t)cc * EPC;
        Chunk<T, EPC> p = ld_chunk_rw<T, EPC>(P + o), m = ld_chunk_rw<T, EPC>(M + o), vv = ld_chunk_rw<T, EPC>(Vv + o);
#pragma unroll
        for (int e = 0; e < EPC; ++e) changed |= adam_elem<T>(p.v[e], m.v[e], vv.v[e], g[qq].v[e], bc, lr) != T(0);
        st_chunk<T, EPC>(P + o, p);
        st_chunk<T, EPC>(M + o, m);
        st_chunk<T, EPC>(Vv + o, vv);
      }
    }
    changed = __any_sync(0xffffffffu, changed);
    if (lane == 0) {
      (side_out ? A.touched_out : A.touched_in)[row] = 1;
      if (changed) (side_out ? A.modified_out : A.modified_in)[row] = 1;
      A.cnt[sg.key] = 0;
      if (A.flag) A.flag[sg.key] = 0;
    }
  }
}

// Heavy pieces as their own kernel: a small footprint (WV_PIECE_GRID CTAs of
// WV_PIECE_THREADS) so it runs concurrently with the light-row owner.
template <typename T, int EPC, int MAXC>
__global__ void __launch_bounds__(WV_PIECE_THREADS) heavy_piece_kernel(OwnerArgs A) {
  const uint32_t np_total = *(volatile const uint32_t*)(A.gctr + GC_PIECES);
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t pc = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); pc < np_total; pc += warps)
    heavy_piece_work<T, EPC, MAXC>(A, pc);
}

// Phase 3c (split mode): RowAdam over every touched row, thread per 16-byte
// chunk.  The row gradients were summed by the owner kernels into gsum, so
// this pass is a pure stream of independent p/m/v/g loads and p/m/v stores
// (the access pattern that runs closest to HBM bandwidth).
template <typename T, int EPC, int MAXC>
__global__ void __launch_bounds__(256) sgns_adam_kernel(OwnerArgs A) {
  const int d = A.d;
  const int C = d / EPC;
  const uint32_t nl = A.seg_count[0], nh = A.seg_count[1];
  const int64_t total = (int64_t)(nl + nh) * C;
  const T lr = (T)A.lr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sgi = i / C;
    const int c = (int)(i - sgi * C);
    const bool heavy_row = sgi >= nl;
    const Segment sg = heavy_row ? A.heavy[sgi - nl] : A.segs[sgi];
    const int64_t grow = heavy_row ? A.n_items - 1 - (sgi - nl) : sgi;
    const bool side_out = sg.key >= (uint32_t)A.V;
    const int64_t row = side_out ? (int64_t)sg.key - A.V : (int64_t)sg.key;
    T* P = (T*)(side_out ? A.out : A.in);
    T* M = (T*)(side_out ? A.m_out : A.m_in);
    T* Vv = (T*)(side_out ? A.v_out : A.v_in);
    const int64_t o = row * d + (int64_t)c * EPC;
    Chunk<T, EPC> p = ld_chunk_rw<T, EPC>(P + o);
    Chunk<T, EPC> m = ld_chunk_rw<T, EPC>(M + o);
    Chunk<T, EPC> vv = ld_chunk_rw<T, EPC>(Vv + o);
    const Chunk<T, EPC> g = ld_chunk_rw<T, EPC>((const T*)A.gsum + grow * d + (int64_t)c * EPC);
    const AdamBC<T> bc(sg.bc1, sg.bc2);
    bool changed = false;
#pragma unroll
    for (int e = 0; e < EPC; ++e) changed |= adam_elem<T>(p.v[e], m.v[e], vv.v[e], g.v[e], bc, lr) != T(0);
    st_chunk<T, EPC>(P + o, p);
    st_chunk<T, EPC>(M + o, m);
    st_chunk<T, EPC>(Vv + o, vv);
    if (changed) (side_out ? A.modified_out : A.modified_in)[row] = 1;
  }
}

// Dense RowAdam (use_sparse=False, w2v.py:396-404): every row decays each
// batch with the global step; the staged gradient is consumed and zeroed.
template <typename T>
__global__ void dense_adam(T* __restrict__ P, T* __restrict__ M, T* __restrict__ Vv, T* __restrict__ Gd,
                           int64_t n, int d, const WvSgnsDevState* state, double lr, uint8_t* __restrict__ modified) {
  const int64_t t = state->step;  // already advanced for this batch
  const T bc1 = (T)(1.0 - pow(0.9, (double)t));
  const T bc2 = (T)(1.0 - pow(0.999, (double)t));
  const T b1 = (T)0.9, b2 = (T)0.999, omb1 = (T)(1.0 - 0.9), omb2 = (T)(1.0 - 0.999), eps = (T)1e-8, lrT = (T)lr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T gr = Gd[i];
    Gd[i] = 0;
    T m = add_rn(mul_rn(b1, M[i]), mul_rn(omb1, gr));
    T v = add_rn(mul_rn(b2, Vv[i]), mul_rn(mul_rn(omb2, gr), gr));
    M[i] = m;
    Vv[i] = v;
    const T upd = div_rn(mul_rn(lrT, div_rn(m, bc1)), add_rn(sqrt_rn(div_rn(v, bc2)), eps));
    const T p = P[i];
    const T np_ = sub_rn(p, upd);
    P[i] = np_;
    if (np_ != p || np_ != np_) modified[i / d] = 1;
  }
}

// ------------------------------------------------------------ init/export -
// Element k of the PCG64 stream SeedSequence([seed,1,0]) -> uniform(-1/d, 1/d).
// Thread per row: one jump, then d sequential steps.
__constant__ PcgJump c_pow2_sg[64];

__device__ __forceinline__ PcgJump jump_sg(uint64_t n) {
  PcgJump r{u128{1, 0}, u128{0, 0}};
  for (int b = 0; n; ++b, n >>= 1)
    if (n & 1) r = jump_compose(r, c_pow2_sg[b]);
  return r;
}

struct InitStream {
  u128 state, inc;
};

template <typename T>
__global__ void init_rows(InitStream g0, int64_t V, int d, int64_t row_begin, int64_t row_count, int matrix,
                          T* __restrict__ dst, const uint8_t* __restrict__ only_if_clear, double* __restrict__ dst64) {
  const double bound = 1.0 / (double)d;
  const double lower = -bound, range = bound - (-bound);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < row_count; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = row_begin + r;
    if (only_if_clear && only_if_clear[row]) continue;
    const uint64_t k0 = (uint64_t)matrix * (uint64_t)V * d + (uint64_t)row * d;
    PcgJump j = jump_sg(k0 + 1);
    u128 x = add128(mul128(j.A, g0.state), mul128(g0.inc, j.S));
    const u128 a1{PCG_MULT_LO, PCG_MULT_HI};
    for (int c = 0; c < d; ++c) {
      const double u = u64_to_double(pcg_output(x));
      const double val = __dadd_rn(lower, __dmul_rn(range, u));
      if (dst64) dst64[row * d + c] = val;
      else dst[row * d + c] = (T)val;
      x = add128(mul128(a1, x), g0.inc);
    }
  }
}

template <typename T>
__global__ void export_rows(const T* __restrict__ src, int64_t n, double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (double)src[i];
}

// ------------------------------------------------------- pair indexing ---
__global__ void walk_len_keys(const int64_t* __restrict__ offsets, int64_t n_walks, uint32_t* __restrict__ keys,
                              uint32_t* __restrict__ vals) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t L = offsets[w + 1] - offsets[w];
    keys[w] = (uint32_t)(L > 0xffffffffLL ? 0xffffffffLL : L);
    vals[w] = (uint32_t)w;
  }
}

__global__ void class_heads(const uint32_t* __restrict__ keys, int64_t n, uint8_t* __restrict__ head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void class_fill(const uint32_t* __restrict__ keys, int64_t n, const uint8_t* __restrict__ head,
                           const int64_t* __restrict__ cls, int64_t* __restrict__ class_len,
                           int64_t* __restrict__ class_walk_start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (head[i]) {
      class_len[cls[i]] = keys[i];
      class_walk_start[cls[i]] = i;
    }
}

__global__ void class_pairs(const int64_t* __restrict__ class_len, const int64_t* __restrict__ class_walk_start,
                            const int64_t* __restrict__ n_classes_p, int64_t n_walks, int window,
                            int64_t* __restrict__ class_pairs_out) {
  const int64_t nc = *n_classes_p;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t end = (c + 1 < nc) ? class_walk_start[c + 1] : n_walks;
    class_pairs_out[c] = (end - class_walk_start[c]) * walk_pairs(class_len[c], window);
  }
}

// Reference-order pair materialisation (generate_pairs, w2v.py:177-190):
// for s in 1..W: block A = (t[i], t[i+s]) over valid flat i, block B swapped.
// shift_start[s-1] = first output row of shift s; walk_prefix[s-1][w] =
// valid positions of shift s in walks before w.
__global__ void pairs_per_walk(const int64_t* __restrict__ offsets, int64_t n_walks, int s,
                               int64_t* __restrict__ cnt) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t L = offsets[w + 1] - offsets[w];
    cnt[w] = L > s ? L - s : 0;
  }
}

// CBOW instances (generate_cbow_instances, w2v.py:194-222): every token of a
// walk of length >= 2 is one instance, in corpus order.
__global__ void cbow_counts(const int64_t* __restrict__ offsets, int64_t n_walks, int64_t* __restrict__ cnt) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t L = offsets[w + 1] - offsets[w];
    cnt[w] = L >= 2 ? L : 0;
  }
}

__global__ void cbow_emit(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets, int64_t n_walks,
                          int window, const int64_t* __restrict__ base, int32_t* __restrict__ inst) {
  const int cols = 2 * window + 1;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = offsets[w], L = offsets[w + 1] - o;
    if (L < 2) continue;
    for (int64_t i = 0; i < L; ++i) {
      int32_t* row = inst + (base[w] + i) * cols;
      for (int s = 1; s <= window; ++s) {
        row[2 * (s - 1)] = i - s >= 0 ? tokens[o + i - s] : -1;
        row[2 * (s - 1) + 1] = i + s < L ? tokens[o + i + s] : -1;
      }
      row[2 * window] = tokens[o + i];
    }
  }
}

__global__ void pairs_emit(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets, int64_t n_walks,
                           int s, const int64_t* __restrict__ prefix, const int64_t* __restrict__ n_s_p,
                           int64_t block_base, int32_t* __restrict__ pairs) {
  const int64_t n_s = *n_s_p;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = offsets[w];
    const int64_t L = offsets[w + 1] - o;
    int64_t r = block_base + prefix[w];
    for (int64_t i = 0; i + s < L; ++i, ++r) {
      const int32_t a = tokens[o + i], b = tokens[o + i + s];
      pairs[2 * r] = a;
      pairs[2 * r + 1] = b;
      pairs[2 * (r + n_s)] = b;
      pairs[2 * (r + n_s) + 1] = a;
    }
  }
}

__global__ void state_reset_epoch(WvSgnsDevState* st, int64_t epoch, int64_t start) {
  st->lo = start;
  st->epoch = epoch;
  st->batch = 0;
  st->epoch_loss_sum = 0.0;
  st->epoch_count = 0;
  st->block_counter = 0;
}

__global__ void flags_to_candidates(const int64_t* __restrict__ freq, int64_t V, int64_t min_count,
                                    uint8_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    keep[i] = freq[i] >= min_count ? 1 : 0;
}

__global__ void scatter_candidates(const uint8_t* __restrict__ keep, const int64_t* __restrict__ pos, int64_t V,
                                   int32_t* __restrict__ cand) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    if (keep[i]) cand[pos[i]] = (int32_t)i;
}

// ------------------------------------------------------- row-sharded --
// Init of the rows this rank owns (global row l * nshard + shard -> local l),
// the same PCG64 elements as init_rows.
template <typename T>
__global__ void init_rows_shard(InitStream g0, int64_t V, int d, int64_t Vl, int nshard, int shard, int matrix,
                                T* __restrict__ dst) {
  const double bound = 1.0 / (double)d;
  const double lower = -bound, range = bound - (-bound);
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < Vl; l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = l * nshard + shard;
    if (row >= V) {
      for (int c = 0; c < d; ++c) dst[l * d + c] = (T)0;
      continue;
    }
    const uint64_t k0 = (uint64_t)matrix * (uint64_t)V * d + (uint64_t)row * d;
    PcgJump j = jump_sg(k0 + 1);
    u128 x = add128(mul128(j.A, g0.state), mul128(g0.inc, j.S));
    const u128 a1{PCG_MULT_LO, PCG_MULT_HI};
    for (int c = 0; c < d; ++c) {
      const double u = u64_to_double(pcg_output(x));
      dst[l * d + c] = (T)__dadd_rn(lower, __dmul_rn(range, u));
      x = add128(mul128(a1, x), g0.inc);
    }
  }
}

// Row requests of this rank's pairs, grouped by owner: pass 0 counts, pass 1
// places (global key = row or V + row, local item index).  ident[i] = item
// index, or -1 for a masked CBOW context column (no row).
__global__ void shard_requests(const int32_t* __restrict__ idx, int64_t item_begin, int64_t n_items, int R, int ctxw,
                               int64_t V, int nshard, int pass, uint32_t* __restrict__ cursor,
                               int64_t* __restrict__ keys, int32_t* __restrict__ items,
                               int32_t* __restrict__ ident) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_items; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = item_begin + i;
    const int j = (int)(gi % R);
    const int32_t t = idx[gi];
    if (pass == 1) ident[i] = t >= 0 ? (int32_t)i : -1;
    if (t < 0) continue;
    const int owner = (int)((uint32_t)t % (uint32_t)nshard);
    const uint32_t at = atomicAdd(cursor + owner, 1u);
    if (pass == 1) {
      keys[at] = (int64_t)t + (j < ctxw ? 0 : V);
      items[at] = (int32_t)i;
    }
  }
}

// requests of a skip-gram batch per (requesting rank, owning rank), from decoded
// rows [rows, R]: pair b belongs to requester b / bl (shard.py's pair shares),
// each of its R rows to owner row % nshard.  Lets every rank know every split
// size of the batch's all-to-alls without exchanging counts (shard lookahead).
__global__ void shard_count_matrix(const int32_t* __restrict__ rows_idx, int64_t rows, int R, int64_t bl,
                                   int nshard, unsigned long long* __restrict__ counts) {
  __shared__ unsigned int local[64 * 64];
  const int nn = nshard * nshard;
  for (int i = threadIdx.x; i < nn; i += blockDim.x) local[i] = 0;
  __syncthreads();
  const int64_t n = rows * R;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = rows_idx[i];
    if (t < 0) continue;
    const int s = (int)((i / R) / bl);
    atomicAdd(local + s * nshard + (int)((uint32_t)t % (uint32_t)nshard), 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nn; i += blockDim.x)
    if (local[i]) atomicAdd(counts + i, (unsigned long long)local[i]);
}

__global__ void shard_offsets(uint32_t* cursor, int nshard, int64_t* counts) {
  // cursor[0..n) holds counts after pass 0: copy them out, turn the cursor into offsets
  uint32_t run = 0;
  for (int o = 0; o < nshard; ++o) {
    const uint32_t c = cursor[o];
    counts[o] = c;
    cursor[o] = run;
    run += c;
  }
}

template <typename T>
__global__ void shard_serve(const T* __restrict__ in, const T* __restrict__ out, const int64_t* __restrict__ keys,
                            int64_t n, int64_t V, int nshard, int d, T* __restrict__ rows) {
  const int C = d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * C; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = i / C;
    const int c = (int)(i - q * C);
    const int64_t key = keys[q];
    const bool side = key >= V;
    const int64_t local = (side ? key - V : key) / nshard;
    rows[i] = (side ? out : in)[local * d + c];
  }
}

template <typename T>
__global__ void shard_place(const T* __restrict__ rows, const int32_t* __restrict__ items, int64_t n, int d,
                            T* __restrict__ itemrows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * d; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = i / d;
    itemrows[(int64_t)items[q] * d + (i - q * d)] = rows[i];
  }
}

static inline unsigned grid_for(int64_t n, int threads, int64_t cap = 148 * 32) {
  int64_t g = (n + threads - 1) / threads;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

static inline int64_t al256(int64_t b) { return (b + 255) & ~(int64_t)255; }

// per-device bias-correction table (built outside any graph capture: at
// workspace init, or on first use by an uncaptured batch)
static double2* g_bc_table[16] = {nullptr};
static cudaError_t bc_table(double2** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
  if (g_bc_table[dev] == nullptr) {
    double2* t = nullptr;
    e = cudaMalloc(&t, sizeof(double2) * kBcTable);
    if (e != cudaSuccess) return e;
    fill_bc_table<<<kBcTable / 256, 256>>>(t);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return e;
    g_bc_table[dev] = t;
  }
  *out = g_bc_table[dev];
  return cudaSuccess;
}

static uint64_t g_sg_table_ready = 0;
static cudaError_t ensure_sg_table() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64 && (g_sg_table_ready >> dev) & 1) return cudaSuccess;
  PcgJump tab[64];
  pcg_jump_table(tab, 64);
  e = cudaMemcpyToSymbol(c_pow2_sg, tab, sizeof(tab));
  if (e == cudaSuccess && dev < 64) g_sg_table_ready |= (1ull << dev);
  return e;
}

// dispatch helper: (T, EPC, MAXC) from (precision, d)
template <template <typename, int, int> class F, typename... Args>
static int dispatch_rows(int precision, int d, Args&&... args) {
  if (precision == WV_FP32) {
    if (d % 4 == 0) {
      const int C = d / 4;
      if (C <= 32) return F<float, 4, 1>::run(args...);
      if (C <= 64) return F<float, 4, 2>::run(args...);
      if (C <= 128) return F<float, 4, 4>::run(args...);
      if (C <= 256) return F<float, 4, 8>::run(args...);
    } else {
      if (d <= 32) return F<float, 1, 1>::run(args...);
      if (d <= 64) return F<float, 1, 2>::run(args...);
      if (d <= 128) return F<float, 1, 4>::run(args...);
      if (d <= 256) return F<float, 1, 8>::run(args...);
    }
  } else if (precision == WV_FP64) {
    if (d % 2 == 0) {
      const int C = d / 2;
      if (C <= 32) return F<double, 2, 1>::run(args...);
      if (C <= 64) return F<double, 2, 2>::run(args...);
      if (C <= 128) return F<double, 2, 4>::run(args...);
      if (C <= 256) return F<double, 2, 8>::run(args...);
    } else {
      if (d <= 32) return F<double, 1, 1>::run(args...);
      if (d <= 64) return F<double, 1, 2>::run(args...);
      if (d <= 128) return F<double, 1, 4>::run(args...);
      if (d <= 256) return F<double, 1, 8>::run(args...);
    }
  }
  set_error("unsupported precision %d / vector_size %d", precision, d);
  return -1;
}

// shared memory of the bulk gather: barriers + per-warp ring of R rows per stage
static inline size_t bulk_smem_bytes(int nw, int d, int R, size_t es, int stages = kBulkStages) {
  return 16 * nw * stages + (size_t)nw * stages * R * d * es;
}
static constexpr size_t kBulkSmemMax = 220 * 1024;

// one bulk-gather instantiation: smem attribute, persistent grid of resident CTAs
template <typename T, int EPC, int MAXC, bool CB, int NW, int KC = 0, int ST = kBulkStages>
static int launch_bulk_gather(const PairArgs& a, const void* in, const void* out, size_t smem, cudaStream_t st) {
  auto kern = sgns_gather_bulk_kernel<T, EPC, MAXC, CB, NW, KC, ST>;
  static size_t attr_set[16] = {0};
  static int resident[16] = {0};
  static size_t resident_smem[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  if (dev >= 0 && dev < 16) {
    if (attr_set[dev] < smem) {
      WV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_set[dev] = smem;
    }
    if (resident[dev] == 0 || resident_smem[dev] != smem) {
      int nb = 0;
      WV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, NW * 32, smem));
      resident[dev] = nb > 0 ? nb : 1;
      resident_smem[dev] = smem;
    }
    WV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int64_t blocks = (a.B + NW - 1) / NW;
  const int64_t cap = (int64_t)sms * (dev >= 0 && dev < 16 ? resident[dev] : 4);
  const unsigned g = (unsigned)(blocks < cap ? blocks : cap);
  kern<<<g, NW * 32, smem, st>>>(a, (const T*)in, (const T*)out);
  WV_LAUNCH_CHECK();
  return 0;
}

template <typename T, int EPC, int MAXC>
struct LaunchPair {
  // register path: negatives gathered per group, as many as fit in registers
  static constexpr int NG = MAXC <= 2 ? 5 : (MAXC <= 4 ? 2 : 1);
  static int run(const PairArgs& a, const void* in, const void* out, unsigned grid, cudaStream_t st) {
    const bool rows16 = (a.d * sizeof(T)) % 16 == 0 && EPC * sizeof(T) == 16;
    if (a.cw > 0) {
      // CBOW: bulk path only, warps per CTA chosen so the ring fits in shared memory
      WV_CHECK_ARG(rows16, "CBOW needs vector_size * element size to be a multiple of 16 bytes");
      for (int nw : {8, 4, 2, 1}) {
        const size_t smem = bulk_smem_bytes(nw, a.d, a.R, sizeof(T));
        if (smem > kBulkSmemMax) continue;
        if (nw == 8) return launch_bulk_gather<T, EPC, MAXC, true, 8>(a, in, out, smem, st);
        if (nw == 4) return launch_bulk_gather<T, EPC, MAXC, true, 4>(a, in, out, smem, st);
        if (nw == 2) return launch_bulk_gather<T, EPC, MAXC, true, 2>(a, in, out, smem, st);
        return launch_bulk_gather<T, EPC, MAXC, true, 1>(a, in, out, smem, st);
      }
      set_error("CBOW window too large for the shared-memory ring (vector_size %d)", a.d);
      return -1;
    }
    const size_t smem = bulk_smem_bytes(kBulkWarps, a.d, 2 + a.k, sizeof(T));
    if (rows16 && smem <= kBulkSmemMax && getenv("WV_SGNS_REG_GATHER") == nullptr) {
      if (a.k == 5) return launch_bulk_gather<T, EPC, MAXC, false, kBulkWarps, 5>(a, in, out, smem, st);
      return launch_bulk_gather<T, EPC, MAXC, false, kBulkWarps>(a, in, out, smem, st);
    }
    // wide rows (float64, large vector_size): half the warps per CTA keep the ring in shared memory
    const size_t smem_h = bulk_smem_bytes(kBulkWarpsWide, a.d, 2 + a.k, sizeof(T), kBulkStagesWide);
    if (rows16 && smem_h <= kBulkSmemMax && getenv("WV_SGNS_REG_GATHER") == nullptr) {
      if (a.k == 5)
        return launch_bulk_gather<T, EPC, MAXC, false, kBulkWarpsWide, 5, kBulkStagesWide>(a, in, out, smem_h, st);
      return launch_bulk_gather<T, EPC, MAXC, false, kBulkWarpsWide, 0, kBulkStagesWide>(a, in, out, smem_h, st);
    }
    const size_t smem_h2 = bulk_smem_bytes(kBulkWarpsWide2, a.d, 2 + a.k, sizeof(T), kBulkStagesWide2);
    if (rows16 && smem_h2 <= kBulkSmemMax && getenv("WV_SGNS_REG_GATHER") == nullptr) {
      if (a.k == 5)
        return launch_bulk_gather<T, EPC, MAXC, false, kBulkWarpsWide2, 5, kBulkStagesWide2>(a, in, out, smem_h2, st);
      return launch_bulk_gather<T, EPC, MAXC, false, kBulkWarpsWide2, 0, kBulkStagesWide2>(a, in, out, smem_h2, st);
    }
    sgns_gather_kernel<T, EPC, MAXC, NG><<<grid, kPairThreads, 0, st>>>(a, (const T*)in, (const T*)out);
    WV_LAUNCH_CHECK();
    return 0;
  }
};

// Streams and events of the batch pipeline (per host thread and device):
//   side  : decode + grouping of batch i+1 while the main stream runs batch i
//   heavy : the CTA-per-heavy-row kernel, concurrent with the light-row owner
// Works eagerly and under CUDA-graph capture: every side-stream segment forks
// from and joins back into the caller's stream through these events.
#ifndef WV_SIDE_AFTER_GATHER
#define WV_SIDE_AFTER_GATHER 0
#endif
struct SideStream {
  int dev = -1;
  cudaStream_t s = nullptr, h = nullptr, b = nullptr;  // b: the split owner's B rows
  cudaEvent_t fork = nullptr, join = nullptr, fork_h = nullptr, join_h = nullptr, fork_b = nullptr;
  cudaEvent_t dec[2] = {nullptr, nullptr}, grp[2] = {nullptr, nullptr}, own[2] = {nullptr, nullptr};
  cudaEvent_t bdone[2] = {nullptr, nullptr};
  cudaEvent_t gdone = nullptr;  // the current batch's gather is done (side-after-gather schedule)
};

static cudaError_t side_stream(SideStream** out) {
  static thread_local SideStream tab[16];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
  SideStream& ss = tab[dev];
  if (ss.s == nullptr) {
    // the side stream (next batch's decode + grouping) gets the highest priority so
    // its CTAs take SM slots as soon as any free up during the current batch
    int lo_prio = 0, hi_prio = 0;
    e = cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
#ifndef WV_SIDE_PRIO
#define WV_SIDE_PRIO 1
#endif
#ifndef WV_HEAVY_PRIO
#define WV_HEAVY_PRIO WV_SINGLES_CONCURRENT
#endif
    if (e == cudaSuccess)
      e = cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, WV_SIDE_PRIO ? hi_prio : lo_prio);
    if (e == cudaSuccess)
      e = cudaStreamCreateWithPriority(&ss.h, cudaStreamNonBlocking, WV_HEAVY_PRIO ? hi_prio : lo_prio);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&ss.b, cudaStreamNonBlocking, lo_prio);
    cudaEvent_t* evs[] = {&ss.fork, &ss.join, &ss.fork_h, &ss.join_h, &ss.fork_b, &ss.dec[0], &ss.dec[1],
                          &ss.grp[0], &ss.grp[1], &ss.own[0], &ss.own[1], &ss.bdone[0], &ss.bdone[1],
                          &ss.gdone};
    for (cudaEvent_t* ev : evs)
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    ss.dev = dev;
  }
  *out = &ss;
  return cudaSuccess;
}

// Workspace of one SGNS replica.  The buffers a batch's decode and grouping
// write come in two halves (by batch parity) so batch i+1 can be decoded and
// grouped while batch i is still being applied; each half holds persistent
// per-row counters (zero between batches).  U, G and the coefficients are
// produced and consumed on the main stream and need one copy.  With
// base == nullptr only the size is computed.
struct BatchHalf {
  uint32_t* cnt;
  uint32_t* gctr;
  int32_t* idx;
  uint32_t* uniq;
  uint32_t* list;
  uint32_t* list_tmp;
  Segment* segs;
  Segment* heavy;
  uint2* ents;
  uint2* pieces;     // heavy-row pieces (row, piece index)
  void* partial;     // [max_pieces, d] piece partial sums
  uint32_t* rowdone; // per heavy row: pieces finished (zero between batches)
  uint32_t* rank;    // [items] claim rank of each item within its row
  uint8_t* flag;     // [2V] 1 for every row key this half's batch touches (set by decode, cleared by the owner)
  Segment* segs2;    // light segments regrouped: rows the next batch also touches first (split owner)
  Segment* singles;  // single-contribution rows (the lean owner)
};

struct BatchWs {
  CorpusDesc* desc;
  void* U[2];  // per half: batch i's update reads half i&1 while batch i+1's gather writes the other
  void* G[2];
  void* coef[2];
  double* partials;
  void* gsum;
  BatchHalf half[2];
};

static bool split_adam_requested() { return getenv("WV_SGNS_SPLIT_ADAM") != nullptr; }

// rows per item: 2 + k (skip-gram) or 2W + 1 + k (CBOW)
static inline int rows_per_item(int k, int cbow_window) { return cbow_window > 0 ? 2 * cbow_window + 1 + k : 2 + k; }

static int64_t carve_batch_ws(char* base, int64_t V, int d, int k, int R, int64_t B, int64_t es, BatchWs& w) {
  const int64_t items = B * R;
  int64_t off = 0;
  auto take = [&](int64_t bytes) -> void* {
    void* p = base ? base + off : nullptr;
    off += al256(bytes);
    return p;
  };
  // the descriptor and the persistent counters sit at offsets that do not
  // depend on B, so a short final batch sees the same ones
  w.desc = (CorpusDesc*)take(sizeof(CorpusDesc));
  for (int h = 0; h < 2; ++h) w.half[h].cnt = (uint32_t*)take(2 * V * 4);
  for (int h = 0; h < 2; ++h) w.half[h].flag = (uint8_t*)take(2 * V);
  for (int h = 0; h < 2; ++h) {
    w.U[h] = take(B * d * es);
    w.G[h] = take(B * d * es);
    w.coef[h] = take(B * (k + 1) * es);
  }
  w.partials = (double*)take(148 * 32 * 8);
  w.gsum = split_adam_requested() ? take(items * d * es) : nullptr;
  for (int h = 0; h < 2; ++h) {
    BatchHalf& x = w.half[h];
    x.gctr = (uint32_t*)take(64);
    x.idx = (int32_t*)take(items * 4);
    x.uniq = (uint32_t*)take(items * 4);
    x.list = (uint32_t*)take(items * 4);
    x.list_tmp = (uint32_t*)take(items * 4);
    x.segs = (Segment*)take(items * (int64_t)sizeof(Segment));
    x.heavy = (Segment*)take((items / (kLightMax + 1) + 1) * (int64_t)sizeof(Segment));
    x.ents = (uint2*)take(items * 8);
    x.pieces = (uint2*)take(max_pieces(items) * 8);
    x.partial = take(max_pieces(items) * d * es);
    x.rowdone = (uint32_t*)take((items / (kLightMax + 1) + 1) * 4);  // zeroed per batch with gctr
    x.rank = (uint32_t*)take(items * 4);
    x.segs2 = (Segment*)take(items * (int64_t)sizeof(Segment));
    x.singles = (Segment*)take(items * (int64_t)sizeof(Segment));
  }
  return off + 1024;
}

static CorpusDesc make_desc(const WvSgnsBatch* b) {
  CorpusDesc c;
  c.mode = b->mode;
  c.window = b->window;
  c.n_classes = (int)b->n_classes;
  c.model = b->model;
  c.N = b->n_pairs;
  c.seed = b->seed;
  c.tokens = b->tokens;
  c.offsets = b->offsets;
  c.class_len = b->class_len;
  c.class_pair_start = b->class_pair_start;
  c.class_walk_start = b->class_walk_start;
  c.walks_by_class = b->walks_by_class;
  c.candidates = b->candidates;
  c.n_candidates = b->n_candidates;
  c.pairs = b->pairs;
  c.perm = b->perm;
  c.negatives = b->negative_table;
  c.inst = b->instances;
  return c;
}

template <typename T, int EPC, int MAXC>
struct LaunchAdam {
  static int run(const OwnerArgs& a, unsigned grid, cudaStream_t st) {
    sgns_adam_kernel<T, EPC, MAXC><<<grid, 256, 0, st>>>(a);
    WV_LAUNCH_CHECK();
    return 0;
  }
};

template <typename T, int EPC, int MAXC>
struct LaunchHeavy {
  static int run(const OwnerArgs& a, unsigned grid, cudaStream_t st) {
    const size_t smem = (kHeavyThreads / 32) * a.d * sizeof(T) + (size_t)heavy_bitmap_words(a.n_items) * 4;
    static bool attr_set[16] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 16 && !attr_set[dev]) {
      WV_CUDA(cudaFuncSetAttribute(sgns_heavy_kernel<T, EPC, MAXC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)((kHeavyThreads / 32) * 256 * 8 + kBitmapMaxWords * 4)));
      attr_set[dev] = true;
    }
    sgns_heavy_kernel<T, EPC, MAXC><<<grid, kHeavyThreads, smem, st>>>(a);
    WV_LAUNCH_CHECK();
    return 0;
  }
};

template <typename T, int EPC, int MAXC>
struct LaunchOwner {
  static int run(const OwnerArgs& a0, unsigned grid, cudaStream_t st) {
    OwnerArgs a = a0;
    if (a.ents != nullptr) {  // flat owner (group_order ran): persistent grid of resident CTAs
      const uint32_t C = (uint32_t)(a.d / EPC);
      a.cmag = C > 1 ? (uint32_t)(0xFFFFFFFFull / C + 1ull) : 0xFFFFFFFFu;
      static int resident[16] = {0};
      int dev = 0;
      cudaGetDevice(&dev);
      int sms = 148;
      if (dev >= 0 && dev < 16) {
        if (resident[dev] == 0) {
          int nb = 0;
          WV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sgns_owner_flat_kernel<T, EPC, MAXC>, 256, 0));
          resident[dev] = nb > 0 ? nb : 1;
        }
        WV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      }
      int per = dev >= 0 && dev < 16 ? resident[dev] : 4;
      const int resident_per = per;
      if (WV_OWNER_PER_SM > 0 && per > WV_OWNER_PER_SM) per = WV_OWNER_PER_SM;
      if (grid >= 1000) per = min(resident_per, (int)grid - 1000);  // the caller's CTAs per SM (serial heavy)
      else if (grid > 0 && (int)grid < per) per = (int)grid;  // caller's cap (split owner part B)
      const unsigned g = (unsigned)(sms * per);
      sgns_owner_flat_kernel<T, EPC, MAXC><<<g, 256, 0, st>>>(a);
      WV_LAUNCH_CHECK();
      return 0;
    }
    const size_t smem = 128 + (size_t)kOwnerBulkWarps * 2 * kOwnerBulkRows * a.d * sizeof(T);
    if (a.sparse && !a.split && (a.d * sizeof(T)) % 16 == 0 && EPC * sizeof(T) == 16 && smem <= 112 * 1024 &&
        getenv("WV_SGNS_REG_OWNER") == nullptr) {
      static bool attr_set[16] = {false};
      static int resident[16] = {0};
      int dev = 0;
      cudaGetDevice(&dev);
      int sms = 148;
      if (dev >= 0 && dev < 16) {
        if (!attr_set[dev]) {
          WV_CUDA(cudaFuncSetAttribute(sgns_owner_bulk_kernel<T, EPC, MAXC>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
          int nb = 0;
          WV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sgns_owner_bulk_kernel<T, EPC, MAXC>,
                                                                 kOwnerBulkWarps * 32, smem));
          resident[dev] = nb > 0 ? nb : 1;
          attr_set[dev] = true;
        }
        WV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      }
      const unsigned g = (unsigned)(sms * (dev >= 0 && dev < 16 ? resident[dev] : 2));
      sgns_owner_bulk_kernel<T, EPC, MAXC><<<g, kOwnerBulkWarps * 32, smem, st>>>(a);
      WV_LAUNCH_CHECK();
      return 0;
    }
    sgns_owner_kernel<T, EPC, MAXC><<<grid, kOwnerThreads, 0, st>>>(a);
    WV_LAUNCH_CHECK();
    return 0;
  }
};

}  // namespace wv

extern "C" {

int wv_sgns_init(int64_t vocab_size, int vector_size, const uint32_t* seed_prefix, int n_prefix, int precision,
                 void* input_matrix, void* output_matrix, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(vocab_size >= 1 && vector_size >= 1, "bad sizes");
  WV_CHECK_ARG(precision == WV_FP32 || precision == WV_FP64, "bad precision");
  WV_CUDA(ensure_sg_table());
  uint32_t pool[4];
  ss_pool(seed_prefix, n_prefix - 1, seed_prefix[n_prefix - 1], pool);
  Pcg64 g = pcg_seed(pool);
  InitStream s{g.state, g.inc};
  cudaStream_t st = (cudaStream_t)stream;
  for (int mtx = 0; mtx < 2; ++mtx) {
    void* dst = mtx == 0 ? input_matrix : output_matrix;
    if (precision == WV_FP32)
      init_rows<float><<<grid_for(vocab_size, 128), 128, 0, st>>>(s, vocab_size, vector_size, 0, vocab_size, mtx,
                                                                  (float*)dst, nullptr, nullptr);
    else
      init_rows<double><<<grid_for(vocab_size, 128), 128, 0, st>>>(s, vocab_size, vector_size, 0, vocab_size, mtx,
                                                                   nullptr, nullptr, (double*)dst);
    WV_LAUNCH_CHECK();
  }
  return 0;
}

// float64 export of one matrix (0 = input, 1 = output): modified rows are
// cast from the parameter store, all others are regenerated bit-exactly
// from the init stream (so untouched rows equal init_embeddings exactly).
int wv_sgns_export(int64_t vocab_size, int vector_size, const uint32_t* seed_prefix, int n_prefix, int precision,
                   int matrix, const void* params, const uint8_t* modified, double* out64, void* stream) {
  using namespace wv;
  WV_CUDA(ensure_sg_table());
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = vocab_size * (int64_t)vector_size;
  if (precision == WV_FP64) {
    WV_CUDA(cudaMemcpyAsync(out64, params, n * 8, cudaMemcpyDeviceToDevice, st));
    return 0;
  }
  export_rows<float><<<grid_for(n, 256), 256, 0, st>>>((const float*)params, n, out64);
  WV_LAUNCH_CHECK();
  uint32_t pool[4];
  ss_pool(seed_prefix, n_prefix - 1, seed_prefix[n_prefix - 1], pool);
  Pcg64 g = pcg_seed(pool);
  InitStream s{g.state, g.inc};
  init_rows<float><<<grid_for(vocab_size, 128), 128, 0, st>>>(s, vocab_size, vector_size, 0, vocab_size, matrix,
                                                              nullptr, modified, out64);
  WV_LAUNCH_CHECK();
  return 0;
}

int64_t wv_pair_index_workspace_bytes(int64_t n_walks) {
  using namespace wv;
  return al256(n_walks * 4) * 2 + al256(radix_ws_bytes(n_walks, 32)) + al256(n_walks) + al256((n_walks + 1) * 8) * 2 +
         al256(scan_tiles(n_walks + 1) * 8) + 1024;
}

// Length-class index of a flat corpus for O(1) pair decode:
// walks_by_class (stable by length), class_len/class_walk_start/class_pair_start
// (each sized n_walks+1 by the caller), *n_classes and *n_pairs (device int64).
int wv_pair_index_build(const int64_t* offsets, int64_t n_walks, int window, int32_t* walks_by_class,
                        int64_t* class_len, int64_t* class_walk_start, int64_t* class_pair_start, int64_t* n_classes,
                        int64_t* n_pairs, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(window >= 1, "window must be >= 1");
  WV_CHECK_ARG(n_walks >= 1 && n_walks < (1ll << 31), "bad walk count");
  WV_CHECK_ARG(ws_bytes >= wv_pair_index_workspace_bytes(n_walks), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  uint32_t* keys = (uint32_t*)w;
  w += al256(n_walks * 4);
  uint32_t* vals = (uint32_t*)walks_by_class;
  w += al256(n_walks * 4);  // (radix scratch values live in rws)
  void* rws = w;
  w += al256(radix_ws_bytes(n_walks, 32));
  uint8_t* head = (uint8_t*)w;
  w += al256(n_walks);
  int64_t* cls = (int64_t*)w;
  w += al256((n_walks + 1) * 8);
  int64_t* cpairs = (int64_t*)w;
  w += al256((n_walks + 1) * 8);
  int64_t* scan_ws = (int64_t*)w;
  walk_len_keys<<<grid_for(n_walks, 256), 256, 0, st>>>(offsets, n_walks, keys, vals);
  WV_LAUNCH_CHECK();
  WV_CUDA(radix_sort_pairs(keys, vals, n_walks, 32, rws, st));
  class_heads<<<grid_for(n_walks, 256), 256, 0, st>>>(keys, n_walks, head);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<uint8_t, int64_t>(head, n_walks, cls, n_classes, scan_ws, st)));
  class_fill<<<grid_for(n_walks, 256), 256, 0, st>>>(keys, n_walks, head, cls, class_len, class_walk_start);
  WV_CUDA(cudaMemsetAsync(cpairs, 0, n_walks * 8, st));
  class_pairs<<<grid_for(n_walks, 256), 256, 0, st>>>(class_len, class_walk_start, n_classes, n_walks, window,
                                                       cpairs);
  WV_LAUNCH_CHECK();
  // class_pair_start = exclusive scan over the (n_classes) entries; entries
  // past n_classes are never read (the kernel is bounded by n_classes).
  WV_CUDA((excl_scan<int64_t, int64_t>(cpairs, n_walks, class_pair_start, n_pairs, scan_ws, st)));
  return 0;
}

int64_t wv_pairs_workspace_bytes(int64_t n_walks) {
  using namespace wv;
  return al256(n_walks * 8) * 2 + al256(scan_tiles(n_walks) * 8) + al256(8) + 256;
}

// Reference-order (N,2) pair table (generate_pairs, w2v.py:161-191).  The
// caller sizes `pairs` from wv_pair_index_build's n_pairs.
int wv_generate_pairs(const int32_t* tokens, const int64_t* offsets, int64_t n_walks, int window, int32_t* pairs,
                      int64_t* n_pairs_out, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(ws_bytes >= wv_pairs_workspace_bytes(n_walks), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  int64_t* cnt = (int64_t*)w;
  w += al256(n_walks * 8);
  int64_t* prefix = (int64_t*)w;
  w += al256(n_walks * 8);
  int64_t* scan_ws = (int64_t*)w;
  w += al256(scan_tiles(n_walks) * 8);
  int64_t* n_s = (int64_t*)w;
  // host needs block bases; shift counts are read back synchronously
  int64_t base = 0;
  for (int s = 1; s <= window; ++s) {
    pairs_per_walk<<<grid_for(n_walks, 256), 256, 0, st>>>(offsets, n_walks, s, cnt);
    WV_LAUNCH_CHECK();
    WV_CUDA((excl_scan<int64_t, int64_t>(cnt, n_walks, prefix, n_s, scan_ws, st)));
    int64_t ns_host = 0;
    WV_CUDA(cudaMemcpyAsync(&ns_host, n_s, 8, cudaMemcpyDeviceToHost, st));
    WV_CUDA(cudaStreamSynchronize(st));
    if (ns_host == 0) break;
    if (pairs)
      pairs_emit<<<grid_for(n_walks, 128), 128, 0, st>>>(tokens, offsets, n_walks, s, prefix, n_s, base, pairs);
    WV_LAUNCH_CHECK();
    base += 2 * ns_host;
  }
  *n_pairs_out = base;
  return 0;
}

int64_t wv_cbow_instances_workspace_bytes(int64_t n_walks) {
  using namespace wv;
  return al256(n_walks * 8) * 2 + al256(scan_tiles(n_walks) * 8) + 256;
}

int wv_cbow_instances(const int32_t* tokens, const int64_t* offsets, int64_t n_walks, int window, int32_t* instances,
                      int64_t* n_instances, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(window >= 1, "window must be >= 1");
  WV_CHECK_ARG(n_walks >= 1, "empty corpus");
  WV_CHECK_ARG(ws_bytes >= wv_cbow_instances_workspace_bytes(n_walks), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  int64_t* cnt = (int64_t*)w;
  w += al256(n_walks * 8);
  int64_t* base = (int64_t*)w;
  w += al256(n_walks * 8);
  int64_t* scan_ws = (int64_t*)w;
  cbow_counts<<<grid_for(n_walks, 256), 256, 0, st>>>(offsets, n_walks, cnt);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<int64_t, int64_t>(cnt, n_walks, base, n_instances, scan_ws, st)));
  if (instances) {
    cbow_emit<<<grid_for(n_walks, 128), 128, 0, st>>>(tokens, offsets, n_walks, window, base, instances);
    WV_LAUNCH_CHECK();
  }
  return 0;
}

int64_t wv_candidates_workspace_bytes(int64_t vocab_size) {
  using namespace wv;
  return al256(vocab_size) + al256(vocab_size * 8) + al256(scan_tiles(vocab_size) * 8) + 256;
}

// candidates = flatnonzero(freq >= min_count) (w2v.py:525-526); keep mask out.
int wv_candidates(const int64_t* freq, int64_t vocab_size, int64_t min_count, uint8_t* keep, int32_t* candidates,
                  int64_t* n_candidates, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(ws_bytes >= wv_candidates_workspace_bytes(vocab_size), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  w += al256(vocab_size);
  int64_t* pos = (int64_t*)w;
  w += al256(vocab_size * 8);
  int64_t* scan_ws = (int64_t*)w;
  flags_to_candidates<<<grid_for(vocab_size, 256), 256, 0, st>>>(freq, vocab_size, min_count, keep);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<uint8_t, int64_t>(keep, vocab_size, pos, n_candidates, scan_ws, st)));
  scatter_candidates<<<grid_for(vocab_size, 256), 256, 0, st>>>(keep, pos, vocab_size, candidates);
  WV_LAUNCH_CHECK();
  return 0;
}

int wv_sgns_decode(const WvSgnsBatch* batch, int64_t epoch, int64_t pos_begin, int64_t n, int32_t* rows,
                   int64_t* pair_index, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(batch != nullptr && rows != nullptr, "null argument");
  WV_CHECK_ARG(batch->model == WV_MODEL_SKIPGRAM, "wv_sgns_decode: skip-gram batches only");
  WV_CHECK_ARG(n >= 0 && pos_begin >= 0 && pos_begin + n <= batch->n_pairs, "positions out of range");
  if (n == 0) return 0;
  const CorpusDesc D = make_desc(batch);
  sgns_decode_positions<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(D, batch->negatives, epoch, pos_begin, n,
                                                                           rows, pair_index);
  WV_LAUNCH_CHECK();
  return 0;
}

int wv_sgns_epoch_begin(WvSgnsDevState* state, int64_t epoch, int64_t start, void* stream) {
  using namespace wv;
  state_reset_epoch<<<1, 1, 0, (cudaStream_t)stream>>>(state, epoch, start);
  WV_LAUNCH_CHECK();
  return 0;
}

int64_t wv_sgns_batch_workspace_bytes(int64_t vocab_size, int vector_size, int negatives, int64_t batch,
                                      int precision, int cbow_window) {
  using namespace wv;
  BatchWs bw;
  return carve_batch_ws(nullptr, vocab_size, vector_size, negatives, rows_per_item(negatives, cbow_window), batch,
                        precision == WV_FP64 ? 8 : 4, bw);
}

// Zero the workspace's persistent per-row counters; required once after the
// workspace is allocated (every batch leaves them zero again).
int wv_sgns_workspace_init(void* ws, int64_t ws_bytes, int64_t vocab_size, int vector_size, int negatives,
                           int64_t batch, int precision, int cbow_window, void* stream) {
  using namespace wv;
  BatchWs bw;
  const int64_t need = carve_batch_ws((char*)ws, vocab_size, vector_size, negatives,
                                      rows_per_item(negatives, cbow_window), batch, precision == WV_FP64 ? 8 : 4, bw);
  WV_CHECK_ARG(ws_bytes >= need, "workspace too small");
  for (int h = 0; h < 2; ++h) WV_CUDA(cudaMemsetAsync(bw.half[h].cnt, 0, 2 * vocab_size * 4, (cudaStream_t)stream));
  double2* bct = nullptr;
  WV_CUDA(bc_table(&bct));  // before any CUDA-graph capture of batches
  return 0;
}

// Write the corpus side of `batch` into the workspace (stream-ordered).  A
// CUDA graph of batches captured against this workspace then trains on the
// newly bound corpus when replayed.  wv_sgns_batch binds by itself when its
// stream is not being captured.
int wv_sgns_bind(const WvSgnsBatch* batch, void* ws, int64_t ws_bytes, int64_t vocab_size, int vector_size,
                 int precision, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(batch->mode == WV_PAIRS_NATIVE || batch->mode == WV_PAIRS_EXPLICIT, "bad pair mode");
  BatchWs bw;
  const int cw = batch->model == WV_MODEL_CBOW ? batch->window : 0;
  const int64_t need = carve_batch_ws((char*)ws, vocab_size, vector_size, batch->negatives,
                                      rows_per_item(batch->negatives, cw), batch->batch_rows,
                                      precision == WV_FP64 ? 8 : 4, bw);
  WV_CHECK_ARG(ws_bytes >= need, "workspace too small");
  const CorpusDesc c = make_desc(batch);
  WV_CUDA(cudaMemcpyAsync(bw.desc, &c, sizeof(c), cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return 0;
}

}  // extern "C"

namespace wv {

// Everything one batch needs, resolved once per call.
struct BatchCtx {
  const WvSgnsModel* model;
  int64_t V, B, items, es;
  int d, k;
  int R, cw;  // rows per item, CBOW window (0: skip-gram)
  SlotMap sm;
  int64_t Vtok;       // token space of the corpus (V unless row-sharded)
  int nshard, shard;  // row-sharded mode (1, 0 otherwise)
  BatchWs bw;
  void* timer;
  int tb;
};

static int batch_ctx(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes, BatchCtx& c) {
  c.model = model;
  c.V = model->vocab_size;
  c.d = model->vector_size;
  c.k = batch->negatives;
  c.B = batch->batch_rows;
  WV_CHECK_ARG(c.B >= 1, "empty batch");
  WV_CHECK_ARG(c.k >= 0 && c.k <= 30, "negative_samples must be in [0, 30]");
  WV_CHECK_ARG(2 * c.V < (int64_t)0xffffffffLL, "vocabulary too large for 32-bit row keys");
  WV_CHECK_ARG(batch->mode == WV_PAIRS_NATIVE || batch->mode == WV_PAIRS_EXPLICIT, "bad pair mode");
  WV_CHECK_ARG(batch->model == WV_MODEL_SKIPGRAM || batch->model == WV_MODEL_CBOW, "bad model %d", batch->model);
  c.cw = batch->model == WV_MODEL_CBOW ? batch->window : 0;
  WV_CHECK_ARG(c.cw == 0 || (c.cw >= 1 && c.cw <= 15 && batch->instances != nullptr),
               "CBOW needs window_size in [1, 15] and an instance table");
  c.R = rows_per_item(c.k, c.cw);
  WV_CHECK_ARG(c.B * c.R < (int64_t)0x7fffffffLL, "batch too large");
  c.es = model->precision == WV_FP64 ? 8 : 4;
  c.items = c.B * c.R;
  c.sm.out_base = c.cw ? 0u : (uint32_t)c.B;
  c.sm.in_div = c.cw ? (uint32_t)(2 * c.cw) : 1u;
  c.sm.in_mag = host_mag(c.sm.in_div);
  c.sm.kmag = host_mag((uint32_t)(c.k > 0 ? c.k : 1));
  const int64_t need = carve_batch_ws((char*)ws, c.V, c.d, c.k, c.R, c.B, c.es, c.bw);
  WV_CHECK_ARG(ws_bytes >= need, "workspace too small");
  c.timer = batch->timer;
  c.tb = (int)batch->timer_base;
  c.Vtok = c.V;
  c.nshard = 1;
  c.shard = 0;
  return 0;
}

static PairArgs pair_args(const BatchCtx& c, int h) {
  PairArgs pa;
  pa.d = c.d;
  pa.k = c.k;
  pa.R = c.R;
  pa.cw = c.cw;
  pa.B = c.B;
  pa.Bn = 0;
  pa.nshard = c.nshard;
  pa.shard = c.shard;
  pa.Vl = c.V;
  pa.V = c.Vtok;
  pa.desc = c.bw.desc;
  pa.U = c.bw.U[h];
  pa.G = c.bw.G[h];
  pa.coef = c.bw.coef[h];
  pa.flag = WV_SPLIT_OWNER ? c.bw.half[h].flag : nullptr;  // row flags only feed the split owner
  pa.cnt = c.bw.half[h].cnt;
  pa.uniq = c.bw.half[h].uniq;
  pa.gctr = c.bw.half[h].gctr;
  pa.idx = c.bw.half[h].idx;
  pa.rank = c.bw.half[h].rank;
  pa.partials = c.bw.partials;
  pa.state = c.model->state;
  return pa;
}

#define WV_STAMP(slot, strm) \
  if (c.timer) WV_CUDA_RC(wv_timer_record(c.timer, c.tb + (slot), (void*)(strm)))

// the flat per-element owner serves sparse RowAdam (default); the warp-per-row
// kernels remain for dense mode, split mode and WV_SGNS_BULK_OWNER=1
static bool flat_owner(const BatchCtx& c);
// single-contribution light rows go to the lean owner kernel (flat owner, sparse RowAdam)
static bool singles_mode(const BatchCtx& c) {
  return (WV_SINGLES == 1 || (WV_SINGLES == 2 && c.model->precision == WV_FP64)) && flat_owner(c) &&
         !WV_SPLIT_OWNER && getenv("WV_NO_SINGLES") == nullptr;
}
static bool flat_owner(const BatchCtx& c) {
  return c.model->sparse && c.bw.gsum == nullptr && getenv("WV_SGNS_BULK_OWNER") == nullptr;
}

// decode: the batch's row indices + row claims (half h)
static int enqueue_decode(const BatchCtx& c, int h, cudaStream_t st) {
  const PairArgs pa = pair_args(c, h);
  WV_CUDA(cudaMemsetAsync(c.bw.half[h].gctr, 0, 8 * sizeof(uint32_t), st));
  if (flat_owner(c))
    WV_CUDA(cudaMemsetAsync(c.bw.half[h].rowdone, 0, (c.items / (kLightMax + 1) + 1) * 4, st));
  if (c.cw > 0)
    cbow_decode_kernel<<<grid_for(c.items, 128, 148 * 32), 128, 0, st>>>(pa);
  else
    sgns_decode_kernel<<<grid_for(c.items, 128, 148 * 32), 128, 0, st>>>(pa);
  WV_LAUNCH_CHECK();
  return 0;
}

// Split owner (pipelined batches): batch i's light rows are regrouped into the
// rows batch i + 1 also touches (A: front of segs2) and the rest (B: back).
// A is applied before batch i + 1's gather; B runs concurrently with that
// gather, which never reads a B row (and batch i + 2's gather waits for B).
__global__ void split_light(const Segment* __restrict__ segs, uint32_t* gctr, const uint8_t* __restrict__ next_flag,
                            Segment* __restrict__ segs2) {
  const uint32_t n = *(volatile const uint32_t*)(gctr + GC_LIGHT);
  const int lane = threadIdx.x & 31;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const bool ok = i < n;
    Segment sg;
    bool in_a = false;
    if (ok) {
      sg = segs[i];
      in_a = next_flag[sg.key] != 0;
    }
    const uint32_t ma = __ballot_sync(0xffffffffu, ok && in_a);
    const uint32_t mb = __ballot_sync(0xffffffffu, ok && !in_a);
    uint32_t pa = 0, pb = 0;
    if (lane == 0) {
      if (ma) pa = atomicAdd(gctr + GC_NA, (uint32_t)__popc(ma));
      if (mb) pb = atomicAdd(gctr + GC_NB, (uint32_t)__popc(mb));
    }
    pa = __shfl_sync(0xffffffffu, pa, 0);
    pb = __shfl_sync(0xffffffffu, pb, 0);
    const uint32_t below = (1u << lane) - 1u;
    if (ok) {
      if (in_a)
        segs2[pa + __popc(ma & below)] = sg;
      else
        segs2[n - 1u - (pb + __popc(mb & below))] = sg;
    }
  }
}

static OwnerArgs owner_args(const BatchCtx& c, int h) {
  const WvSgnsModel* model = c.model;
  const BatchHalf& x = c.bw.half[h];
  const int64_t items = c.items;
  const int k = c.k;
  OwnerArgs oa;
  oa.V = c.V;
  oa.d = c.d;
  oa.k = k;
  oa.B = c.B;
  oa.n_items = items;
  oa.list = x.list;
  oa.list_tmp = x.list_tmp;
  oa.cnt = x.cnt;
  oa.slot_bits = bits_for((uint64_t)(items - 1));
  oa.sm = c.sm;
  oa.cmag = 0;
  oa.ents = flat_owner(c) ? x.ents : nullptr;
  oa.pieces = x.pieces;
  oa.partial = x.partial;
  oa.rowdone = x.rowdone;
  oa.gctr = x.gctr;
  oa.segs = x.segs;
  oa.heavy = x.heavy;
  oa.seg_count = x.gctr + GC_LIGHT;
  oa.U = c.bw.U[h];
  oa.G = c.bw.G[h];
  oa.coef = c.bw.coef[h];
  oa.flag = WV_SPLIT_OWNER ? x.flag : nullptr;
  oa.seg_base = nullptr;
  oa.bookkeep = 1;
  oa.singles = x.singles;
  oa.piece = model->precision == WV_FP64 ? (uint32_t)WV_PIECE_FP64 : (uint32_t)kPiece;
  oa.in = model->input;
  oa.out = model->output;
  oa.m_in = model->m_in;
  oa.v_in = model->v_in;
  oa.m_out = model->m_out;
  oa.v_out = model->v_out;
  oa.touched_in = model->touched_in;
  oa.touched_out = model->touched_out;
  oa.modified_in = model->modified_in;
  oa.modified_out = model->modified_out;
  oa.lr = model->learning_rate;
  oa.sparse = model->sparse;
  oa.dense_g_in = model->dense_g_in;
  oa.dense_g_out = model->dense_g_out;
  oa.gsum = c.bw.gsum;
  oa.split = (model->sparse && c.bw.gsum != nullptr) ? 1 : 0;
  oa.state = model->state;
  return oa;
}

// grouping: per-row slot lists + RowAdam steps; advances the decode cursor
static int enqueue_group(const BatchCtx& c, int h, cudaStream_t st) {
  const BatchHalf& x = c.bw.half[h];
  const WvSgnsModel* m = c.model;
  double2* bct = nullptr;
  WV_CUDA(bc_table(&bct));
  group_segments<<<grid_for(c.items, 256, 148 * 8), 256, 0, st>>>(x.uniq, x.cnt, x.gctr, c.V, m->sparse, m->steps_in,
                                                                  m->steps_out, x.segs, x.heavy, c.items, m->state,
                                                                  c.B, bct, singles_mode(c) ? x.singles : nullptr);
  WV_LAUNCH_CHECK();
  group_place_rank<<<grid_for(c.items, 256, 148 * 8), 256, 0, st>>>(x.idx, x.rank, c.B, c.k, c.R, c.cw, c.Vtok,
                                                                    x.cnt, x.list, c.nshard, c.shard, c.V);
  WV_LAUNCH_CHECK();
  if (flat_owner(c)) {
    group_order<<<grid_for(c.items, 256, 148 * 8), 256, 0, st>>>(x.segs, x.gctr, x.list, x.ents, c.V, c.B, c.k, c.sm,
                                                                 singles_mode(c) ? x.singles : nullptr);
    WV_LAUNCH_CHECK();
    OwnerArgs oa = owner_args(c, h);
    const size_t smem = (size_t)heavy_bitmap_words(c.items) * 4;
    static size_t attr[16] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 16 && attr[dev] < smem) {
      WV_CUDA(cudaFuncSetAttribute(heavy_order, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr[dev] = smem;
    }
    // enough CTAs for every heavy row in one round (rows beyond exit at once)
    const int64_t max_heavy = c.items / (kLightMax + 1) + 1;
    heavy_order<<<(unsigned)(max_heavy < 148 * 8 ? max_heavy : 148 * 8), kHeavyThreads, smem, st>>>(oa, x.gctr,
                                                                                                  x.pieces);
    WV_LAUNCH_CHECK();
  }
  return 0;
}

static int enqueue_gather(const BatchCtx& c, int h, cudaStream_t st) {
  const PairArgs pa = pair_args(c, h);
  const WvSgnsModel* m = c.model;
  const unsigned pgrid = grid_for(c.B, kPairWarps, 148 * 32);
  return dispatch_rows<LaunchPair>(m->precision, c.d, pa, (const void*)m->input, (const void*)m->output, pgrid, st);
}

template <typename T, int EPC, int MAXC>
struct LaunchSingles {
  static int run(const OwnerArgs& a0, cudaStream_t st, bool tiles = false) {
    OwnerArgs a = a0;
    const uint32_t C = (uint32_t)(a.d / EPC);
    a.cmag = C > 1 ? (uint32_t)(0xFFFFFFFFull / C + 1ull) : 0xFFFFFFFFu;
    static int resident[16] = {0};
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 16 && resident[dev] == 0) {
      int nb = 0;
      WV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sgns_owner_single_kernel<T, EPC>, 256, 0));
      resident[dev] = nb > 0 ? nb : 1;
    }
    WV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int per = dev >= 0 && dev < 16 ? resident[dev] : 4;
    if (tiles) {
      // grid for the largest possible singles count (every slot its own row); surplus tiles exit
      const uint64_t items = (uint64_t)a.n_items * C, per_cta = 256ull * WV_SINGLE_TILE;
      sgns_owner_single_kernel<T, EPC><<<(unsigned)((items + per_cta - 1) / per_cta), 256, 0, st>>>(a, true);
    } else {
      sgns_owner_single_kernel<T, EPC><<<(unsigned)(sms * per), 256, 0, st>>>(a, false);
    }
    WV_LAUNCH_CHECK();
    return 0;
  }
};

template <typename T, int EPC, int MAXC>
struct LaunchPieces {
  static int run(const OwnerArgs& a, cudaStream_t st, unsigned grid = WV_PIECE_GRID) {
    heavy_piece_kernel<T, EPC, MAXC><<<grid, WV_PIECE_THREADS, 0, st>>>(a);
    WV_LAUNCH_CHECK();
    return 0;
  }
};

// owner phase: heavy rows on ss->h concurrently with the light rows on `st`,
// then (split mode) the Adam pass and (dense mode) the dense Adam sweep
// part: 0 = the whole batch; 1 = split part A (heavy pieces + light rows the next
// batch touches, from segs2); 2 = split part B (the other light rows, on ss->b)
static int enqueue_update(const BatchCtx& c, int h, SideStream* ss, cudaStream_t st, int t_light = -1,
                          int t_heavy = -1, int part = 0) {
  const WvSgnsModel* model = c.model;
  const int64_t V = c.V, items = c.items;
  const int d = c.d;
  OwnerArgs oa = owner_args(c, h);
  if (part == 2) {
    oa.segs = c.bw.half[h].segs2;
    oa.seg_count = c.bw.half[h].gctr + GC_NB;
    oa.seg_base = c.bw.half[h].gctr + GC_NA;
    oa.bookkeep = 0;
    return dispatch_rows<LaunchOwner>(model->precision, d, oa, (unsigned)WV_SPLIT_B_PER_SM, st);
  }
  if (part == 1) {
    oa.segs = c.bw.half[h].segs2;
    oa.seg_count = c.bw.half[h].gctr + GC_NA;
  }
  if (flat_owner(c) && part == 0 && singles_mode(c)) {
    // heavy pieces (side stream) beside the multi-contribution light rows, then the single-
    // contribution rows alone with every SM (the lean kernel's CTAs fill them)
    const unsigned pgrid = (unsigned)(model->precision == WV_FP64 ? WV_SERIAL_PIECE_GRID : WV_PIECE_GRID);
    int rc;
    if (WV_SINGLES_CONCURRENT) {
      // heavy pieces then the multi-contribution rows on the high-priority ss->h, beside the
      // single-contribution rows' tiles on `st` (all three touch disjoint rows)
      WV_CUDA(cudaEventRecord(ss->fork_h, st));
      WV_CUDA(cudaStreamWaitEvent(ss->h, ss->fork_h, 0));
      rc = dispatch_rows<LaunchPieces>(model->precision, d, oa, ss->h, pgrid);
      if (rc) return rc;
      if (t_heavy >= 0) WV_STAMP(t_heavy, ss->h);
      rc = dispatch_rows<LaunchOwner>(model->precision, d, oa, (unsigned)(WV_MULTI_PER_SM ? 1000 + WV_MULTI_PER_SM : 0),
                                      ss->h);
      if (rc) return rc;
      rc = dispatch_rows<LaunchSingles>(model->precision, d, oa, st, true);
      if (rc) return rc;
      if (t_light >= 0) WV_STAMP(t_light, st);
      WV_CUDA(cudaEventRecord(ss->join_h, ss->h));
      WV_CUDA(cudaStreamWaitEvent(st, ss->join_h, 0));
      return 0;
    }
    if (WV_SINGLES_SERIAL) {  // heavy pieces, then the multi-contribution rows, on one stream
      rc = dispatch_rows<LaunchPieces>(model->precision, d, oa, st, pgrid);
      if (rc) return rc;
      if (t_heavy >= 0) WV_STAMP(t_heavy, st);
      rc = dispatch_rows<LaunchOwner>(model->precision, d, oa, (unsigned)(WV_MULTI_PER_SM ? 1000 + WV_MULTI_PER_SM : 0),
                                      st);
      if (rc) return rc;
    } else {
      WV_CUDA(cudaEventRecord(ss->fork_h, st));
      WV_CUDA(cudaStreamWaitEvent(ss->h, ss->fork_h, 0));
      rc = dispatch_rows<LaunchPieces>(model->precision, d, oa, ss->h, pgrid);
      if (rc) return rc;
      if (t_heavy >= 0) WV_STAMP(t_heavy, ss->h);
      rc = dispatch_rows<LaunchOwner>(model->precision, d, oa, (unsigned)(WV_MULTI_PER_SM ? 1000 + WV_MULTI_PER_SM : 0),
                                      st);
      if (rc) return rc;
      WV_CUDA(cudaEventRecord(ss->join_h, ss->h));
      WV_CUDA(cudaStreamWaitEvent(st, ss->join_h, 0));
    }
    rc = dispatch_rows<LaunchSingles>(model->precision, d, oa, st);
    if (rc) return rc;
    if (t_light >= 0) WV_STAMP(t_light, st);
    return 0;
  }
  if (flat_owner(c)) {
    if (WV_OWNER_FUSED_HEAVY) return dispatch_rows<LaunchOwner>(model->precision, d, oa, 0u, st);
    if (WV_HEAVY_SERIAL == 1 || (WV_HEAVY_SERIAL == 2 && model->precision == WV_FP64)) {
      int rc = dispatch_rows<LaunchPieces>(model->precision, d, oa, st, (unsigned)WV_SERIAL_PIECE_GRID);
      if (rc) return rc;
      if (t_heavy >= 0) WV_STAMP(t_heavy, st);
      rc = dispatch_rows<LaunchOwner>(model->precision, d, oa, (unsigned)(1000 + WV_SERIAL_OWNER_PER_SM), st);
      if (rc) return rc;
      if (t_light >= 0) WV_STAMP(t_light, st);
      return 0;
    }
    // heavy pieces on the side stream (small footprint), concurrent with the light rows
    WV_CUDA(cudaEventRecord(ss->fork_h, st));
    WV_CUDA(cudaStreamWaitEvent(ss->h, ss->fork_h, 0));
    int rc = dispatch_rows<LaunchPieces>(model->precision, d, oa, ss->h);
    if (rc) return rc;
    if (t_heavy >= 0) WV_STAMP(t_heavy, ss->h);
    rc = dispatch_rows<LaunchOwner>(model->precision, d, oa, 0u, st);
    if (rc) return rc;
    if (t_light >= 0) WV_STAMP(t_light, st);
    WV_CUDA(cudaEventRecord(ss->join_h, ss->h));
    WV_CUDA(cudaStreamWaitEvent(st, ss->join_h, 0));
    return 0;
  }
  const unsigned ogrid = grid_for(items * ((d + 127) / 128), kOwnerThreads / 32, 148 * 32);
  // heavy rows (side) and light rows (main) are disjoint: run both at once
  WV_CUDA(cudaEventRecord(ss->fork_h, st));
  WV_CUDA(cudaStreamWaitEvent(ss->h, ss->fork_h, 0));
  int rc = dispatch_rows<LaunchHeavy>(model->precision, d, oa, (unsigned)(WV_HEAVY_GRID), ss->h);
  if (rc) return rc;
  rc = dispatch_rows<LaunchOwner>(model->precision, d, oa, ogrid, st);
  if (rc) return rc;
  WV_CUDA(cudaEventRecord(ss->join_h, ss->h));
  WV_CUDA(cudaStreamWaitEvent(st, ss->join_h, 0));
  if (oa.split) {
    rc = dispatch_rows<LaunchAdam>(model->precision, d, oa, (unsigned)(148 * 16), st);
    if (rc) return rc;
  }
  if (!model->sparse) {
    const int64_t n = V * (int64_t)d;
    if (model->precision == WV_FP32) {
      dense_adam<float><<<grid_for(n, 256), 256, 0, st>>>((float*)model->input, (float*)model->m_in,
                                                          (float*)model->v_in, (float*)model->dense_g_in, n, d,
                                                          model->state, model->learning_rate, model->modified_in);
      dense_adam<float><<<grid_for(n, 256), 256, 0, st>>>((float*)model->output, (float*)model->m_out,
                                                          (float*)model->v_out, (float*)model->dense_g_out, n, d,
                                                          model->state, model->learning_rate, model->modified_out);
    } else {
      dense_adam<double><<<grid_for(n, 256), 256, 0, st>>>((double*)model->input, (double*)model->m_in,
                                                           (double*)model->v_in, (double*)model->dense_g_in, n, d,
                                                           model->state, model->learning_rate, model->modified_in);
      dense_adam<double><<<grid_for(n, 256), 256, 0, st>>>((double*)model->output, (double*)model->m_out,
                                                           (double*)model->v_out, (double*)model->dense_g_out, n, d,
                                                           model->state, model->learning_rate, model->modified_out);
    }
    WV_LAUNCH_CHECK();
  }
  return 0;
}

static int bind_if_eager(const WvSgnsBatch* batch, const BatchCtx& c, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  WV_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs == cudaStreamCaptureStatusNone) {
    const CorpusDesc d = make_desc(batch);
    WV_CUDA(cudaMemcpyAsync(c.bw.desc, &d, sizeof(d), cudaMemcpyHostToDevice, st));
  }
  return 0;
}

}  // namespace wv

extern "C" {

// One SGNS batch: decode -> (gather || grouping) -> owner Adam phase.
// Every launch is stream-ordered and reads the batch cursor from `state`, so
// the sequence is CUDA-graph capturable and replayable.
int wv_sgns_batch(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes, void* stream) {
  return wv_sgns_batch_phases(model, batch, ws, ws_bytes, WV_PHASE_ALL, stream);
}

// The batch split into its phases (PAIRS = decode + gather, GROUP = row
// grouping, UPDATE = owner Adam) so callers can run them separately; all state
// flows through the workspace, so calling the phases in order equals one batch.
// Uses workspace half 0; optional device timestamps (timer) at: 0 batch start,
// 1 decode end, 2 gather end, 3 join, 4 owner end, 5 sort start, 6 sort end.
int wv_sgns_batch_phases(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes, int phases,
                         void* stream) {
  using namespace wv;
  BatchCtx c;
  WV_CUDA_RC(batch_ctx(model, batch, ws, ws_bytes, c));
  cudaStream_t st = (cudaStream_t)stream;
  WV_CUDA_RC(bind_if_eager(batch, c, st));
  SideStream* ss = nullptr;
  WV_CUDA(side_stream(&ss));
  WV_STAMP(0, st);
  if (phases & WV_PHASE_PAIRS) WV_CUDA_RC(enqueue_decode(c, 0, st));
  WV_STAMP(1, st);
  // when both PAIRS and GROUP are asked for, the grouping runs on the side
  // stream concurrently with the gather
  const bool overlap = (phases & WV_PHASE_PAIRS) && (phases & WV_PHASE_GROUP);
  cudaStream_t sort_st = st;
  if (overlap) {
    WV_CUDA(cudaEventRecord(ss->fork, st));
    WV_CUDA(cudaStreamWaitEvent(ss->s, ss->fork, 0));
    sort_st = ss->s;
  }
  if (phases & WV_PHASE_GROUP) {
    WV_STAMP(5, sort_st);
    WV_CUDA_RC(enqueue_group(c, 0, sort_st));
    WV_STAMP(6, sort_st);
  }
  if (phases & WV_PHASE_PAIRS) WV_CUDA_RC(enqueue_gather(c, 0, st));
  WV_STAMP(2, st);
  if (overlap) {
    WV_CUDA(cudaEventRecord(ss->join, ss->s));
    WV_CUDA(cudaStreamWaitEvent(st, ss->join, 0));
  }
  WV_STAMP(3, st);
  if (phases & WV_PHASE_UPDATE) WV_CUDA_RC(enqueue_update(c, 0, ss, st));
  WV_STAMP(4, st);
  return 0;
}

// `count` consecutive batches of `batch->batch_rows` pairs, software-pipelined
// across two workspace halves: the side stream decodes and groups batch i+1
// while the caller's stream gathers and applies batch i.  Batch i+1's decode
// waits for batch i-1's update (its half is reused); the gather of batch i+1
// follows batch i's update on the caller's stream (parameter order), so the
// result equals `count` calls of wv_sgns_batch.  Capturable as one CUDA graph.
int wv_sgns_batches(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes, int64_t count,
                    void* stream) {
  using namespace wv;
  WV_CHECK_ARG(count >= 1, "count must be >= 1");
  BatchCtx c;
  WV_CUDA_RC(batch_ctx(model, batch, ws, ws_bytes, c));
  cudaStream_t st = (cudaStream_t)stream;
  WV_CUDA_RC(bind_if_eager(batch, c, st));
  SideStream* ss = nullptr;
  WV_CUDA(side_stream(&ss));
  const bool split = WV_SPLIT_OWNER && flat_owner(c) && !WV_OWNER_FUSED_HEAVY && getenv("WV_NO_SPLIT") == nullptr;
  // side-after-gather: batch i+1's decode + grouping start when batch i's gather ends, so the
  // gather has the SMs to itself and the side work overlaps the (HBM-bound) update instead
  static const int side_after_gather =
      getenv("WV_SIDE_AFTER_GATHER") ? atoi(getenv("WV_SIDE_AFTER_GATHER")) : WV_SIDE_AFTER_GATHER;
  WV_CUDA(cudaEventRecord(ss->fork, st));
  WV_CUDA(cudaStreamWaitEvent(ss->s, ss->fork, 0));
  // optional timeline (profiling): per batch i, slots timer_base + 7i + {0 side start,
  // 1 side end, 2 gather start, 3 gather end, 4 update end (part A when split), 5 light-row
  // owner end, 6 heavy pieces end}
  auto side_batch = [&](int64_t j) -> int {  // decode + grouping of batch j on the side stream
    const int hj = (int)(j & 1);
    const int tj = 7 * (int)j;
    if (j >= 2) {  // half hj was batch j-2's: its update (main part and B part) must be done
      WV_CUDA(cudaStreamWaitEvent(ss->s, ss->own[hj], 0));
      WV_CUDA(cudaStreamWaitEvent(ss->s, ss->bdone[hj], 0));
    }
    if (j >= 1 && side_after_gather == 1) WV_CUDA(cudaStreamWaitEvent(ss->s, ss->gdone, 0));
    WV_STAMP(tj + 0, ss->s);
    WV_CUDA_RC(enqueue_decode(c, hj, ss->s));
    WV_CUDA(cudaEventRecord(ss->dec[hj], ss->s));
    if (j >= 1 && side_after_gather == 2) WV_CUDA(cudaStreamWaitEvent(ss->s, ss->gdone, 0));  // grouping only
    WV_CUDA_RC(enqueue_group(c, hj, ss->s));
    WV_STAMP(tj + 1, ss->s);
    WV_CUDA(cudaEventRecord(ss->grp[hj], ss->s));
    return 0;
  };
  WV_CUDA_RC(side_batch(0));
  for (int64_t i = 0; i < count; ++i) {
    const int h = (int)(i & 1);
    const int t0 = 7 * (int)i;
    WV_CUDA(cudaStreamWaitEvent(st, ss->dec[h], 0));
    // batch i-2's B rows may be rows of this batch (and half h's U/G is theirs)
    if (i >= 2) WV_CUDA(cudaStreamWaitEvent(st, ss->bdone[h], 0));
    WV_STAMP(t0 + 2, st);
    WV_CUDA_RC(enqueue_gather(c, h, st));
    WV_STAMP(t0 + 3, st);
    if (side_after_gather) WV_CUDA(cudaEventRecord(ss->gdone, st));
    // the next batch's decode (its row flags) and grouping overlap this batch
    if (i + 1 < count) WV_CUDA_RC(side_batch(i + 1));
    WV_CUDA(cudaStreamWaitEvent(st, ss->grp[h], 0));
    if (split && i + 1 < count) {
      // regroup this batch's light rows by membership in batch i+1 (its decode is done)
      WV_CUDA(cudaStreamWaitEvent(st, ss->dec[h ^ 1], 0));
      split_light<<<grid_for(c.items, 256, 148 * 8), 256, 0, st>>>(c.bw.half[h].segs, c.bw.half[h].gctr,
                                                                   c.bw.half[h ^ 1].flag, c.bw.half[h].segs2);
      WV_LAUNCH_CHECK();
      // part B on its own stream: never read by batch i+1; batch i+2 waits for it
      WV_CUDA(cudaEventRecord(ss->fork_b, st));
      WV_CUDA(cudaStreamWaitEvent(ss->b, ss->fork_b, 0));
      WV_CUDA_RC(enqueue_update(c, h, ss, ss->b, -1, -1, 2));
      WV_CUDA(cudaEventRecord(ss->bdone[h], ss->b));
      WV_CUDA_RC(enqueue_update(c, h, ss, st, c.timer ? t0 + 5 : -1, c.timer ? t0 + 6 : -1, 1));
    } else {
      WV_CUDA_RC(enqueue_update(c, h, ss, st, c.timer ? t0 + 5 : -1, c.timer ? t0 + 6 : -1, 0));
      WV_CUDA(cudaEventRecord(ss->bdone[h], st));
    }
    WV_STAMP(t0 + 4, st);
    WV_CUDA(cudaEventRecord(ss->own[h], st));
  }
  // join: the last B parts and the side stream
  if (count >= 2) WV_CUDA(cudaStreamWaitEvent(st, ss->bdone[(count - 2) & 1], 0));
  WV_CUDA(cudaStreamWaitEvent(st, ss->bdone[(count - 1) & 1], 0));
  WV_CUDA(cudaEventRecord(ss->join, ss->s));
  WV_CUDA(cudaStreamWaitEvent(st, ss->join, 0));
  return 0;
}

// ---------------------------------------------------------- row-sharded --
// cfg5 mode: rank `shard` of `nshard` owns the rows r with
// r % nshard == shard of both matrices (local row r / nshard) plus their
// RowAdam state; `model` describes that local store (vocab_size = ceil(V /
// nshard)), `vocab_global` is V.  One global batch (batch->batch_rows pairs):
//   wv_shard_decode_group   every rank decodes the whole batch and groups
//                           the contribution slots of its own rows
//   wv_shard_requests       row requests of the rank's share of pairs, by owner
//   (caller: all-to-all of the requests)   wv_shard_serve: rows for them
//   (caller: all-to-all back)              wv_shard_place: rows -> item order
//   wv_shard_gather         the rank's pairs: loss, coefficients, U/G rows
//   (caller: all-gather of U, G, coef into global-batch order)
//   wv_shard_update         slot-ordered sums + RowAdam on the rank's rows
// The result equals single-GPU training with the same global batch size.

static int shard_ctx(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes,
                     int64_t vocab_global, int nshard, int shard, wv::BatchCtx& c) {
  using namespace wv;
  WV_CHECK_ARG(nshard >= 1 && shard >= 0 && shard < nshard, "bad shard %d of %d", shard, nshard);
  WV_CHECK_ARG(model->vocab_size == (vocab_global + nshard - 1) / nshard, "local store must hold ceil(V / nshard) rows");
  WV_CHECK_ARG(model->sparse, "row-sharded training implements sparse RowAdam");
  WV_CUDA_RC(batch_ctx(model, batch, ws, ws_bytes, c));
  WV_CHECK_ARG(flat_owner(c), "row-sharded training needs the flat owner path");
  c.Vtok = vocab_global;
  c.nshard = nshard;
  c.shard = shard;
  return 0;
}

int wv_shard_init(int64_t vocab_global, int vector_size, const uint32_t* seed_prefix, int n_prefix, int precision,
                  int nshard, int shard, void* input_local, void* output_local, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(nshard >= 1 && shard >= 0 && shard < nshard, "bad shard");
  WV_CUDA(ensure_sg_table());
  uint32_t pool[4];
  ss_pool(seed_prefix, n_prefix - 1, seed_prefix[n_prefix - 1], pool);
  Pcg64 g = pcg_seed(pool);
  InitStream sg{g.state, g.inc};
  const int64_t Vl = (vocab_global + nshard - 1) / nshard;
  cudaStream_t st = (cudaStream_t)stream;
  for (int mtx = 0; mtx < 2; ++mtx) {
    void* dst = mtx == 0 ? input_local : output_local;
    if (precision == WV_FP32)
      init_rows_shard<float><<<grid_for(Vl, 128), 128, 0, st>>>(sg, vocab_global, vector_size, Vl, nshard, shard, mtx,
                                                                 (float*)dst);
    else
      init_rows_shard<double><<<grid_for(Vl, 128), 128, 0, st>>>(sg, vocab_global, vector_size, Vl, nshard, shard,
                                                                  mtx, (double*)dst);
    WV_LAUNCH_CHECK();
  }
  return 0;
}

int wv_shard_decode_group(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes,
                          int64_t vocab_global, int nshard, int shard, void* stream) {
  using namespace wv;
  BatchCtx c;
  WV_CUDA_RC(shard_ctx(model, batch, ws, ws_bytes, vocab_global, nshard, shard, c));
  cudaStream_t st = (cudaStream_t)stream;
  WV_CUDA_RC(bind_if_eager(batch, c, st));
  WV_CUDA_RC(enqueue_decode(c, 0, st));
  return enqueue_group(c, 0, st);
}

// requests of items [item_begin, item_begin + n_items) of the decoded batch;
// keys/items (sized n_items) come out grouped by owner, counts[nshard] (device
// int64) per owner; cursor is device scratch of nshard u32
int wv_shard_requests(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes,
                      int64_t vocab_global, int nshard, int shard, int64_t item_begin, int64_t n_items,
                      uint32_t* cursor, int64_t* keys, int32_t* items, int32_t* ident, int64_t* counts,
                      void* stream) {
  using namespace wv;
  BatchCtx c;
  WV_CUDA_RC(shard_ctx(model, batch, ws, ws_bytes, vocab_global, nshard, shard, c));
  cudaStream_t st = (cudaStream_t)stream;
  WV_CUDA(cudaMemsetAsync(cursor, 0, nshard * 4, st));
  const int ctxw = c.cw ? 2 * c.cw : 1;
  if (n_items > 0) {
    shard_requests<<<grid_for(n_items, 256), 256, 0, st>>>(c.bw.half[0].idx, item_begin, n_items, c.R, ctxw,
                                                           vocab_global, nshard, 0, cursor, keys, items, ident);
    WV_LAUNCH_CHECK();
  }
  shard_offsets<<<1, 1, 0, st>>>(cursor, nshard, counts);
  WV_LAUNCH_CHECK();
  if (n_items > 0) {
    shard_requests<<<grid_for(n_items, 256), 256, 0, st>>>(c.bw.half[0].idx, item_begin, n_items, c.R, ctxw,
                                                           vocab_global, nshard, 1, cursor, keys, items, ident);
    WV_LAUNCH_CHECK();
  }
  return 0;
}

int wv_shard_count_requests(const WvSgnsBatch* batch, int64_t epoch, int64_t pos_begin, int64_t rows, int nshard,
                            int32_t* scratch_rows, int64_t* counts, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(nshard >= 1 && nshard <= 64, "nshard must be in [1, 64]");
  WV_CHECK_ARG(batch != nullptr && batch->model == WV_MODEL_SKIPGRAM, "skip-gram batches only");
  cudaStream_t st = (cudaStream_t)stream;
  WV_CUDA(cudaMemsetAsync(counts, 0, (size_t)nshard * nshard * 8, st));
  if (rows <= 0) return 0;
  const int rc = wv_sgns_decode(batch, epoch, pos_begin, rows, scratch_rows, nullptr, stream);
  if (rc) return rc;
  const int R = 2 + batch->negatives;
  const int64_t bl = (rows + nshard - 1) / nshard;
  shard_count_matrix<<<grid_for(rows * R, 256, 148 * 2), 256, 0, st>>>(scratch_rows, rows, R, bl, nshard,
                                                                     (unsigned long long*)counts);
  WV_LAUNCH_CHECK();
  return 0;
}

int wv_shard_serve(const WvSgnsModel* model, const int64_t* keys, int64_t n, int64_t vocab_global, int nshard,
                   void* rows, void* stream) {
  using namespace wv;
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int d = model->vector_size;
  if (model->precision == WV_FP32)
    shard_serve<float><<<grid_for(n * d, 256), 256, 0, st>>>((const float*)model->input, (const float*)model->output,
                                                             keys, n, vocab_global, nshard, d, (float*)rows);
  else
    shard_serve<double><<<grid_for(n * d, 256), 256, 0, st>>>((const double*)model->input,
                                                              (const double*)model->output, keys, n, vocab_global,
                                                              nshard, d, (double*)rows);
  WV_LAUNCH_CHECK();
  return 0;
}

int wv_shard_place(const void* rows, const int32_t* items, int64_t n, int vector_size, int precision,
                   void* itemrows, void* stream) {
  using namespace wv;
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int d = vector_size;
  if (precision == WV_FP32)
    shard_place<float><<<grid_for(n * d, 256), 256, 0, st>>>((const float*)rows, items, n, d, (float*)itemrows);
  else
    shard_place<double><<<grid_for(n * d, 256), 256, 0, st>>>((const double*)rows, items, n, d, (double*)itemrows);
  WV_LAUNCH_CHECK();
  return 0;
}

// the rank's pairs [pair_begin, pair_begin + pair_count) of the global batch:
// rows from itemrows (item order, ident = item index or -1), U/G/coef out in
// local pair order; gradients normalised by the global batch's rows
int wv_shard_gather(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes,
                    int64_t vocab_global, int nshard, int shard, const void* itemrows, const int32_t* ident,
                    int64_t pair_count, void* U, void* G, void* coef, void* stream) {
  using namespace wv;
  BatchCtx c;
  WV_CUDA_RC(shard_ctx(model, batch, ws, ws_bytes, vocab_global, nshard, shard, c));
  if (pair_count == 0) return 0;
  PairArgs pa = pair_args(c, 0);
  pa.Bn = c.B;
  pa.B = pair_count;
  pa.idx = const_cast<int32_t*>(ident);
  pa.U = U;
  pa.G = G;
  pa.coef = coef;
  const unsigned pgrid = grid_for(pair_count, kPairWarps, 148 * 32);
  return dispatch_rows<LaunchPair>(model->precision, c.d, pa, itemrows, itemrows, pgrid, (cudaStream_t)stream);
}

// slot-ordered sums + RowAdam on the rank's rows, U/G/coef in global-batch order
int wv_shard_update(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes,
                    int64_t vocab_global, int nshard, int shard, const void* U, const void* G, const void* coef,
                    void* stream) {
  using namespace wv;
  BatchCtx c;
  WV_CUDA_RC(shard_ctx(model, batch, ws, ws_bytes, vocab_global, nshard, shard, c));
  c.bw.U[0] = const_cast<void*>(U);
  c.bw.G[0] = const_cast<void*>(G);
  c.bw.coef[0] = const_cast<void*>(coef);
  SideStream* ss = nullptr;
  WV_CUDA(side_stream(&ss));
  return enqueue_update(c, 0, ss, (cudaStream_t)stream);
}

#undef WV_STAMP

}  // extern "C"
