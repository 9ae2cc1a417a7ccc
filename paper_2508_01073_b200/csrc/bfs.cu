// BFS predecessor-tree walks: one CTA per root, level-synchronous.
//
// Reference: walks._bfs_tree / bfs_walks (pkg/src/walkvec/walks.py:207-310).
// Per level the candidates are the frontier's adjacency slices concatenated
// in frontier order (position p); the first occurrence of each undiscovered
// target wins (np.unique(return_index) + sort, :229-240).  Here every
// candidate does find-or-insert of its target in a hash and an atomicMin of
// (PENDING | p) on the entry; entries of earlier levels hold their discovery
// index (< PENDING) and are left untouched by the min.  A second ordered pass
// over p (block scan) emits exactly the candidates that won, in ascending p,
// which is the reference's discovery order.  Leaves are discovered vertices
// that are nobody's parent, in discovery order (:281-284); each yields one
// walk root -> leaf (:285-301).  max_walks_per_root keeps the first walks of
// that order (the reference is uncapped: pass <= 0).
//
// Two tiers: the hash lives in shared memory (16K entries); a root whose
// tree outgrows it is re-run by a second launch with a global-memory hash.
#include "common.cuh"
#include "primitives.cuh"
#include "../../include/walkvec_b200.h"

namespace wv {

constexpr int kBfsThreads = 1024;
constexpr int kSmemCap = 16384;  // hash entries in the shared tier (128 KB)
constexpr uint32_t kEmpty = 0xffffffffu;
constexpr uint32_t kPending = 0x80000000u;

struct BfsArgs {
  const int64_t* off;
  const uint64_t* edges;
  const int64_t* roots;
  int64_t n_roots;
  int depth;
  int width;
  int64_t cap_walks;       // <= 0: uncapped
  // scratch (per CTA slice of size scratch_cap)
  uint32_t* ord_v;
  uint32_t* ord_parent;
  uint32_t* ord_pred;
  uint8_t* is_parent;
  int64_t* pf;
  uint32_t* g_hkey;        // global tier hash (per CTA slice of hash_cap)
  uint32_t* g_hval;
  int64_t scratch_cap;     // order-array capacity per CTA
  int64_t hash_cap;        // power of two
  // root selection
  const int64_t* root_list;  // optional: indices into roots (fallback tier)
  const int64_t* root_list_n;
  // outputs
  int64_t* walk_counts;    // count phase
  int64_t* overflow_list;
  int64_t* overflow_n;
  const int64_t* walk_base;  // emit phase: first walk row per root
  int32_t* corpus;
  int32_t* lengths;
  int emit;
};

__device__ __forceinline__ uint32_t hslot(uint32_t t, uint32_t mask) { return (t * 0x9E3779B1u) & mask; }

// find-or-insert; returns slot or -1 when the table is full
__device__ __forceinline__ int64_t h_insert(uint32_t* hk, uint32_t mask, uint32_t t, int* inserted) {
  uint32_t s = hslot(t, mask);
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    uint32_t k = hk[s];
    if (k == t) return s;
    if (k == kEmpty) {
      uint32_t prev = atomicCAS(&hk[s], kEmpty, t);
      if (prev == kEmpty) {
        atomicAdd(inserted, 1);
        return s;
      }
      if (prev == t) return s;
    }
    s = (s + 1) & mask;
  }
  return -1;
}

__device__ __forceinline__ int64_t h_find(const uint32_t* hk, uint32_t mask, uint32_t t) {
  uint32_t s = hslot(t, mask);
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    uint32_t k = hk[s];
    if (k == t) return s;
    if (k == kEmpty) return -1;
    s = (s + 1) & mask;
  }
  return -1;
}

__device__ __forceinline__ int upper_frontier(const int64_t* pf, int nf, int64_t p) {
  int lo = 0, hi = nf;  // last i with pf[i] <= p
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (pf[mid] <= p) lo = mid; else hi = mid;
  }
  return lo;
}

template <bool SMEM>
__global__ void __launch_bounds__(kBfsThreads) bfs_kernel(BfsArgs A) {
  extern __shared__ uint32_t s_hash[];
  uint32_t* s_hk = s_hash;
  uint32_t* s_hv = s_hash + kSmemCap;
  __shared__ int s_inserted, s_overflow;
  __shared__ int64_t s_total, s_chunk_tot, s_ndisc, s_f0;
  const int tid = threadIdx.x;
  uint32_t* hk = SMEM ? s_hk : A.g_hkey + (int64_t)blockIdx.x * A.hash_cap;
  uint32_t* hv = SMEM ? s_hv : A.g_hval + (int64_t)blockIdx.x * A.hash_cap;
  const int64_t hcap = SMEM ? kSmemCap : A.hash_cap;
  const uint32_t mask = (uint32_t)(hcap - 1);
  const int64_t ocap = A.scratch_cap;
  uint32_t* ord_v = A.ord_v + (int64_t)blockIdx.x * ocap;
  uint32_t* ord_parent = A.ord_parent + (int64_t)blockIdx.x * ocap;
  uint32_t* ord_pred = A.ord_pred + (int64_t)blockIdx.x * ocap;
  uint8_t* is_parent = A.is_parent + (int64_t)blockIdx.x * ocap;
  int64_t* pf = A.pf + (int64_t)blockIdx.x * (ocap + 1);
  const int64_t n_work = A.root_list ? *A.root_list_n : A.n_roots;

  for (int64_t wi = blockIdx.x; wi < n_work; wi += gridDim.x) {
    const int64_t ri = A.root_list ? A.root_list[wi] : wi;
    const uint32_t root = (uint32_t)A.roots[ri];
    for (int64_t i = tid; i < hcap; i += kBfsThreads) {
      hk[i] = kEmpty;
      hv[i] = kEmpty;
    }
    if (tid == 0) {
      s_inserted = 0;
      s_overflow = 0;
      s_ndisc = 1;
      s_f0 = 0;
      ord_v[0] = root;
      ord_parent[0] = kEmpty;
      ord_pred[0] = kEmpty;
    }
    __syncthreads();
    if (tid == 0) {
      int64_t s = h_insert(hk, mask, root, &s_inserted);
      hv[s] = 0;
    }
    __syncthreads();
    for (int level = 0; level < A.depth; ++level) {
      const int64_t f0 = s_f0, ndisc = s_ndisc;
      const int nf = (int)(ndisc - f0);
      // frontier degree prefix
      {
        int64_t carry = 0;
        for (int64_t base = 0; base < nf; base += kBfsThreads) {
          const int64_t i = base + tid;
          int64_t deg = 0;
          if (i < nf) {
            const uint32_t v = ord_v[f0 + i];
            deg = A.off[v + 1] - A.off[v];
          }
          int64_t tot;
          __shared__ int64_t tot_s;
          int64_t ex = block_excl_scan<int64_t, kBfsThreads>(deg, &tot_s);
          tot = tot_s;
          if (i < nf) pf[i] = carry + ex;
          carry += tot;
        }
        if (tid == 0) {
          pf[nf] = carry;
          s_total = carry;
        }
        __syncthreads();
      }
      const int64_t total = s_total;
      if (total == 0) break;
      // pass 1: first occurrence per target (atomicMin on candidate position)
      for (int64_t p = tid; p < total; p += kBfsThreads) {
        const int fi = upper_frontier(pf, nf, p);
        const uint32_t v = ord_v[f0 + fi];
        const uint64_t e = A.edges[A.off[v] + (p - pf[fi])];
        const uint32_t t = (uint32_t)e;
        const int64_t s = h_insert(hk, mask, t, &s_inserted);
        if (s < 0) {
          s_overflow = 1;
          continue;
        }
        atomicMin(&hv[s], kPending | (uint32_t)p);
      }
      __syncthreads();
      if (s_overflow || (int64_t)s_inserted * 2 > hcap || s_inserted > ocap || total >= (int64_t)kPending) {
        s_overflow = 1;
        break;
      }
      // pass 2: emit discoveries in ascending candidate position
      int64_t found = 0;
      for (int64_t base = 0; base < total; base += kBfsThreads) {
        const int64_t p = base + tid;
        int disc = 0;
        int fi = 0;
        uint32_t t = 0, pr = 0;
        if (p < total) {
          fi = upper_frontier(pf, nf, p);
          const uint32_t v = ord_v[f0 + fi];
          const uint64_t e = A.edges[A.off[v] + (p - pf[fi])];
          t = (uint32_t)e;
          pr = (uint32_t)(e >> 32);
          const int64_t s = h_find(hk, mask, t);
          disc = (s >= 0 && hv[s] == (kPending | (uint32_t)p)) ? 1 : 0;
        }
        const int64_t ex = block_excl_scan<int64_t, kBfsThreads>((int64_t)disc, &s_chunk_tot);
        const int64_t idx = ndisc + found + ex;
        if (disc && idx < ocap) {
          ord_v[idx] = t;
          ord_parent[idx] = (uint32_t)(f0 + fi);
          ord_pred[idx] = pr;
        }
        found += s_chunk_tot;
      }
      if (ndisc + found > ocap) {
        if (tid == 0) s_overflow = 1;
        __syncthreads();
        break;
      }
      __syncthreads();
      for (int64_t i = tid; i < found; i += kBfsThreads) {
        const int64_t s = h_find(hk, mask, ord_v[ndisc + i]);
        hv[s] = (uint32_t)(ndisc + i);
      }
      __syncthreads();
      if (found == 0) break;
      if (tid == 0) {
        s_f0 = ndisc;
        s_ndisc = ndisc + found;
      }
      __syncthreads();
    }
    __syncthreads();
    if (s_overflow) {
      if (!A.emit && tid == 0) {
        int64_t slot = atomicAdd((unsigned long long*)A.overflow_n, 1ull);
        A.overflow_list[slot] = ri;
        A.walk_counts[ri] = -1;
      }
      __syncthreads();
      continue;
    }
    const int64_t ndisc = s_ndisc;
    for (int64_t i = tid; i < ndisc; i += kBfsThreads) is_parent[i] = 0;
    __syncthreads();
    for (int64_t i = 1 + tid; i < ndisc; i += kBfsThreads) is_parent[ord_parent[i]] = 1;
    __syncthreads();
    // leaves in discovery order
    int64_t nleaf = 0;
    const int64_t cap = A.cap_walks > 0 ? A.cap_walks : INT64_MAX;
    for (int64_t base = 0; base < ndisc; base += kBfsThreads) {
      const int64_t i = base + tid;
      const int leaf = (i < ndisc && !is_parent[i]) ? 1 : 0;
      const int64_t ex = block_excl_scan<int64_t, kBfsThreads>((int64_t)leaf, &s_chunk_tot);
      const int64_t j = nleaf + ex;
      if (A.emit && leaf && j < cap) {
        // climb to the root, then write root -> leaf
        int D = 0;
        for (uint32_t x = (uint32_t)i; x != 0; x = ord_parent[x]) ++D;
        const int64_t row = A.walk_base[ri] + j;
        int32_t* out = A.corpus + row * A.width;
        uint32_t x = (uint32_t)i;
        for (int q = D; q > 0; --q) {
          out[2 * q] = (int32_t)ord_v[x];
          out[2 * q - 1] = (int32_t)ord_pred[x];
          x = ord_parent[x];
        }
        out[0] = (int32_t)root;
        for (int q = 2 * D + 1; q < A.width; ++q) out[q] = -1;
        A.lengths[row] = 2 * D + 1;
      }
      nleaf += s_chunk_tot;
    }
    if (!A.emit && tid == 0) A.walk_counts[ri] = nleaf < cap ? nleaf : cap;
    __syncthreads();
  }
}

}  // namespace wv

namespace wv {

__global__ void path_rows(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets, int64_t n_walks,
                          int64_t* __restrict__ src, int64_t* __restrict__ dst, int64_t* __restrict__ wid) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = offsets[w], L = offsets[w + 1] - o;
    const int64_t r0 = (o - w) / 2;  // every walk has an odd length 2D+1 -> D rows
    const int64_t D = (L - 1) / 2;
    for (int64_t i = 0; i < D; ++i) {
      src[r0 + i] = tokens[o + L - 3 - 2 * i];
      dst[r0 + i] = tokens[o + L - 1 - 2 * i];
      wid[r0 + i] = w;
    }
  }
}

static inline int64_t al256(int64_t b) { return (b + 255) & ~(int64_t)255; }
constexpr int kFallbackCtas = 16;

struct BfsWs {
  uint32_t *ord_v, *ord_parent, *ord_pred, *g_hkey, *g_hval, *g_ord_v, *g_ord_parent, *g_ord_pred;
  uint8_t *is_parent, *g_is_parent;
  int64_t *pf, *g_pf, *overflow_list, *overflow_n;
  int64_t smem_ocap, g_ocap, g_hcap;
  int64_t bytes;
};

static int64_t next_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

static BfsWs bfs_layout(void* base, int64_t V, int64_t n_roots) {
  BfsWs L;
  L.smem_ocap = kSmemCap / 2 + 1;
  L.g_ocap = V + 1;
  L.g_hcap = next_pow2(2 * (V + 1));
  if (L.g_hcap < 1024) L.g_hcap = 1024;
  char* w = (char*)base;
  auto take = [&](int64_t bytes) {
    char* r = w;
    w += al256(bytes);
    return (void*)r;
  };
  const int64_t S = 148;
  L.ord_v = (uint32_t*)take(S * L.smem_ocap * 4);
  L.ord_parent = (uint32_t*)take(S * L.smem_ocap * 4);
  L.ord_pred = (uint32_t*)take(S * L.smem_ocap * 4);
  L.is_parent = (uint8_t*)take(S * L.smem_ocap);
  L.pf = (int64_t*)take(S * (L.smem_ocap + 1) * 8);
  const int64_t F = kFallbackCtas;
  L.g_ord_v = (uint32_t*)take(F * L.g_ocap * 4);
  L.g_ord_parent = (uint32_t*)take(F * L.g_ocap * 4);
  L.g_ord_pred = (uint32_t*)take(F * L.g_ocap * 4);
  L.g_is_parent = (uint8_t*)take(F * L.g_ocap);
  L.g_pf = (int64_t*)take(F * (L.g_ocap + 1) * 8);
  L.g_hkey = (uint32_t*)take(F * L.g_hcap * 4);
  L.g_hval = (uint32_t*)take(F * L.g_hcap * 4);
  L.overflow_list = (int64_t*)take(n_roots * 8);
  L.overflow_n = (int64_t*)take(8);
  L.bytes = (int64_t)(w - (char*)base) + 256;
  return L;
}

static int bfs_launch(const BfsWs& L, BfsArgs A, bool smem_tier, cudaStream_t st) {
  if (smem_tier) {
    A.ord_v = L.ord_v;
    A.ord_parent = L.ord_parent;
    A.ord_pred = L.ord_pred;
    A.is_parent = L.is_parent;
    A.pf = L.pf;
    A.scratch_cap = L.smem_ocap;
    A.hash_cap = kSmemCap;
    A.root_list = nullptr;
    A.root_list_n = nullptr;
    const int smem = 2 * kSmemCap * 4;
    WV_CUDA(cudaFuncSetAttribute(bfs_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    bfs_kernel<true><<<148, kBfsThreads, smem, st>>>(A);
  } else {
    A.ord_v = L.g_ord_v;
    A.ord_parent = L.g_ord_parent;
    A.ord_pred = L.g_ord_pred;
    A.is_parent = L.g_is_parent;
    A.pf = L.g_pf;
    A.g_hkey = L.g_hkey;
    A.g_hval = L.g_hval;
    A.scratch_cap = L.g_ocap;
    A.hash_cap = L.g_hcap;
    A.root_list = L.overflow_list;
    A.root_list_n = L.overflow_n;
    bfs_kernel<false><<<kFallbackCtas, kBfsThreads, 0, st>>>(A);
  }
  WV_LAUNCH_CHECK();
  return 0;
}

}  // namespace wv

extern "C" {

int64_t wv_bfs_workspace_bytes(int64_t vertex_count, int64_t n_roots) {
  return wv::bfs_layout(nullptr, vertex_count, n_roots).bytes;
}

// Phase 1: walks per root (capped), written to walk_counts[n_roots].  The
// workspace must be kept unchanged for the matching wv_bfs_emit call.
int wv_bfs_count(const int64_t* row_offsets, const uint64_t* packed_edges, int64_t vertex_count, const int64_t* roots,
                 int64_t n_roots, int walk_depth, int64_t max_walks_per_root, int64_t* walk_counts, void* ws,
                 int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(walk_depth >= 1, "walk_depth must be >= 1");
  WV_CHECK_ARG(n_roots >= 1, "start_vertices must be non-empty");
  WV_CHECK_ARG(vertex_count < (int64_t)0x7fffffff, "graph too large for BFS scratch");
  BfsWs L = bfs_layout(ws, vertex_count, n_roots);
  WV_CHECK_ARG(ws_bytes >= L.bytes, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  WV_CUDA(cudaMemsetAsync(L.overflow_n, 0, 8, st));
  BfsArgs A{};
  A.off = row_offsets;
  A.edges = packed_edges;
  A.roots = roots;
  A.n_roots = n_roots;
  A.depth = walk_depth;
  A.width = 2 * walk_depth + 1;
  A.cap_walks = max_walks_per_root;
  A.walk_counts = walk_counts;
  A.overflow_list = L.overflow_list;
  A.overflow_n = L.overflow_n;
  A.emit = 0;
  int rc = bfs_launch(L, A, true, st);
  if (rc) return rc;
  return bfs_launch(L, A, false, st);
}

// Phase 2: walk_base[n_roots] = exclusive scan of walk_counts; writes rows
// [walk_base[r], walk_base[r] + walk_counts[r]) of the fixed-width corpus.
int wv_bfs_emit(const int64_t* row_offsets, const uint64_t* packed_edges, int64_t vertex_count, const int64_t* roots,
                int64_t n_roots, int walk_depth, int64_t max_walks_per_root, const int64_t* walk_base, int32_t* corpus,
                int32_t* lengths, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  BfsWs L = bfs_layout(ws, vertex_count, n_roots);
  WV_CHECK_ARG(ws_bytes >= L.bytes, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  BfsArgs A{};
  A.off = row_offsets;
  A.edges = packed_edges;
  A.roots = roots;
  A.n_roots = n_roots;
  A.depth = walk_depth;
  A.width = 2 * walk_depth + 1;
  A.cap_walks = max_walks_per_root;
  A.walk_base = walk_base;
  A.corpus = corpus;
  A.lengths = lengths;
  A.emit = 1;
  int rc = bfs_launch(L, A, true, st);
  if (rc) return rc;
  return bfs_launch(L, A, false, st);
}

// PathTable rows (walks.py:284-293) of a flat BFS corpus: per walk, leaf edge
// first, climbing to the root.  Row r of walk w starts at (offsets[w]-w)/2.
int wv_path_table(const int32_t* tokens, const int64_t* offsets, int64_t n_walks, int64_t* sources, int64_t* targets,
                  int64_t* walk_ids, void* stream) {
  using namespace wv;
  if (n_walks <= 0) return 0;
  int64_t g = (n_walks + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  path_rows<<<(unsigned)g, 256, 0, (cudaStream_t)stream>>>(tokens, offsets, n_walks, sources, targets, walk_ids);
  WV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
