// Synthetic knowledge graphs on the device (the measurement inputs of
// BASELINE.json's configs) and first-occurrence token encoding.
//
// Reference (pkg/src/walkvec/benchgen.py, ingest.py):
//   gen_barabasi      benchgen.py:78-109  vertex v >= 1 draws min(m, v) distinct
//                                         targets from the attachment bag, a list
//                                         holding [0] then, per vertex u, the block
//                                         [t1, u, t2, u, ..., tk, u, u]; all draws of
//                                         v see the bag as it was before v's block
//   build_vocabulary  ingest.py:368-396   token = rank of first occurrence over the
//                                         flattened (s, p, o) stream
//
// The reference grows the bag one vertex at a time in a Python loop (35 s at
// 1M vertices, infeasible at 1e8).  The bag layout is closed-form, so a draw
// at bag position q resolves in O(1) to either a vertex's own slot (value
// known) or the target slot of an earlier edge (a pointer).  Every edge draws
// its position in parallel, pointers are chased (they only point to earlier
// vertices), duplicate targets within a vertex are redrawn, and the rounds
// repeat until no vertex holds a duplicate.  Same process and distribution as
// the reference; not the same numpy stream (draws are counter-based Philox).
#include "common.cuh"
#include "primitives.cuh"
#include "../../include/walkvec_b200.h"

namespace wv {

struct BaShape {
  int64_t n;
  int64_t m;
  int64_t small_edges;  // edges of vertices 1..m+1 : (m)(m+1)/2
  int64_t small_bag;    // bag length before vertex m+1 : (m+1)^2
};

__device__ __forceinline__ int64_t ba_k(const BaShape& s, int64_t v) { return v < s.m ? v : s.m; }

// first edge index of vertex v >= 1
__device__ __forceinline__ int64_t ba_edge_base(const BaShape& s, int64_t v) {
  if (v <= s.m + 1) return (v - 1) * v / 2;
  return s.small_edges + (v - 1 - s.m) * s.m;
}

// bag length before vertex v's block (= start of v's block)
__device__ __forceinline__ int64_t ba_bag_base(const BaShape& s, int64_t v) {
  if (v <= s.m + 1) return v * v;
  return s.small_bag + (v - s.m - 1) * (2 * s.m + 1);
}

// vertex u whose block holds bag position q
__device__ __forceinline__ int64_t ba_block_of(const BaShape& s, int64_t q) {
  if (q < s.small_bag) {
    int64_t u = (int64_t)sqrt((double)q);
    while (u * u > q) --u;
    while ((u + 1) * (u + 1) <= q) ++u;
    return u;
  }
  return s.m + 1 + (q - s.small_bag) / (2 * s.m + 1);
}

__device__ __forceinline__ uint64_t ba_draw(uint64_t seed, int64_t e, uint32_t attempt) {
  uint32_t c[4] = {(uint32_t)e, (uint32_t)((uint64_t)e >> 32), attempt, 0x42415247u};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  return ((uint64_t)c[1] << 32) | c[0];
}

// One thread per vertex: draw/resolve every slot of v; slots pointing at an
// earlier edge's target store that edge (ptr >= 0), others store the value.
__global__ void ba_resolve(BaShape s, uint64_t seed, const uint32_t* __restrict__ attempt,
                           int64_t* __restrict__ ptr, int64_t* __restrict__ val) {
  for (int64_t v = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < s.n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = ba_k(s, v), e0 = ba_edge_base(s, v), L = (int64_t)ba_bag_base(s, v);
    for (int64_t j = 0; j < k; ++j) {
      const int64_t e = e0 + j;
      const int64_t q = (int64_t)mulhi64(ba_draw(seed, e, attempt[e]), (uint64_t)L);
      const int64_t u = ba_block_of(s, q);
      int64_t p = -1, x = u;
      if (u > 0) {
        const int64_t off = q - ba_bag_base(s, u);
        if (off < 2 * ba_k(s, u) && (off & 1) == 0) {
          p = ba_edge_base(s, u) + off / 2;
          x = -1;
        }
      }
      ptr[e] = p;
      val[e] = x;
    }
  }
}

// chase pointers to a value; pointers strictly decrease, so chains end
__global__ void ba_chase(int64_t E, const int64_t* __restrict__ ptr, const int64_t* __restrict__ val,
                         int64_t* __restrict__ dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = e;
    while (ptr[x] >= 0) x = ptr[x];
    dst[e] = val[x];
  }
}

// a later slot equal to an earlier one is redrawn (the reference's rejection)
__global__ void ba_dups(BaShape s, const int64_t* __restrict__ dst, uint32_t* __restrict__ attempt,
                        int64_t* __restrict__ src, unsigned int* __restrict__ n_dup) {
  unsigned local = 0;
  for (int64_t v = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < s.n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = ba_k(s, v), e0 = ba_edge_base(s, v);
    for (int64_t j = 0; j < k; ++j) {
      src[e0 + j] = v;
      const int64_t t = dst[e0 + j];
      bool dup = false;
      for (int64_t i = 0; i < j && !dup; ++i) dup = dst[e0 + i] == t;
      if (dup) {
        attempt[e0 + j] += 1;
        ++local;
      }
    }
  }
  if (local) atomicAdd(n_dup, local);
}

// ------------------------------------------------------------- encoding ----
__device__ __forceinline__ int64_t stream_key(const int64_t* src, const int64_t* pred, const int64_t* dst,
                                              int64_t n_entities, int64_t p) {
  const int64_t e = p / 3;
  const int r = (int)(p - 3 * e);
  return r == 0 ? src[e] : (r == 1 ? n_entities + pred[e] : dst[e]);
}

__global__ void enc_first(const int64_t* __restrict__ src, const int64_t* __restrict__ pred,
                          const int64_t* __restrict__ dst, int64_t E, int64_t n_entities,
                          unsigned long long* __restrict__ first) {
  const int64_t n = 3 * E;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t key = stream_key(src, pred, dst, n_entities, p);
    // hot keys (predicates) are set early: a plain read skips most atomics
    if ((unsigned long long)p < *(volatile unsigned long long*)&first[key]) atomicMin(&first[key], (unsigned long long)p);
  }
}

__global__ void enc_flags(const int64_t* __restrict__ src, const int64_t* __restrict__ pred,
                          const int64_t* __restrict__ dst, int64_t E, int64_t n_entities,
                          const unsigned long long* __restrict__ first, uint8_t* __restrict__ flag) {
  const int64_t n = 3 * E;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    flag[p] = first[stream_key(src, pred, dst, n_entities, p)] == (unsigned long long)p;
}

__global__ void enc_token_of_key(const unsigned long long* __restrict__ first, const int64_t* __restrict__ rank,
                                 int64_t n_keys, int64_t* __restrict__ token_of_key, int64_t* __restrict__ key_of_token) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_keys; k += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long f = first[k];
    int64_t t = -1;
    if (f != ~0ull) {
      t = rank[f];
      if (key_of_token) key_of_token[t] = k;
    }
    token_of_key[k] = t;
  }
}

__global__ void enc_edges(const int64_t* __restrict__ src, const int64_t* __restrict__ pred,
                          const int64_t* __restrict__ dst, int64_t E, int64_t n_entities,
                          const int64_t* __restrict__ token_of_key, int64_t* __restrict__ out) {
  const int64_t n = 3 * E;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    out[p] = token_of_key[stream_key(src, pred, dst, n_entities, p)];
}

// ------------------------------------------------ Erdos-Renyi, uniform --
// benchgen.gen_erdos_renyi (benchgen.py:112-127): ordered pair (u, v), u != v,
// present with probability p, edges in row-major (u, v) order; and
// benchgen.gen_uniform_attachment (benchgen.py:130-149): vertex v >= 1 draws m
// targets uniformly from [0, v), duplicates collapse, targets ascending.
// Counter-based draws (Philox4x32 keyed by seed), not numpy's stream.
__device__ __forceinline__ uint64_t gen_draw(uint64_t seed, uint64_t a, uint64_t b, uint32_t tag) {
  uint32_t c[4] = {(uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32) ^ tag};
  philox4x32_10(c, (uint32_t)seed ^ 0x5bd1e995u, (uint32_t)(seed >> 32) ^ 0x27d4eb2fu);
  return ((uint64_t)c[1] << 32) | c[0];
}

__device__ __forceinline__ bool er_cell(uint64_t seed, int64_t u, int64_t v, double p) {
  return u != v && (double)(gen_draw(seed, (uint64_t)u, (uint64_t)v, 0x45u) >> 11) * (1.0 / 9007199254740992.0) < p;
}

// block per row: count (pass 0) or emit in column order (pass 1)
__global__ void er_rows(int64_t n, double p, uint64_t seed, int pass, int64_t* __restrict__ row_count,
                        const int64_t* __restrict__ row_off, int64_t* __restrict__ src, int64_t* __restrict__ dst) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t run;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t u = blockIdx.x; u < n; u += gridDim.x) {
    if (threadIdx.x == 0) run = pass ? row_off[u] : 0;
    __syncthreads();
    for (int64_t v0 = 0; v0 < n; v0 += blockDim.x) {
      const int64_t v = v0 + threadIdx.x;
      const bool hit = v < n && er_cell(seed, u, v, p);
      const uint32_t m = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) warp_tot[warp] = __popc(m);
      __syncthreads();
      if (pass && hit) {
        int64_t before = run;
        for (int w = 0; w < warp; ++w) before += warp_tot[w];
        before += __popc(m & ((1u << lane) - 1u));
        src[before] = u;
        dst[before] = v;
      }
      __syncthreads();
      if (threadIdx.x == 0)
        for (int w = 0; w < nw; ++w) run += warp_tot[w];
      __syncthreads();
    }
    if (!pass && threadIdx.x == 0) row_count[u] = run;
    __syncthreads();
  }
}

// thread per vertex: the sorted distinct targets of vertex v (m <= 64)
__device__ int ua_targets(uint64_t seed, int64_t v, int m, int64_t* t) {
  for (int j = 0; j < m; ++j) t[j] = (int64_t)mulhi64(gen_draw(seed, (uint64_t)v, (uint64_t)j, 0x55u), (uint64_t)v);
  for (int i = 1; i < m; ++i) {
    const int64_t x = t[i];
    int j = i - 1;
    while (j >= 0 && t[j] > x) {
      t[j + 1] = t[j];
      --j;
    }
    t[j + 1] = x;
  }
  int k = 0;
  for (int i = 0; i < m; ++i)
    if (i == 0 || t[i] != t[i - 1]) t[k++] = t[i];
  return k;
}

__global__ void ua_vertices(int64_t n, int m, uint64_t seed, int pass, int64_t* __restrict__ count,
                            const int64_t* __restrict__ off, int64_t* __restrict__ src, int64_t* __restrict__ dst) {
  int64_t t[64];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    if (v == 0) {
      if (!pass) count[0] = 0;
      continue;
    }
    const int k = ua_targets(seed, v, m, t);
    if (!pass) {
      count[v] = k;
      continue;
    }
    const int64_t o = off[v];
    for (int j = 0; j < k; ++j) {
      src[o + j] = v;
      dst[o + j] = t[j];
    }
  }
}

static inline unsigned grid_of(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return (unsigned)g;
}

static inline int64_t al256(int64_t b) { return (b + 255) & ~(int64_t)255; }

static BaShape ba_shape(int64_t n, int64_t m) {
  BaShape s;
  s.n = n;
  s.m = m;
  s.small_edges = m * (m + 1) / 2;
  s.small_bag = (m + 1) * (m + 1);
  return s;
}

}  // namespace wv

extern "C" {

int64_t wv_barabasi_edge_count(int64_t n, int m) {
  if (n < 2 || m < 1) return 0;
  // sum_{v=1}^{n-1} min(m, v)
  const int64_t M = m;
  if (n - 1 <= M) return (n - 1) * n / 2;
  return M * (M + 1) / 2 + (n - 1 - M) * M;
}

int64_t wv_barabasi_workspace_bytes(int64_t n, int m) {
  const int64_t E = wv_barabasi_edge_count(n, m);
  return wv::al256(E * 4) + 2 * wv::al256(E * 8) + 256;
}

int wv_gen_barabasi(int64_t n, int m, uint64_t seed, int64_t* src, int64_t* dst, void* ws, int64_t ws_bytes,
                    void* stream) {
  using namespace wv;
  WV_CHECK_ARG(n >= 2, "n must be >= 2");
  WV_CHECK_ARG(m >= 1, "m must be >= 1");
  WV_CHECK_ARG(ws_bytes >= wv_barabasi_workspace_bytes(n, m), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t E = wv_barabasi_edge_count(n, m);
  char* w = (char*)ws;
  uint32_t* attempt = (uint32_t*)w;
  w += al256(E * 4);
  int64_t* ptr = (int64_t*)w;
  w += al256(E * 8);
  int64_t* val = (int64_t*)w;
  w += al256(E * 8);
  unsigned int* n_dup = (unsigned int*)w;
  WV_CUDA(cudaMemsetAsync(attempt, 0, E * 4, st));
  const BaShape s = ba_shape(n, m);
  for (int round = 0; round < 4096; ++round) {
    WV_CUDA(cudaMemsetAsync(n_dup, 0, 4, st));
    ba_resolve<<<grid_of(n, 256), 256, 0, st>>>(s, seed, attempt, ptr, val);
    WV_LAUNCH_CHECK();
    ba_chase<<<grid_of(E, 256), 256, 0, st>>>(E, ptr, val, dst);
    WV_LAUNCH_CHECK();
    ba_dups<<<grid_of(n, 256), 256, 0, st>>>(s, dst, attempt, src, n_dup);
    WV_LAUNCH_CHECK();
    unsigned h = 0;
    WV_CUDA(cudaMemcpyAsync(&h, n_dup, 4, cudaMemcpyDeviceToHost, st));
    WV_CUDA(cudaStreamSynchronize(st));
    if (h == 0) return 0;
  }
  set_error("barabasi generator did not converge");
  return -2;
}

int64_t wv_encode_workspace_bytes(int64_t E, int64_t n_keys) {
  using namespace wv;
  const int64_t n = 3 * E;
  return al256(n_keys * 8) + al256(n) + al256(n * 8) + al256(scan_tiles(n) * 8) + 256;
}

int wv_encode_triples(const int64_t* src, const int64_t* preds, const int64_t* dst, int64_t E, int64_t n_entities,
                      int64_t n_predicates, int64_t* edges_out, int64_t* token_of_key, int64_t* key_of_token,
                      int64_t* vocab_size, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(E >= 0 && n_entities >= 1 && n_predicates >= 1, "bad sizes");
  const int64_t n_keys = n_entities + n_predicates;
  WV_CHECK_ARG(ws_bytes >= wv_encode_workspace_bytes(E, n_keys), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = 3 * E;
  char* w = (char*)ws;
  unsigned long long* first = (unsigned long long*)w;
  w += al256(n_keys * 8);
  uint8_t* flag = (uint8_t*)w;
  w += al256(n);
  int64_t* rank = (int64_t*)w;
  w += al256(n * 8);
  int64_t* scan_ws = (int64_t*)w;
  WV_CUDA(cudaMemsetAsync(first, 0xff, n_keys * 8, st));
  if (key_of_token) WV_CUDA(cudaMemsetAsync(key_of_token, 0xff, n_keys * 8, st));
  if (E == 0) {
    WV_CUDA(cudaMemsetAsync(vocab_size, 0, 8, st));
    WV_CUDA(cudaMemsetAsync(token_of_key, 0xff, n_keys * 8, st));
    return 0;
  }
  enc_first<<<grid_of(n, 256), 256, 0, st>>>(src, preds, dst, E, n_entities, first);
  WV_LAUNCH_CHECK();
  enc_flags<<<grid_of(n, 256), 256, 0, st>>>(src, preds, dst, E, n_entities, first, flag);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<uint8_t, int64_t>(flag, n, rank, vocab_size, scan_ws, st)));
  enc_token_of_key<<<grid_of(n_keys, 256), 256, 0, st>>>(first, rank, n_keys, token_of_key, key_of_token);
  WV_LAUNCH_CHECK();
  if (edges_out) {
    enc_edges<<<grid_of(n, 256), 256, 0, st>>>(src, preds, dst, E, n_entities, token_of_key, edges_out);
    WV_LAUNCH_CHECK();
  }
  return 0;
}

// Erdos-Renyi / uniform attachment on the device: call with src = dst = NULL to
// get the edge count (*n_edges, device int64), then again with buffers of that size.
int64_t wv_gen_rows_workspace_bytes(int64_t n) {
  using namespace wv;
  return al256(n * 8) * 2 + al256(scan_tiles(n) * 8) + 256;
}

static int gen_rows(int kind, int64_t n, double p, int m, uint64_t seed, int64_t* src, int64_t* dst,
                    int64_t* n_edges, void* ws, int64_t ws_bytes, cudaStream_t st) {
  using namespace wv;
  WV_CHECK_ARG(ws_bytes >= wv_gen_rows_workspace_bytes(n), "workspace too small");
  char* w = (char*)ws;
  int64_t* cnt = (int64_t*)w;
  w += al256(n * 8);
  int64_t* off = (int64_t*)w;
  w += al256(n * 8);
  int64_t* scan_ws = (int64_t*)w;
  if (kind == 0)
    er_rows<<<grid_of(n, 1), 256, 0, st>>>(n, p, seed, 0, cnt, nullptr, nullptr, nullptr);
  else
    ua_vertices<<<grid_of(n, 128), 128, 0, st>>>(n, m, seed, 0, cnt, nullptr, nullptr, nullptr);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<int64_t, int64_t>(cnt, n, off, n_edges, scan_ws, st)));
  if (src == nullptr) return 0;
  if (kind == 0)
    er_rows<<<grid_of(n, 1), 256, 0, st>>>(n, p, seed, 1, nullptr, off, src, dst);
  else
    ua_vertices<<<grid_of(n, 128), 128, 0, st>>>(n, m, seed, 1, nullptr, off, src, dst);
  WV_LAUNCH_CHECK();
  return 0;
}

int wv_gen_erdos_renyi(int64_t n, double p, uint64_t seed, int64_t* src, int64_t* dst, int64_t* n_edges, void* ws,
                       int64_t ws_bytes, void* stream) {
  WV_CHECK_ARG(n >= 1, "n must be >= 1");
  WV_CHECK_ARG(p > 0.0 && p < 1.0, "p must be in (0, 1)");
  return gen_rows(0, n, p, 0, seed, src, dst, n_edges, ws, ws_bytes, (cudaStream_t)stream);
}

int wv_gen_uniform_attachment(int64_t n, int m, uint64_t seed, int64_t* src, int64_t* dst, int64_t* n_edges,
                              void* ws, int64_t ws_bytes, void* stream) {
  WV_CHECK_ARG(n >= 2, "n must be >= 2");
  WV_CHECK_ARG(m >= 1 && m <= 64, "m must be in [1, 64]");
  return gen_rows(1, n, 0.0, m, seed, src, dst, n_edges, ws, ws_bytes, (cudaStream_t)stream);
}

}  // extern "C"
