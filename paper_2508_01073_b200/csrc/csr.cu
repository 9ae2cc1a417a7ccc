// CSR build: (E,3) int64 (src, pred, dst) token rows -> row_offsets int64[V+1]
// and packed 8-byte edges (pred << 32 | dst), stable by source.
//
// Replaces graph.build_graph (reference pkg/src/walkvec/graph.py:74-98):
// np.argsort(src, kind="stable") + bincount + cumsum.  Stability comes from
// the LSD radix sort (equal sources keep input order), so the adjacency
// order inside each row is the input order exactly as in the reference.
#include "common.cuh"
#include "primitives.cuh"
#include "../../include/walkvec_b200.h"

namespace wv {

__global__ void csr_keys(const int64_t* __restrict__ edges, int64_t E, uint32_t* __restrict__ keys,
                         uint32_t* __restrict__ vals, uint32_t* __restrict__ counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t s = (uint32_t)edges[3 * i];
    keys[i] = s;
    vals[i] = (uint32_t)i;
    atomicAdd(&counts[s], 1u);
  }
}

__global__ void csr_gather(const int64_t* __restrict__ edges, int64_t E, const uint32_t* __restrict__ order,
                           uint64_t* __restrict__ packed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = order[i];
    uint64_t p = (uint64_t)edges[3 * j + 1], d = (uint64_t)edges[3 * j + 2];
    packed[i] = (p << 32) | (d & 0xffffffffull);
  }
}

__global__ void csr_unpack(const uint64_t* __restrict__ packed, int64_t E, int64_t* __restrict__ targets,
                           int64_t* __restrict__ preds) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t e = packed[i];
    if (targets) targets[i] = (int64_t)(e & 0xffffffffull);
    if (preds) preds[i] = (int64_t)(e >> 32);
  }
}

static inline int64_t al256(int64_t b) { return (b + 255) & ~(int64_t)255; }

static inline unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace wv

extern "C" {

int64_t wv_csr_workspace_bytes(int64_t E, int64_t V) {
  using namespace wv;
  int bits = bits_for(V > 0 ? (uint64_t)(V - 1) : 0);
  return al256(E * 4) * 2 + al256(radix_ws_bytes(E, bits)) + al256((V + 1) * 4) +
         al256(scan_tiles(V + 1) * 8) + 256;
}

int wv_csr_build(const int64_t* edges, int64_t E, int64_t V, int64_t* row_offsets, uint64_t* packed, void* ws,
                 int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(E >= 0 && V >= 1, "bad sizes E=%lld V=%lld", (long long)E, (long long)V);
  WV_CHECK_ARG(V < (int64_t)0xffffffffLL && E < (int64_t)0xffffffffLL, "graph exceeds 32-bit token/edge ids");
  WV_CHECK_ARG(ws_bytes >= wv_csr_workspace_bytes(E, V), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  int bits = bits_for((uint64_t)(V - 1));
  char* w = (char*)ws;
  uint32_t* keys = (uint32_t*)w;
  w += al256(E * 4);
  uint32_t* vals = (uint32_t*)w;
  w += al256(E * 4);
  void* rws = w;
  w += al256(radix_ws_bytes(E, bits));
  uint32_t* counts = (uint32_t*)w;
  w += al256((V + 1) * 4);
  int64_t* scan_ws = (int64_t*)w;
  WV_CUDA(cudaMemsetAsync(counts, 0, (V + 1) * 4, st));
  if (E > 0) {
    csr_keys<<<grid_for(E, 256), 256, 0, st>>>(edges, E, keys, vals, counts);
    WV_LAUNCH_CHECK();
    WV_CUDA(radix_sort_pairs(keys, vals, E, bits, rws, st));
    csr_gather<<<grid_for(E, 256), 256, 0, st>>>(edges, E, vals, packed);
    WV_LAUNCH_CHECK();
  }
  // offsets = exclusive scan of counts over V+1 entries (counts[V] = 0 -> offsets[V] = E)
  WV_CUDA((excl_scan<uint32_t, int64_t>(counts, V + 1, row_offsets, (int64_t*)nullptr, scan_ws, st)));
  return 0;
}

int wv_csr_unpack(const uint64_t* packed, int64_t E, int64_t* targets, int64_t* preds, void* stream) {
  using namespace wv;
  if (E <= 0) return 0;
  csr_unpack<<<grid_for(E, 256), 256, 0, (cudaStream_t)stream>>>(packed, E, targets, preds);
  WV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
