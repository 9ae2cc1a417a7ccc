// Device primitives shared by the CSR, walk and SGNS kernels:
//   * exclusive prefix scan (3-phase: tile reduce -> carry scan -> tile scan)
//   * stable LSD radix sort of (u32 key, u32 value) pairs, 8-bit digits,
//     warp-match ranking so equal keys keep input order (the stability the
//     reference gets from np.argsort(kind="stable"), graph.py:89, and the
//     slot order np.add.at sums in, w2v.py:415).
// Caller-owned workspace only; every launch takes an explicit stream.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace wv {

// host-side count of kernels this library has enqueued (abi.cu); graph
// captures count once per captured launch
void note_launches(int n);

constexpr int kScanThreads = 512;
constexpr int kScanIpt = 8;
constexpr int64_t kScanTile = (int64_t)kScanThreads * kScanIpt;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total to *total.
template <typename T, int NT>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T warp_tot[NT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T incl = warp_incl_scan(v);
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T w = lane < NT / 32 ? warp_tot[lane] : T(0);
    T wi = warp_incl_scan(w);
    if (lane < NT / 32) warp_tot[lane] = wi - w;
    if (lane == NT / 32 - 1) *total = wi;
  }
  __syncthreads();
  T r = incl - v + warp_tot[warp];
  __syncthreads();
  return r;
}

template <typename Tin, typename T>
__global__ void scan_tile_reduce(const Tin* __restrict__ in, int64_t n, T* __restrict__ tile_sums) {
  const int64_t base = blockIdx.x * kScanTile;
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanIpt; ++i) {
    int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (idx < n) s += (T)in[idx];
  }
  __shared__ T tot;
  block_excl_scan<T, kScanThreads>(s, &tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// Single block: exclusive scan of tile sums in place, chunk by chunk.
// Writes the grand total to *total (if non-null).
template <typename T>
__global__ void scan_carry(T* __restrict__ sums, int64_t n, T* __restrict__ total) {
  __shared__ T chunk_tot;
  T carry = 0;
  for (int64_t base = 0; base < n; base += kScanThreads) {
    int64_t idx = base + threadIdx.x;
    T v = idx < n ? sums[idx] : T(0);
    T ex = block_excl_scan<T, kScanThreads>(v, &chunk_tot);
    if (idx < n) sums[idx] = ex + carry;
    carry += chunk_tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

template <typename Tin, typename T>
__global__ void scan_tile_apply(const Tin* __restrict__ in, int64_t n, const T* __restrict__ tile_sums,
                                T* __restrict__ out) {
  const int64_t base = blockIdx.x * kScanTile;
  // blocked arrangement: thread t owns kScanIpt consecutive items
  T v[kScanIpt];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanIpt; ++i) {
    int64_t idx = base + (int64_t)threadIdx.x * kScanIpt + i;
    v[i] = idx < n ? (T)in[idx] : T(0);
    s += v[i];
  }
  __shared__ T tot;
  T ex = block_excl_scan<T, kScanThreads>(s, &tot) + tile_sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanIpt; ++i) {
    int64_t idx = base + (int64_t)threadIdx.x * kScanIpt + i;
    if (idx < n) out[idx] = ex;
    ex += v[i];
  }
}

inline int64_t scan_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }

// Workspace: scan_tiles(n) elements of T.  out may alias in.  If total is
// non-null the grand total is written there (device pointer).
template <typename Tin, typename T>
inline cudaError_t excl_scan(const Tin* in, int64_t n, T* out, T* total, T* ws, cudaStream_t st) {
  if (n <= 0) {
    if (total) return cudaMemsetAsync(total, 0, sizeof(T), st);
    return cudaSuccess;
  }
  int64_t tiles = scan_tiles(n);
  note_launches(3);
  scan_tile_reduce<Tin, T><<<(unsigned)tiles, kScanThreads, 0, st>>>(in, n, ws);
  scan_carry<T><<<1, kScanThreads, 0, st>>>(ws, tiles, total);
  scan_tile_apply<Tin, T><<<(unsigned)tiles, kScanThreads, 0, st>>>(in, n, ws, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------ radix sort --
constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;

template <int IPT>
__global__ void radix_hist(const uint32_t* __restrict__ keys, int64_t n, int shift,
                           uint32_t* __restrict__ hist, int64_t num_tiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = blockIdx.x * (int64_t)(kRadixThreads * IPT);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    int64_t idx = base + (int64_t)i * kRadixThreads + threadIdx.x;
    if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * num_tiles + blockIdx.x] = h[threadIdx.x];
}

template <int IPT>
__global__ void __launch_bounds__(kRadixThreads) radix_scatter(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n, int shift, const uint32_t* __restrict__ hist_scanned,
    int64_t num_tiles) {
  __shared__ uint32_t wcnt[kRadixWarps][257];
  __shared__ uint32_t toff[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kRadixWarps * 257; i += kRadixThreads) (&wcnt[0][0])[i] = 0;
  toff[threadIdx.x] = hist_scanned[(int64_t)threadIdx.x * num_tiles + blockIdx.x];
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t base = blockIdx.x * (int64_t)(kRadixThreads * IPT) + (int64_t)warp * (32 * IPT);
  uint32_t key[IPT], val[IPT], loc[IPT], dig[IPT];
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    int64_t idx = base + it * 32 + lane;
    bool ok = idx < n;
    key[it] = ok ? kin[idx] : 0u;
    val[it] = ok ? vin[idx] : 0u;
    uint32_t d = ok ? ((key[it] >> shift) & 255u) : 256u;
    dig[it] = d;
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t cnt = wcnt[warp][d];
    __syncwarp();
    if ((peers & lt) == 0) wcnt[warp][d] = cnt + __popc(peers);
    __syncwarp();
    loc[it] = cnt + __popc(peers & lt);
  }
  __syncthreads();
  {
    uint32_t run = 0;
    for (int w = 0; w < kRadixWarps; ++w) {
      uint32_t c = wcnt[w][threadIdx.x];
      wcnt[w][threadIdx.x] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    if (dig[it] < 256u) {
      uint32_t pos = toff[dig[it]] + wcnt[warp][dig[it]] + loc[it];
      kout[pos] = key[it];
      vout[pos] = val[it];
    }
  }
}

struct RadixPlan {
  int64_t n;
  int passes;
  int ipt;
  int64_t tiles;
};

inline RadixPlan radix_plan(int64_t n, int key_bits) {
  RadixPlan p;
  p.n = n;
  p.passes = key_bits <= 0 ? 1 : (key_bits + 7) / 8;
  p.ipt = n >= (int64_t)(1 << 22) ? 16 : 4;
  p.tiles = (n + (int64_t)kRadixThreads * p.ipt - 1) / ((int64_t)kRadixThreads * p.ipt);
  if (p.tiles < 1) p.tiles = 1;
  return p;
}

// Workspace bytes: alt keys + alt values + histogram + scan scratch.
inline int64_t radix_ws_bytes(int64_t n, int key_bits) {
  RadixPlan p = radix_plan(n, key_bits);
  int64_t hist = p.tiles * 256;
  auto al = [](int64_t b) { return (b + 255) & ~(int64_t)255; };
  return al(n * 4) * 2 + al(hist * 4) + al(scan_tiles(hist) * 4) + 256;
}

// Sorts (keys, vals) in place (result lands back in keys/vals).
inline cudaError_t radix_sort_pairs(uint32_t* keys, uint32_t* vals, int64_t n, int key_bits, void* ws,
                                    cudaStream_t st) {
  if (n <= 1) return cudaSuccess;
  RadixPlan p = radix_plan(n, key_bits);
  auto al = [](int64_t b) { return (b + 255) & ~(int64_t)255; };
  char* w = (char*)ws;
  uint32_t* k2 = (uint32_t*)w;
  w += al(n * 4);
  uint32_t* v2 = (uint32_t*)w;
  w += al(n * 4);
  uint32_t* hist = (uint32_t*)w;
  w += al(p.tiles * 256 * 4);
  uint32_t* scan_ws = (uint32_t*)w;
  uint32_t *ka = keys, *va = vals, *kb = k2, *vb = v2;
  for (int pass = 0; pass < p.passes; ++pass) {
    int shift = pass * 8;
    note_launches(2);
    if (p.ipt == 16) {
      radix_hist<16><<<(unsigned)p.tiles, kRadixThreads, 0, st>>>(ka, n, shift, hist, p.tiles);
    } else {
      radix_hist<4><<<(unsigned)p.tiles, kRadixThreads, 0, st>>>(ka, n, shift, hist, p.tiles);
    }
    cudaError_t e = excl_scan<uint32_t, uint32_t>(hist, p.tiles * 256, hist, (uint32_t*)nullptr, scan_ws, st);
    if (e != cudaSuccess) return e;
    if (p.ipt == 16) {
      radix_scatter<16><<<(unsigned)p.tiles, kRadixThreads, 0, st>>>(ka, va, kb, vb, n, shift, hist, p.tiles);
    } else {
      radix_scatter<4><<<(unsigned)p.tiles, kRadixThreads, 0, st>>>(ka, va, kb, vb, n, shift, hist, p.tiles);
    }
    uint32_t* t = ka;
    ka = kb;
    kb = t;
    t = va;
    va = vb;
    vb = t;
  }
  if (ka != keys) {
    cudaError_t e = cudaMemcpyAsync(keys, ka, n * 4, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(vals, va, n * 4, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

inline int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b)) ++b;
  return b;
}

}  // namespace wv
