// Micro-benchmark (tooling, not product): RowAdam over a random list of unique
// rows of a [V, d] fp32 store (p, m, v) with one gradient row each, as in the
// SGNS owner phase at cfg2 (V = 2 x 1,000,200 keys, ~122k unique rows per
// batch, d = 200).  Measures which load strategy reaches the HBM roofline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rows_bench rows_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int D = 200;
constexpr int C4 = D / 4;  // 50 float4 chunks

__device__ __forceinline__ float4 adam4(float4& p, float4& m, float4& v, float4 g, float r1, float r2, float lr) {
  auto one = [&](float& pp, float& mm, float& vv, float gg) {
    mm = 0.9f * mm + 0.1f * gg;
    vv = 0.999f * vv + 0.001f * gg * gg;
    pp = pp - __fdividef(lr * mm * r1, __fsqrt_rn(vv * r2) + 1e-8f);
  };
  one(p.x, m.x, v.x, g.x); one(p.y, m.y, v.y, g.y); one(p.z, m.z, v.z, g.z); one(p.w, m.w, v.w, g.w);
  return p;
}

// A: warp per row, lanes own chunks lane and lane+32; all loads then compute
template <int RPW>
__global__ void __launch_bounds__(256) k_ldg(const uint32_t* __restrict__ rows, int n, float* P, float* M, float* Vv,
                                             const float* __restrict__ G, float lr) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * 256 + threadIdx.x) >> 5;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t r0 = gw * RPW; r0 < n; r0 += nw * RPW) {
    float4 p[RPW][2], m[RPW][2], v[RPW][2], g[RPW][2];
    int64_t row[RPW];
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
      row[q] = r0 + q < n ? rows[r0 + q] : -1;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int cc = lane + 32 * c;
        if (row[q] >= 0 && cc < C4) {
          const int64_t o = row[q] * D + cc * 4;
          p[q][c] = *(const float4*)(P + o);
          m[q][c] = *(const float4*)(M + o);
          v[q][c] = *(const float4*)(Vv + o);
          g[q][c] = __ldg((const float4*)(G + (r0 + q) * D + cc * 4));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int cc = lane + 32 * c;
        if (row[q] >= 0 && cc < C4) {
          const int64_t o = row[q] * D + cc * 4;
          adam4(p[q][c], m[q][c], v[q][c], g[q][c], 1.1f, 1.2f, lr);
          *(float4*)(P + o) = p[q][c];
          *(float4*)(M + o) = m[q][c];
          *(float4*)(Vv + o) = v[q][c];
        }
      }
  }
}

// B: thread-chunk mapping: a CTA of 256 threads handles rows in a flat
// (row, chunk) space so no lane idles (50 chunks per row, 256/50 rows per pass)
template <int U>
__global__ void __launch_bounds__(256) k_flat(const uint32_t* __restrict__ rows, int n, float* P, float* M, float* Vv,
                                              const float* __restrict__ G, float lr) {
  const int64_t total = (int64_t)n * C4;
  const int64_t stride = (int64_t)gridDim.x * 256 * U;
  for (int64_t i0 = blockIdx.x * 256LL * U + threadIdx.x; i0 < total; i0 += stride) {
    float4 p[U], m[U], v[U], g[U];
    int64_t o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * 256;
      o[u] = -1;
      if (i < total) {
        const int64_t r = i / C4;
        const int c = (int)(i - r * C4);
        o[u] = (int64_t)rows[r] * D + c * 4;
        p[u] = *(const float4*)(P + o[u]);
        m[u] = *(const float4*)(M + o[u]);
        v[u] = *(const float4*)(Vv + o[u]);
        g[u] = __ldg((const float4*)(G + r * D + c * 4));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (o[u] >= 0) {
        adam4(p[u], m[u], v[u], g[u], 1.1f, 1.2f, lr);
        *(float4*)(P + o[u]) = p[u];
        *(float4*)(M + o[u]) = m[u];
        *(float4*)(Vv + o[u]) = v[u];
      }
  }
}

// C: bulk copy (cp.async.bulk) of p, m, v, g into a per-warp 2-stage ring
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_bulk(const uint32_t* __restrict__ rows, int n, float* P, float* M,
                                                  float* Vv, const float* __restrict__ G, float lr) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* bar = (uint64_t*)sm + 2 * warp;
  float* ring = (float*)(sm + 256) + warp * 2 * 4 * D;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar + 1)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const int64_t nw = (int64_t)gridDim.x * NW;
  int64_t r = blockIdx.x * NW + warp;
  auto issue = [&](int64_t rr, int st) {
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar + st)), "r"(4 * D * 4) : "memory");
    __syncwarp();
    if (lane < 4) {
      const int64_t row = rows[rr];
      const float* src = lane == 0 ? P + row * D : lane == 1 ? M + row * D : lane == 2 ? Vv + row * D : G + rr * D;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su(ring + (st * 4 + lane) * D)),
                   "l"(src), "r"(D * 4), "r"(su(bar + st))
                   : "memory");
    }
  };
  if (r < n) issue(r, 0);
  uint32_t ph[2] = {0, 0};
  for (int it = 0; r < n; ++it, r += nw) {
    const int st = it & 1;
    if (r + nw < n) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(r + nw, st ^ 1);
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(su(bar + st)), "r"(ph[st]) : "memory");
    ph[st] ^= 1;
    const int64_t row = rows[r];
    const float* s = ring + st * 4 * D;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int cc = lane + 32 * c;
      if (cc < C4) {
        float4 p = *(const float4*)(s + cc * 4), m = *(const float4*)(s + D + cc * 4),
               v = *(const float4*)(s + 2 * D + cc * 4), g = *(const float4*)(s + 3 * D + cc * 4);
        adam4(p, m, v, g, 1.1f, 1.2f, lr);
        const int64_t o = row * D + cc * 4;
        *(float4*)(P + o) = p;
        *(float4*)(M + o) = m;
        *(float4*)(Vv + o) = v;
      }
    }
    __syncwarp();
  }
}

// D: plain gather-copy of rows (read 1 row, write 1 row): the gather bound
__global__ void k_copy(const uint32_t* __restrict__ rows, int n, const float* __restrict__ P, float* out) {
  const int64_t total = (int64_t)n * C4;
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int64_t r = i / C4;
    const int c = (int)(i - r * C4);
    *(float4*)(out + i * 4) = __ldg((const float4*)(P + (int64_t)rows[r] * D + c * 4));
  }
}

int main(int argc, char** argv) {
  const int64_t V = 2000400;
  const int n = argc > 1 ? atoi(argv[1]) : 122579;
  float *P, *M, *Vv, *G, *F;
  uint32_t* rows;
  CK(cudaMalloc(&P, V * D * 4)); CK(cudaMalloc(&M, V * D * 4)); CK(cudaMalloc(&Vv, V * D * 4));
  CK(cudaMalloc(&G, (int64_t)n * D * 4));
  CK(cudaMalloc(&F, 256 << 20));
  CK(cudaMalloc(&rows, n * 4));
  CK(cudaMemset(P, 0, V * D * 4)); CK(cudaMemset(M, 0, V * D * 4)); CK(cudaMemset(Vv, 0, V * D * 4));
  CK(cudaMemset(G, 0, (int64_t)n * D * 4));
  std::vector<uint32_t> all(V);
  for (int64_t i = 0; i < V; ++i) all[i] = (uint32_t)i;
  std::mt19937_64 rng(1);
  std::shuffle(all.begin(), all.end(), rng);
  CK(cudaMemcpy(rows, all.data(), n * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const double bytes = (double)n * D * 4 * 7;  // read p m v g, write p m v
  auto flush = [&]() { CK(cudaMemsetAsync(F, 1, 256 << 20)); };
  auto run = [&](const char* name, auto launch, double by) {
    float best = 1e9, sum = 0;
    for (int i = 0; i < 12; ++i) {
      flush();
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (i >= 2) { best = std::min(best, ms); sum += ms; }
    }
    CK(cudaGetLastError());
    printf("%-28s best %8.1f us  mean %8.1f us  %7.0f GB/s (best)\n", name, best * 1e3, sum / 10 * 1e3, by / (best * 1e-3) / 1e9);
  };
  int sms = 148;
  printf("rows %d, d %d, bytes/launch %.1f MB\n", n, D, bytes / 1e6);
  for (int g : {148 * 4, 148 * 8, 148 * 16, 148 * 32})
  {
    char nm[64];
    snprintf(nm, 64, "ldg rpw1 grid %d", g);
    run(nm, [&]() { k_ldg<1><<<g, 256>>>(rows, n, P, M, Vv, G, 0.01f); }, bytes);
    snprintf(nm, 64, "ldg rpw2 grid %d", g);
    run(nm, [&]() { k_ldg<2><<<g, 256>>>(rows, n, P, M, Vv, G, 0.01f); }, bytes);
    snprintf(nm, 64, "flat u1 grid %d", g);
    run(nm, [&]() { k_flat<1><<<g, 256>>>(rows, n, P, M, Vv, G, 0.01f); }, bytes);
    snprintf(nm, 64, "flat u2 grid %d", g);
    run(nm, [&]() { k_flat<2><<<g, 256>>>(rows, n, P, M, Vv, G, 0.01f); }, bytes);
  }
  {
    const int smem8 = 256 + 8 * 2 * 4 * D * 4;
    CK(cudaFuncSetAttribute(k_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem8));
    const int smem4 = 256 + 4 * 2 * 4 * D * 4;
    for (int per : {2, 3, 4, 6}) {
      char nm[64];
      snprintf(nm, 64, "bulk nw8 %d/SM", per);
      run(nm, [&]() { k_bulk<8><<<sms * per, 256, smem8>>>(rows, n, P, M, Vv, G, 0.01f); }, bytes);
      snprintf(nm, 64, "bulk nw4 %d/SM", per * 2);
      run(nm, [&]() { k_bulk<4><<<sms * per * 2, 128, smem4>>>(rows, n, P, M, Vv, G, 0.01f); }, bytes);
    }
  }
  run("copy rows (r+w)", [&]() { k_copy<<<148 * 16, 256>>>(rows, n, P, F); }, (double)n * D * 8);
  run("memcpy 1 GB d2d", [&]() { CK(cudaMemcpyAsync(M, P, 1 << 29, cudaMemcpyDeviceToDevice)); }, 2.0 * (1 << 29));
  return 0;
}
