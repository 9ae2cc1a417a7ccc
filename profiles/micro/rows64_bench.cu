// Micro-benchmark (tooling, not product): fp64 RowAdam traffic of the SGNS update
// phase at cfg2 (d = 200 doubles = 1600 B rows, ~122.6k unique rows of 2 x 1,000,200
// per batch).  Which layout / order / mapping reaches the HBM roofline?
//   separate : p, m, v in three [2V, d] arrays (the current store)
//   inter    : one [2V, 3, d] array (p, m, v of a row contiguous: 4800 B)
//   sorted   : the unique rows visited in ascending row order instead of claim order
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rows64_bench rows64_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int D = 200;
constexpr int C2 = D / 2;  // 100 double2 chunks per row

template <bool FAST>
__device__ __forceinline__ void adam2(double2& p, double2& m, double2& v, double2 g, double r1, double r2, double lr) {
  auto one = [&](double& pp, double& mm, double& vv, double gg) {
    mm = __dadd_rn(__dmul_rn(0.9, mm), __dmul_rn(0.1, gg));
    vv = __dadd_rn(__dmul_rn(0.999, vv), __dmul_rn(__dmul_rn(0.001, gg), gg));
    if (FAST)  // per-row reciprocals of the bias corrections, one division
      pp = pp - __ddiv_rn(lr * (mm * r1), __dsqrt_rn(vv * r2) + 1e-8);
    else       // numpy's order: three correctly rounded divisions + sqrt
      pp = pp - __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mm, r1)), __dadd_rn(__dsqrt_rn(__ddiv_rn(vv, r2)), 1e-8));
  };
  one(p.x, m.x, v.x, g.x);
  one(p.y, m.y, v.y, g.y);
}

__global__ void k_fill(double* a, int64_t n, double lo, double hi, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    a[i] = lo + (hi - lo) * (double)(x >> 11) * (1.0 / 9007199254740992.0);
  }
}

// flat (row, chunk) space; pstride = elements between rows; moff = offset of m from p, voff of v
template <int U>
__global__ void __launch_bounds__(256) k_flat(const uint32_t* __restrict__ rows, int n, double* P, int64_t pstride,
                                              int64_t moff, int64_t voff, const double* __restrict__ G, double lr,
                                              int mode) {
  const int64_t total = (int64_t)n * C2;
  const int64_t stride = (int64_t)gridDim.x * 256 * U;
  for (int64_t i0 = blockIdx.x * 256LL * U + threadIdx.x; i0 < total; i0 += stride) {
    double2 p[U], m[U], v[U], g[U];
    int64_t o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * 256;
      o[u] = -1;
      if (i < total) {
        const int64_t r = i / C2;
        const int c = (int)(i - r * C2);
        o[u] = (int64_t)rows[r] * pstride + c * 2;
        if (mode != 2) {
          p[u] = *(const double2*)(P + o[u]);
          m[u] = *(const double2*)(P + moff + o[u]);
          v[u] = *(const double2*)(P + voff + o[u]);
        } else {
          p[u] = m[u] = v[u] = make_double2(1.0, 1.0);
        }
        g[u] = __ldg((const double2*)(G + r * D + c * 2));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (o[u] >= 0) {
        if (mode == 4) {  // bandwidth only: trivial math
          p[u].x += g[u].x; p[u].y += g[u].y; m[u].x += g[u].x; m[u].y += g[u].y; v[u].x += g[u].x; v[u].y += g[u].y;
        } else if (mode == 3)
          adam2<true>(p[u], m[u], v[u], g[u], 1.0 / 0.1, 1.0 / 0.001, lr);
        else
          adam2<false>(p[u], m[u], v[u], g[u], 0.1, 0.001, lr);
        if (mode == 1) {  // read-only: keep the result alive without storing rows
          if (p[u].x == 12345.0) *(double2*)(P + o[u]) = p[u];
        } else {
          *(double2*)(P + o[u]) = p[u];
          *(double2*)(P + moff + o[u]) = m[u];
          *(double2*)(P + voff + o[u]) = v[u];
        }
      }
  }
}

int main(int argc, char** argv) {
  const int64_t V = 2000400;
  const int n = argc > 1 ? atoi(argv[1]) : 122579;
  double *S, *I, *G, *F;
  uint32_t *rows, *rows_sorted;
  const int64_t NE = V * D;
  CK(cudaMalloc(&S, 3 * NE * 8));  // separate: P | M | V
  CK(cudaMalloc(&I, 3 * NE * 8));  // interleaved rows
  CK(cudaMalloc(&G, (int64_t)n * D * 8));
  CK(cudaMalloc(&F, 256 << 20));
  CK(cudaMalloc(&rows, n * 4));
  CK(cudaMalloc(&rows_sorted, n * 4));
  // realistic magnitudes (zeros would send sqrt / division down their special-case paths)
  for (double* base : {S, I}) {
    k_fill<<<1184, 256>>>(base, NE, -0.01, 0.01, 1);
    k_fill<<<1184, 256>>>(base + NE, NE, -1e-5, 1e-5, 2);
    k_fill<<<1184, 256>>>(base + 2 * NE, NE, 1e-13, 1e-10, 3);
  }
  k_fill<<<1184, 256>>>(G, (int64_t)n * D, -1e-5, 1e-5, 4);
  CK(cudaDeviceSynchronize());
  std::vector<uint32_t> all(V);
  for (int64_t i = 0; i < V; ++i) all[i] = (uint32_t)i;
  std::mt19937_64 rng(1);
  std::shuffle(all.begin(), all.end(), rng);
  all.resize(n);
  CK(cudaMemcpy(rows, all.data(), n * 4, cudaMemcpyHostToDevice));
  std::sort(all.begin(), all.end());
  CK(cudaMemcpy(rows_sorted, all.data(), n * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
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
      if (i >= 2) {
        best = std::min(best, ms);
        sum += ms;
      }
    }
    CK(cudaGetLastError());
    printf("%-40s best %8.1f us  mean %8.1f us  %7.0f GB/s (best)\n", name, best * 1e3, sum / 10 * 1e3,
           by / (best * 1e-3) / 1e9);
  };
  const double rw = (double)n * D * 8 * 7;  // read p m v g, write p m v
  const double ro = (double)n * D * 8 * 4;
  const double wo = (double)n * D * 8 * 4;
  printf("rows %d, d %d fp64, bytes/launch %.1f MB (r+w)\n", n, D, rw / 1e6);
  for (int grid : {148 * 8, 148 * 16, 148 * 32}) {
    for (int srt = 0; srt < 2; ++srt) {
      const uint32_t* rr = srt ? rows_sorted : rows;
      char nm[80];
      snprintf(nm, 80, "separate %s u1 g%d", srt ? "sorted" : "random", grid);
      run(nm, [&]() { k_flat<1><<<grid, 256>>>(rr, n, S, D, NE, 2 * NE, G, 0.01, 0); }, rw);
      snprintf(nm, 80, "separate %s u2 g%d", srt ? "sorted" : "random", grid);
      run(nm, [&]() { k_flat<2><<<grid, 256>>>(rr, n, S, D, NE, 2 * NE, G, 0.01, 0); }, rw);
      snprintf(nm, 80, "inter    %s u1 g%d", srt ? "sorted" : "random", grid);
      run(nm, [&]() { k_flat<1><<<grid, 256>>>(rr, n, I, 3 * D, D, 2 * D, G, 0.01, 0); }, rw);
      snprintf(nm, 80, "inter    %s u2 g%d", srt ? "sorted" : "random", grid);
      run(nm, [&]() { k_flat<2><<<grid, 256>>>(rr, n, I, 3 * D, D, 2 * D, G, 0.01, 0); }, rw);
    }
  }
  run("separate random read-only g2368", [&]() { k_flat<2><<<148 * 16, 256>>>(rows, n, S, D, NE, 2 * NE, G, 0.01, 1); },
      ro);
  run("separate random write-only g2368",
      [&]() { k_flat<2><<<148 * 16, 256>>>(rows, n, S, D, NE, 2 * NE, G, 0.01, 2); }, wo);
  run("inter random read-only g2368", [&]() { k_flat<2><<<148 * 16, 256>>>(rows, n, I, 3 * D, D, 2 * D, G, 0.01, 1); },
      ro);
  run("separate random FAST-math g2368", [&]() { k_flat<2><<<148 * 16, 256>>>(rows, n, S, D, NE, 2 * NE, G, 0.01, 3); },
      rw);
  run("separate random NO-math g2368", [&]() { k_flat<2><<<148 * 16, 256>>>(rows, n, S, D, NE, 2 * NE, G, 0.01, 4); },
      rw);
  run("separate random NO-math u1 g4736", [&]() { k_flat<1><<<148 * 32, 256>>>(rows, n, S, D, NE, 2 * NE, G, 0.01, 4); },
      rw);
  run("memcpy 1 GB d2d", [&]() { CK(cudaMemcpyAsync(I, S, 1 << 30, cudaMemcpyDeviceToDevice)); }, 2.0 * (1 << 30));
  return 0;
}
