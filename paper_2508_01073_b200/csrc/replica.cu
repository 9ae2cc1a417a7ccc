// Data-parallel replica exchange for multi-GPU SGNS.
//
// Reference: w2v._train_multi (pkg/src/walkvec/w2v.py:662-746).  Each worker
// trains a private replica; at a sync boundary the per-row deltas against the
// round-start values are merged as shared[r] += mean over the workers that
// touched r of delta_w[r] (_merge_bundles, :642-659), then every replica
// copies the merged rows back (:719-724).  Here a worker is a GPU rank: the
// deltas and touch counts are summed with one NCCL all-reduce (issued by the
// host through torch.distributed) and these two kernels bracket it.
#include "common.cuh"
#include "../../include/walkvec_b200.h"

namespace wv {

template <typename T>
__global__ void delta_kernel(const T* __restrict__ p, const T* __restrict__ s, int64_t n, T* __restrict__ d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = p[i] - s[i];
}

template <typename T>
__global__ void apply_kernel(T* __restrict__ p, T* __restrict__ s, const T* __restrict__ dsum,
                             const float* __restrict__ cnt, int64_t rows, int dim) {
  const int64_t n = rows * dim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float c = cnt[i / dim];
    if (c > 0.f) {
      const T v = s[i] + dsum[i] / (T)c;
      p[i] = v;
      s[i] = v;
    } else {
      s[i] = p[i];
    }
  }
}

static inline unsigned grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace wv

extern "C" {

int wv_replica_delta(const void* params, const void* snapshot, int64_t n, int precision, void* delta, void* stream) {
  using namespace wv;
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return 0;
  if (precision == WV_FP32)
    delta_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)params, (const float*)snapshot, n, (float*)delta);
  else if (precision == WV_FP64)
    delta_kernel<double><<<grid_for(n), 256, 0, st>>>((const double*)params, (const double*)snapshot, n,
                                                      (double*)delta);
  else
    WV_CHECK_ARG(false, "bad precision");
  WV_LAUNCH_CHECK();
  return 0;
}

int wv_replica_apply(void* params, void* snapshot, const void* delta_sum, const float* touch_count, int64_t rows,
                     int vector_size, int precision, void* stream) {
  using namespace wv;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = rows * vector_size;
  if (n <= 0) return 0;
  if (precision == WV_FP32)
    apply_kernel<float><<<grid_for(n), 256, 0, st>>>((float*)params, (float*)snapshot, (const float*)delta_sum,
                                                     touch_count, rows, vector_size);
  else if (precision == WV_FP64)
    apply_kernel<double><<<grid_for(n), 256, 0, st>>>((double*)params, (double*)snapshot, (const double*)delta_sum,
                                                      touch_count, rows, vector_size);
  else
    WV_CHECK_ARG(false, "bad precision");
  WV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
