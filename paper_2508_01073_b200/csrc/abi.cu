// C-ABI plumbing: thread-local error text, version, device queries.
#include <cstdarg>
#include <cstdio>
#include <atomic>
#include <cstdlib>

#include "common.cuh"
#include "../../include/walkvec_b200.h"

namespace wv {
static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void note_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace wv

extern "C" {

const char* wv_last_error(void) { return wv::g_err; }

int wv_abi_version(void) { return WV_ABI_VERSION; }

int64_t wv_launch_count(void) { return (int64_t)wv::g_launches.load(std::memory_order_relaxed); }

int64_t wv_struct_size(int which) {
  switch (which) {
    case 0: return (int64_t)sizeof(WvSgnsDevState);
    case 1: return (int64_t)sizeof(WvSgnsModel);
    case 2: return (int64_t)sizeof(WvSgnsBatch);
    default: return -1;
  }
}

int wv_stream_sync(void* stream) {
  WV_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return 0;
}

// Host-side SeedSequence -> generator state, for host code that wants to
// pre-seed streams without a device (also used by the CPU symbol tests).
int wv_seedseq_generate(const uint32_t* entropy_prefix, int n_prefix, uint64_t index, int n64,
                        uint64_t* out) {
  WV_CHECK_ARG(n_prefix >= 0 && n_prefix <= 13, "n_prefix out of range");
  WV_CHECK_ARG(n64 >= 1 && n64 <= 8, "n64 out of range");
  uint32_t pool[4];
  wv::ss_pool(entropy_prefix, n_prefix, index, pool);
  wv::ss_generate_u64(pool, n64, out);
  return 0;
}

// Host-side numpy-compatible stream element k for a generator seeded from
// SeedSequence(prefix + [index]).  kind: WV_RNG_PCG64 or WV_RNG_PHILOX.
int wv_stream_u64(const uint32_t* entropy_prefix, int n_prefix, uint64_t index, int kind,
                  uint64_t k, uint64_t* out) {
  WV_CHECK_ARG(n_prefix >= 0 && n_prefix <= 13, "n_prefix out of range");
  uint32_t pool[4];
  wv::ss_pool(entropy_prefix, n_prefix, index, pool);
  if (kind == WV_RNG_PCG64) {
    wv::Pcg64 g = wv::pcg_seed(pool);
    wv::PcgJump tab[64];
    wv::pcg_jump_table(tab, 64);
    wv::PcgJump j = wv::pcg_jump_n(tab, k + 1);
    wv::u128 s = wv::add128(wv::mul128(j.A, g.state), wv::mul128(g.inc, j.S));
    *out = wv::pcg_output(s);
    return 0;
  }
  if (kind == WV_RNG_PHILOX) {
    uint64_t key[2];
    wv::ss_generate_u64(pool, 2, key);
    *out = wv::philox_numpy_u64(key[0], key[1], k);
    return 0;
  }
  wv::set_error("unknown rng kind %d", kind);
  return -1;
}

// ---- device timers usable inside CUDA-graph capture (external event records)
struct WvTimer {
  int n;
  cudaEvent_t ev[1];
};

void* wv_timer_create(int n) {
  if (n < 1) {
    wv::set_error("timer needs >= 1 event");
    return nullptr;
  }
  WvTimer* t = (WvTimer*)malloc(sizeof(WvTimer) + sizeof(cudaEvent_t) * (n - 1));
  if (!t) return nullptr;
  t->n = n;
  for (int i = 0; i < n; ++i) {
    if (cudaEventCreate(&t->ev[i]) != cudaSuccess) {
      for (int j = 0; j < i; ++j) cudaEventDestroy(t->ev[j]);
      free(t);
      wv::set_error("cudaEventCreate failed");
      return nullptr;
    }
  }
  return t;
}

int wv_timer_record(void* timer, int i, void* stream) {
  WvTimer* t = (WvTimer*)timer;
  WV_CHECK_ARG(t && i >= 0 && i < t->n, "bad timer slot");
  cudaStream_t st = (cudaStream_t)stream;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  WV_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    WV_CUDA(cudaEventRecordWithFlags(t->ev[i], st, cudaEventRecordExternal));
  else
    WV_CUDA(cudaEventRecord(t->ev[i], st));
  return 0;
}

int wv_timer_elapsed(void* timer, int i, int j, float* ms) {
  WvTimer* t = (WvTimer*)timer;
  WV_CHECK_ARG(t && i >= 0 && i < t->n && j >= 0 && j < t->n, "bad timer slot");
  WV_CUDA(cudaEventElapsedTime(ms, t->ev[i], t->ev[j]));
  return 0;
}

int wv_timer_destroy(void* timer) {
  WvTimer* t = (WvTimer*)timer;
  if (!t) return 0;
  for (int i = 0; i < t->n; ++i) cudaEventDestroy(t->ev[i]);
  free(t);
  return 0;
}

}  // extern "C"
