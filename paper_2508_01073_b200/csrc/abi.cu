// C-ABI plumbing: thread-local error text, version, device queries.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"
#include "../../include/walkvec_b200.h"

namespace wv {
static thread_local char g_err[1024] = "";

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

}  // extern "C"
