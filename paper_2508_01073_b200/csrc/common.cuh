// Shared device/host helpers for the walkvec B200 hot path.
//
// Bit-exact restatements of the numpy generators the reference draws from
// (numpy is the reference's only dependency, pkg/pyproject.toml:10):
//   * SeedSequence pool mixing + generate_state  (walks.py:172, w2v.py:127,548-549)
//   * PCG64 (XSL-RR 128/64) with O(log n) jump-ahead  -> default_rng streams
//   * Philox4x64-10 counter addressing               -> Generator(Philox(ss))
// All arithmetic is integer; the only float step is the numpy
// next_double = (u64 >> 11) * 2^-53 conversion.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define WV_HD __host__ __device__ __forceinline__

namespace wv {

// ----------------------------------------------------------------- u128 ----
struct u128 {
  uint64_t lo, hi;
};

WV_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

WV_HD u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

WV_HD u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}

// --------------------------------------------------------- SeedSequence ----
// numpy/random/bit_generator.pyx: pool_size 4, 32-bit hash mixing.
constexpr uint32_t SS_INIT_A = 0x43b0d7e5u;
constexpr uint32_t SS_MULT_A = 0x931e8875u;
constexpr uint32_t SS_INIT_B = 0x8b51f9ddu;
constexpr uint32_t SS_MULT_B = 0x58f38dedu;
constexpr uint32_t SS_MIX_L = 0xca01f9ddu;
constexpr uint32_t SS_MIX_R = 0x4973f715u;

WV_HD uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= SS_MULT_A;
  v *= hc;
  v ^= v >> 16;
  return v;
}

WV_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> 16;
  return r;
}

// Entropy = prefix words (already little-endian u32 encoded by the host)
// followed by the words of `index` (one word if < 2^32, else two).
// Fills pool[4].
WV_HD void ss_pool(const uint32_t* prefix, int n_prefix, uint64_t index, uint32_t pool[4]) {
  uint32_t ent[16];
  int n = 0;
  for (int i = 0; i < n_prefix && n < 14; ++i) ent[n++] = prefix[i];
  ent[n++] = (uint32_t)index;
  if (index >> 32) ent[n++] = (uint32_t)(index >> 32);
  uint32_t hc = SS_INIT_A;
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < n ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], hc));
}

// generate_state(n64, uint64): 2*n64 u32 words paired little-endian.
WV_HD void ss_generate_u64(const uint32_t pool[4], int n64, uint64_t* out) {
  uint32_t hc = SS_INIT_B;
  for (int i = 0; i < n64; ++i) {
    uint32_t w[2];
    for (int h = 0; h < 2; ++h) {
      uint32_t v = pool[(2 * i + h) & 3];
      v ^= hc;
      hc *= SS_MULT_B;
      v *= hc;
      v ^= v >> 16;
      w[h] = v;
    }
    out[i] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  }
}

// ---------------------------------------------------------------- PCG64 ----
constexpr uint64_t PCG_MULT_HI = 0x2360ED051FC65DA4ull;
constexpr uint64_t PCG_MULT_LO = 0x4385DF649FCCF645ull;

struct Pcg64 {
  u128 state, inc;
};

WV_HD u128 pcg_mult() { return u128{PCG_MULT_LO, PCG_MULT_HI}; }

WV_HD void pcg_step(Pcg64& g) { g.state = add128(mul128(g.state, pcg_mult()), g.inc); }

WV_HD uint64_t pcg_output(u128 s) {
  uint64_t v = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (v >> rot) | (v << ((64u - rot) & 63u));
}

// PCG64(SeedSequence(entropy)): initstate = g0<<64|g1, initseq = g2<<64|g3.
WV_HD Pcg64 pcg_seed(const uint32_t pool[4]) {
  uint64_t g[4];
  ss_generate_u64(pool, 4, g);
  Pcg64 r;
  r.state = u128{0, 0};
  u128 initseq{g[3], g[2]};
  r.inc = u128{(initseq.lo << 1) | 1ull, (initseq.hi << 1) | (initseq.lo >> 63)};
  pcg_step(r);
  r.state = add128(r.state, u128{g[1], g[0]});
  pcg_step(r);
  return r;
}

// Affine jump x -> A x + inc * S ; composition of (A1,S1) then (A2,S2):
// A = A2 A1, S = A2 S1 + S2.
struct PcgJump {
  u128 A, S;
};

WV_HD PcgJump jump_compose(PcgJump first, PcgJump second) {
  return PcgJump{mul128(second.A, first.A), add128(mul128(second.A, first.S), second.S)};
}

// Jump table entry b = 2^b steps, b in [0, 64).
WV_HD void pcg_jump_table(PcgJump* tab, int nbits) {
  PcgJump j{pcg_mult(), u128{1, 0}};
  for (int b = 0; b < nbits; ++b) {
    tab[b] = j;
    j = jump_compose(j, j);
  }
}

WV_HD PcgJump pcg_jump_n(const PcgJump* tab, uint64_t n) {
  PcgJump r{u128{1, 0}, u128{0, 0}};
  for (int b = 0; n; ++b, n >>= 1)
    if (n & 1) r = jump_compose(r, tab[b]);
  return r;
}

WV_HD double u64_to_double(uint64_t u) { return (double)(u >> 11) * (1.0 / 9007199254740992.0); }

// --------------------------------------------------------- Philox4x64 ----
constexpr uint64_t PH_M0 = 0xD2E7470EE14C6C93ull;
constexpr uint64_t PH_M1 = 0xCA5A826395121157ull;
constexpr uint64_t PH_W0 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t PH_W1 = 0xBB67AE8584CAA73Bull;

struct u64x4 {
  uint64_t x, y, z, w;
};

WV_HD u64x4 philox4x64_10(u64x4 c, uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += PH_W0;
      k1 += PH_W1;
    }
    uint64_t hi0 = mulhi64(PH_M0, c.x), lo0 = PH_M0 * c.x;
    uint64_t hi1 = mulhi64(PH_M1, c.z), lo1 = PH_M1 * c.z;
    c = u64x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

// numpy Philox stream element k (0-based) of a generator with counter 0:
// block counter 1 + k/4, word k%4.
WV_HD uint64_t philox_numpy_u64(uint64_t k0, uint64_t k1, uint64_t k) {
  u64x4 c{1 + (k >> 2), 0, 0, 0};
  if (c.x == 0) c.y = 1;  // carry (k near 2^64; never in practice)
  u64x4 o = philox4x64_10(c, k0, k1);
  switch (k & 3) {
    case 0: return o.x;
    case 1: return o.y;
    case 2: return o.z;
    default: return o.w;
  }
}

// ------------------------------------------------------- Philox4x32 -------
// Cheap device-native counter RNG for SGNS negatives (not numpy-compatible;
// numpy-stream parity for negatives is the explicit replay mode).
WV_HD void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = (uint32_t)p1;
    c[2] = n2;
    c[3] = (uint32_t)p0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

WV_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

}  // namespace wv

// ------------------------------------------------------ error handling ----
namespace wv {
void set_error(const char* fmt, ...);
void note_launches(int n);
}

#define WV_CHECK_ARG(cond, ...)          \
  do {                                   \
    if (!(cond)) {                       \
      ::wv::set_error(__VA_ARGS__);      \
      return -1;                         \
    }                                    \
  } while (0)

#define WV_CUDA(expr)                                                           \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::wv::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return -2;                                                                \
    }                                                                           \
  } while (0)

#define WV_CUDA_RC(expr)    \
  do {                      \
    int _rc = (expr);       \
    if (_rc) return _rc;    \
  } while (0)

#define WV_LAUNCH_CHECK()                                                          \
  do {                                                                             \
    ::wv::note_launches(1);                                                        \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) {                                                       \
      ::wv::set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return -2;                                                                   \
    }                                                                              \
  } while (0)
