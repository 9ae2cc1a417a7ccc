// Output formats: word2vec text / TSV embedding writers and
// the WVC1 walk-corpus writer, formatted on the device.
//
// Reference:
//   pipeline.save_embeddings_text  pipeline.py:236-243  "<count> <dim>" header, then
//                                  "<lexical> <d x %.8g>" per token
//   pipeline.save_embeddings_tsv   pipeline.py:246-251  escaped lexical, tab, d x %.8g
//   walks.save_corpus_binary       walks.py:344-364     "WVC1", strategy, projection,
//                                  u16 0, u32 count, then per walk u32 length + tokens
//   (walks.load_corpus_binary, walks.py:367-388, is a chain of length headers:
//    inherently sequential, it stays a host read)
//
// %.8g is Python's correctly rounded format (round-half-even on the exact binary
// value): the 8 significant digits are computed exactly with 192-bit integer
// arithmetic, then laid out with format()'s 'g' rules.  The device path covers
// zero and 1e-30 <= |x| < 1e16 (every trained embedding value); other values
// are reported so the caller can refuse them.
#include "common.cuh"
#include "primitives.cuh"
#include "../../include/walkvec_b200.h"

namespace wv {

struct U192 {
  uint64_t w[3];  // little-endian limbs
};

__device__ __forceinline__ U192 mul_64x128(uint64_t a, uint64_t blo, uint64_t bhi) {
  U192 r;
  r.w[0] = a * blo;
  const uint64_t c0 = __umul64hi(a, blo);
  const uint64_t lo1 = a * bhi;
  const uint64_t hi1 = __umul64hi(a, bhi);
  r.w[1] = c0 + lo1;
  r.w[2] = hi1 + (r.w[1] < c0 ? 1ull : 0ull);
  return r;
}

// bits [s, s+64) of v (s < 192)
__device__ __forceinline__ uint64_t bits64(const U192& v, int s) {
  const int li = s >> 6, sh = s & 63;
  uint64_t lo = li < 3 ? v.w[li] : 0ull;
  uint64_t hi = li + 1 < 3 ? v.w[li + 1] : 0ull;
  return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
}

// compare the low s bits of v with 2^(s-1): -1 below, 0 equal, 1 above
__device__ int cmp_half(const U192& v, int s) {
  const int hb = s - 1;
  const int li = hb >> 6;
  const uint64_t bit = (v.w[li] >> (hb & 63)) & 1ull;
  // any lower bit set?
  bool lower = (v.w[li] & ((1ull << (hb & 63)) - 1ull)) != 0ull;
  for (int i = 0; i < li; ++i) lower |= v.w[i] != 0ull;
  if (!bit) return -1;
  return lower ? 1 : 0;
}

__device__ __forceinline__ uint64_t round_shift(const U192& v, int s) {
  if (s <= 0) return v.w[0] << (-s);
  uint64_t q = bits64(v, s);
  const int c = cmp_half(v, s);
  if (c > 0 || (c == 0 && (q & 1ull))) ++q;
  return q;
}

__device__ __forceinline__ uint64_t round_div(unsigned __int128 num, unsigned __int128 den) {
  unsigned __int128 q = num / den, r = num - q * den;
  const unsigned __int128 twice = r * 2;
  if (twice > den || (twice == den && (q & 1))) ++q;
  return (uint64_t)q;
}

// 10^k, k in [0, 38), as (lo, hi)
__device__ __forceinline__ void pow10_128(int k, uint64_t& lo, uint64_t& hi) {
  unsigned __int128 p = 1;
  for (int i = 0; i < k; ++i) p *= 10;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
}

// N = round_half_even(|x| * 10^(7 - e10)); |x| = m 2^q
__device__ uint64_t scaled_digits(uint64_t m, int q, int e10) {
  const int k = 7 - e10;
  if (k >= 0) {
    uint64_t lo, hi;
    pow10_128(k, lo, hi);
    const U192 v = mul_64x128(m, lo, hi);
    return round_shift(v, -q);
  }
  const int j = -k;
  unsigned __int128 den = 1;
  for (int i = 0; i < j; ++i) den *= 10;
  unsigned __int128 num = m;
  if (q >= 0)
    num <<= q;
  else
    den <<= -q;
  return round_div(num, den);
}

// Python format(x, '.8g') -> out (<= 16 bytes), returns length or -1 (unsupported)
__device__ int fmt_g8(double x, char* out) {
  const uint64_t bits = (uint64_t)__double_as_longlong(x);
  const bool neg = bits >> 63;
  const int E = (int)((bits >> 52) & 0x7FF);
  const uint64_t M = bits & ((1ull << 52) - 1);
  int n = 0;
  if (E == 0x7FF) {  // inf / nan
    if (M) {
      out[0] = 'n'; out[1] = 'a'; out[2] = 'n';
      return 3;
    }
    if (neg) out[n++] = '-';
    out[n++] = 'i'; out[n++] = 'n'; out[n++] = 'f';
    return n;
  }
  if (neg) out[n++] = '-';
  if (E == 0 && M == 0) {
    out[n++] = '0';
    return n;
  }
  const double ax = fabs(x);
  if (!(ax >= 1e-30 && ax < 1e16)) return -1;
  const uint64_t m = M | (1ull << 52);
  const int q = E - 1075;
  int e10 = (int)floor(log10(ax));
  uint64_t N = scaled_digits(m, q, e10);
  if (N >= 100000000ull) {
    ++e10;
    N = scaled_digits(m, q, e10);
  } else if (N < 10000000ull) {
    --e10;
    N = scaled_digits(m, q, e10);
  }
  if (N >= 100000000ull) {  // rounding carried into a ninth digit (9.99999995 -> 10.000000)
    ++e10;
    N = scaled_digits(m, q, e10);
  }
  char dg[8];
  for (int i = 7; i >= 0; --i) {
    dg[i] = (char)('0' + N % 10);
    N /= 10;
  }
  int nd = 8;
  while (nd > 1 && dg[nd - 1] == '0') --nd;  // significant digits after stripping
  if (e10 >= -4 && e10 < 8) {
    if (e10 >= 0) {
      for (int i = 0; i <= e10; ++i) out[n++] = i < nd ? dg[i] : '0';
      if (nd > e10 + 1) {
        out[n++] = '.';
        for (int i = e10 + 1; i < nd; ++i) out[n++] = dg[i];
      }
    } else {
      out[n++] = '0';
      out[n++] = '.';
      for (int i = 0; i < -e10 - 1; ++i) out[n++] = '0';
      for (int i = 0; i < nd; ++i) out[n++] = dg[i];
    }
    return n;
  }
  out[n++] = dg[0];
  if (nd > 1) {
    out[n++] = '.';
    for (int i = 1; i < nd; ++i) out[n++] = dg[i];
  }
  out[n++] = 'e';
  int ex = e10;
  out[n++] = ex < 0 ? '-' : '+';
  if (ex < 0) ex = -ex;
  if (ex >= 100) out[n++] = (char)('0' + ex / 100);
  out[n++] = (char)('0' + (ex / 10) % 10);
  out[n++] = (char)('0' + ex % 10);
  return n;
}

// pass 1: every value formatted into a 16-byte cell; per-row byte counts
template <typename T>
__global__ void fmt_cells(const T* __restrict__ vec, int64_t rows, int d, const int64_t* __restrict__ lex_off,
                          char* __restrict__ cells, uint8_t* __restrict__ cell_len, int64_t* __restrict__ row_bytes,
                          int* __restrict__ bad) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t tot = (lex_off[r + 1] - lex_off[r]) + 1;  // lexical + '\n'
    for (int c = 0; c < d; ++c) {
      const int64_t i = r * d + c;
      const int len = fmt_g8((double)vec[i], cells + i * 16);
      if (len < 0) {
        atomicExch(bad, 1);
        cell_len[i] = 0;
        continue;
      }
      cell_len[i] = (uint8_t)len;
      tot += len + 1;  // separator before the value
    }
    row_bytes[r] = tot;
  }
}

// pass 2: lines "<lexical><sep><v0><sep>...<v{d-1}>\n" at the scanned offsets
__global__ void fmt_lines(const char* __restrict__ lex, const int64_t* __restrict__ lex_off, int64_t rows, int d,
                          const char* __restrict__ cells, const uint8_t* __restrict__ cell_len,
                          const int64_t* __restrict__ row_off, char sep, char* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    char* o = out + row_off[r];
    for (int64_t i = lex_off[r]; i < lex_off[r + 1]; ++i) *o++ = lex[i];
    for (int c = 0; c < d; ++c) {
      *o++ = sep;
      const int64_t i = r * d + c;
      const char* cc = cells + i * 16;
      for (int q = 0; q < cell_len[i]; ++q) *o++ = cc[q];
    }
    *o = '\n';
  }
}

// WVC1 body: per walk its u32 length then its tokens
__global__ void wvc1_pack(const int32_t* __restrict__ tokens, const int64_t* __restrict__ offsets, int64_t n_walks,
                          uint32_t* __restrict__ body) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_walks; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = offsets[w], L = offsets[w + 1] - o;
    uint32_t* dst = body + o + w;
    dst[0] = (uint32_t)L;
    for (int64_t j = 0; j < L; ++j) dst[1 + j] = (uint32_t)tokens[o + j];
  }
}


// ------------------------------------------------------------ WVC1 reader ---
// load_corpus_binary (walks.py:368-389): the body is a chain of records
// [len, tok_1 .. tok_len]; record r's header position depends on every earlier
// length.  Speculative chunk parsing: the body is cut into chunks of kRdChunk
// words; for each chunk and each candidate entry offset j < kRdCand (the first
// header at or after the chunk start lies within kRdCand words of it whenever
// records are shorter than kRdCand), one thread parses the chunk and records
// where the chain leaves it and how many records started inside.  One thread
// then follows the true entries chunk to chunk (one table lookup per chunk);
// every chunk is finally re-parsed from its true entry to emit offsets and
// tokens.  A record of kRdCand words or more sends the whole file to a
// sequential single-thread parse (correct for any file, slow).
constexpr int kRdChunk = 8192;
constexpr int kRdCand = 128;

static inline int64_t al256(int64_t b) { return (b + 255) & ~(int64_t)255; }

__global__ void wvc1_spec(const uint32_t* __restrict__ body, int64_t n, int64_t n_chunks, int32_t* __restrict__ exit_off,
                          int32_t* __restrict__ nrec) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_chunks * kRdCand) return;
  const int64_t c = t / kRdCand;
  const int j = (int)(t - c * kRdCand);
  const int64_t s0 = c * kRdChunk;
  const int64_t s1 = s0 + kRdChunk < n ? s0 + kRdChunk : n;  // the last chunk ends at the body's end
  int64_t p = s0 + j;
  int32_t cnt = 0, ex;
  bool long_rec = false;
  while (p < s1) {
    const uint32_t L = body[p];
    if ((int64_t)L + 1 >= kRdCand) {
      long_rec = true;
      break;
    }
    p += 1 + (int64_t)L;
    ++cnt;
  }
  // exit: -2 a record of kRdCand words or more; -1 the chain runs past the body;
  // else the entry offset into the next chunk (0 at the body's end = a clean end)
  if (long_rec) ex = -2;
  else if (p > n) ex = -1;
  else ex = (int32_t)(p - s1);
  exit_off[t] = ex;
  nrec[t] = cnt;
}

// follow the chain: chunk c's true entry offset and first record index; status 0 ok,
// 1 a long record (sequential fallback), 2 corrupt (overrun or trailing words),
// 3 the body ends before `count` records
__global__ void wvc1_resolve(const int32_t* __restrict__ exit_off, const int32_t* __restrict__ nrec, int64_t n_chunks,
                             int64_t count, int32_t* __restrict__ entry, int64_t* __restrict__ rec_base, int* status) {
  int64_t e = 0, r = 0;
  for (int64_t c = 0; c < n_chunks; ++c) {
    entry[c] = (int32_t)e;
    rec_base[c] = r;
    const int32_t ex = exit_off[c * kRdCand + e];
    if (ex == -2) {
      *status = 1;
      return;
    }
    if (ex == -1) {
      *status = 2;
      return;
    }
    r += nrec[c * kRdCand + e];
    e = ex;
  }
  *status = e != 0 ? 2 : (r == count ? 0 : (r < count ? 3 : 2));
}

__global__ void wvc1_emit(const uint32_t* __restrict__ body, int64_t n, int64_t n_chunks,
                          const int32_t* __restrict__ entry, const int64_t* __restrict__ rec_base,
                          int64_t* __restrict__ offsets, int32_t* __restrict__ tokens) {
  // warp per chunk: lane 0 walks the headers, the warp copies each record's tokens
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp; c < n_chunks; c += nw) {
    const int64_t s1 = (c + 1) * kRdChunk;
    int64_t p = c * kRdChunk + entry[c];
    int64_t r = rec_base[c];
    while (p < s1 && p < n) {
      const int64_t L = body[p];
      if (lane == 0) offsets[r + 1] = p + 1 + L - (r + 1);  // tokens before record r + 1
      for (int64_t q = lane; q < L; q += 32) tokens[p + 1 + q - (r + 1)] = (int32_t)body[p + 1 + q];
      p += 1 + L;
      ++r;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) offsets[0] = 0;
}

// any-length fallback: one thread, the reference's own loop
__global__ void wvc1_sequential(const uint32_t* __restrict__ body, int64_t n, int64_t count,
                                int64_t* __restrict__ offsets, int32_t* __restrict__ tokens, int* status) {
  int64_t p = 0, pos = 0;
  offsets[0] = 0;
  for (int64_t i = 0; i < count; ++i) {
    if (p >= n) {
      *status = 3;
      return;
    }
    const int64_t L = body[p];
    if (p + 1 + L > n) {
      *status = 2;
      return;
    }
    for (int64_t q = 0; q < L; ++q) tokens[pos + q] = (int32_t)body[p + 1 + q];
    p += 1 + L;
    pos += L;
    offsets[i + 1] = pos;
  }
  *status = p == n ? 0 : 2;
}

// ------------------------------------------------------ vocabulary TSV ----
// Vocabulary.save_tsv (ingest.py:307-323): per token "<token>\t<lexical with \\,
// \t, \n, \r escaped>\t<roles e/p>\t<count>\n" (_escape_field, ingest.py:345-346).
__device__ __forceinline__ int dec_digits(uint64_t v) {
  int n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

__device__ __forceinline__ bool tsv_special(uint8_t c) { return c == '\\' || c == '\t' || c == '\n' || c == '\r'; }

__global__ void vtsv_len(const uint8_t* __restrict__ lex, const int64_t* __restrict__ lex_off, int64_t rows,
                         const uint8_t* __restrict__ roles, const int64_t* __restrict__ counts, int64_t* __restrict__ len) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = dec_digits((uint64_t)r) + 1;
    for (int64_t i = lex_off[r]; i < lex_off[r + 1]; ++i) n += tsv_special(lex[i]) ? 2 : 1;
    n += 1 + ((roles[r] & 1) ? 1 : 0) + ((roles[r] & 2) ? 1 : 0) + 1 + dec_digits((uint64_t)counts[r]) + 1;
    len[r] = n;
  }
}

__device__ __forceinline__ char* put_dec(char* o, uint64_t v) {
  const int n = dec_digits(v);
  for (int i = n - 1; i >= 0; --i) {
    o[i] = (char)('0' + (int)(v % 10));
    v /= 10;
  }
  return o + n;
}

__global__ void vtsv_emit(const uint8_t* __restrict__ lex, const int64_t* __restrict__ lex_off, int64_t rows,
                          const uint8_t* __restrict__ roles, const int64_t* __restrict__ counts,
                          const int64_t* __restrict__ line_off, char* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    char* o = out + line_off[r];
    o = put_dec(o, (uint64_t)r);
    *o++ = '\t';
    for (int64_t i = lex_off[r]; i < lex_off[r + 1]; ++i) {
      const uint8_t c = lex[i];
      if (tsv_special(c)) {
        *o++ = '\\';
        *o++ = c == '\\' ? '\\' : (c == '\t' ? 't' : (c == '\n' ? 'n' : 'r'));
      } else {
        *o++ = (char)c;
      }
    }
    *o++ = '\t';
    if (roles[r] & 1) *o++ = 'e';
    if (roles[r] & 2) *o++ = 'p';
    *o++ = '\t';
    o = put_dec(o, (uint64_t)counts[r]);
    *o++ = '\n';
  }
}
}  // namespace wv

extern "C" {

int64_t wv_format_workspace_bytes(int64_t rows, int d) {
  return (rows * d * 16 + 255) / 256 * 256 + (rows * d + 255) / 256 * 256 + ((rows + 1) * 8 + 255) / 256 * 256 * 2 +
         (wv::scan_tiles(rows + 1) * 8 + 255) / 256 * 256 + 1024;
}

// Phase 1 of a text export: total bytes (*total, device) of the lines for
// `rows` vectors (fp32 or fp64) with the given lexical bytes (lex[lex_off[r],
// lex_off[r+1]) per row); *bad = 1 when a value is outside the device
// formatter's range.  Phase 2 (wv_format_emit) writes them into `out`.
int wv_format_plan(const void* vec, int precision, int64_t rows, int d, const int64_t* lex_off, int64_t* total,
                   int* bad, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(rows >= 1 && d >= 1, "bad sizes");
  WV_CHECK_ARG(ws_bytes >= wv_format_workspace_bytes(rows, d), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  char* cells = w;
  w += (rows * d * 16 + 255) / 256 * 256;
  uint8_t* cell_len = (uint8_t*)w;
  w += (rows * d + 255) / 256 * 256;
  int64_t* row_bytes = (int64_t*)w;
  w += ((rows + 1) * 8 + 255) / 256 * 256;
  int64_t* row_off = (int64_t*)w;
  w += ((rows + 1) * 8 + 255) / 256 * 256;
  int64_t* scan_ws = (int64_t*)w;
  WV_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const unsigned g = (unsigned)((rows + 127) / 128 < 148 * 16 ? (rows + 127) / 128 : 148 * 16);
  if (precision == WV_FP32)
    fmt_cells<float><<<g, 128, 0, st>>>((const float*)vec, rows, d, lex_off, cells, cell_len, row_bytes, bad);
  else
    fmt_cells<double><<<g, 128, 0, st>>>((const double*)vec, rows, d, lex_off, cells, cell_len, row_bytes, bad);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<int64_t, int64_t>(row_bytes, rows, row_off, total, scan_ws, st)));
  return 0;
}

int wv_format_emit(const char* lex, const int64_t* lex_off, int64_t rows, int d, char sep, char* out, void* ws,
                   int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(ws_bytes >= wv_format_workspace_bytes(rows, d), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  char* cells = w;
  w += (rows * d * 16 + 255) / 256 * 256;
  uint8_t* cell_len = (uint8_t*)w;
  w += (rows * d + 255) / 256 * 256;
  w += ((rows + 1) * 8 + 255) / 256 * 256;
  int64_t* row_off = (int64_t*)w;
  const unsigned g = (unsigned)((rows + 127) / 128 < 148 * 16 ? (rows + 127) / 128 : 148 * 16);
  fmt_lines<<<g, 128, 0, st>>>(lex, lex_off, rows, d, cells, cell_len, row_off, sep, out);
  WV_LAUNCH_CHECK();
  return 0;
}

// WVC1 body (u32 length + tokens per walk; the 12-byte header is the caller's)
int wv_wvc1_pack(const int32_t* tokens, const int64_t* offsets, int64_t n_walks, uint32_t* body, void* stream) {
  using namespace wv;
  if (n_walks == 0) return 0;
  const unsigned g = (unsigned)((n_walks + 255) / 256 < 148 * 32 ? (n_walks + 255) / 256 : 148 * 32);
  wvc1_pack<<<g, 256, 0, (cudaStream_t)stream>>>(tokens, offsets, n_walks, body);
  WV_LAUNCH_CHECK();
  return 0;
}


int64_t wv_wvc1_read_workspace_bytes(int64_t n_words) {
  const int64_t chunks = (n_words + wv::kRdChunk - 1) / wv::kRdChunk;
  return 2 * wv::al256(chunks * wv::kRdCand * 4) + wv::al256(chunks * 4) + wv::al256(chunks * 8) + 256 + 1024;
}

int wv_wvc1_read(const uint32_t* body, int64_t n_words, int64_t count, int64_t* offsets, int32_t* tokens, int* status,
                 void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(n_words >= 0 && count >= 0, "bad sizes");
  WV_CHECK_ARG(ws_bytes >= wv_wvc1_read_workspace_bytes(n_words), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t chunks = (n_words + kRdChunk - 1) / kRdChunk;
  char* w = (char*)ws;
  int32_t* exit_off = (int32_t*)w;
  w += al256(chunks * kRdCand * 4);
  int32_t* nrec = (int32_t*)w;
  w += al256(chunks * kRdCand * 4);
  int32_t* entry = (int32_t*)w;
  w += al256(chunks * 4);
  int64_t* rec_base = (int64_t*)w;
  WV_CUDA(cudaMemsetAsync(status, 0, sizeof(int), st));
  if (n_words == 0) {
    WV_CUDA(cudaMemsetAsync(offsets, 0, 8, st));
    if (count != 0) {
      static const int three = 3;  // the body ends before `count` records
      WV_CUDA(cudaMemcpyAsync(status, &three, sizeof(int), cudaMemcpyHostToDevice, st));
      WV_CUDA(cudaStreamSynchronize(st));
    }
    return 0;
  }
  const int64_t nt = chunks * kRdCand;
  wvc1_spec<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(body, n_words, chunks, exit_off, nrec);
  WV_LAUNCH_CHECK();
  wvc1_resolve<<<1, 1, 0, st>>>(exit_off, nrec, chunks, count, entry, rec_base, status);
  WV_LAUNCH_CHECK();
  int h_status = 0;
  WV_CUDA(cudaMemcpyAsync(&h_status, status, sizeof(int), cudaMemcpyDeviceToHost, st));
  WV_CUDA(cudaStreamSynchronize(st));
  if (h_status == 1) {
    WV_CUDA(cudaMemsetAsync(status, 0, sizeof(int), st));
    wvc1_sequential<<<1, 1, 0, st>>>(body, n_words, count, offsets, tokens, status);
    WV_LAUNCH_CHECK();
    return 0;
  }
  if (h_status != 0) return 0;  // corrupt: the caller raises (status stays 2)
  const unsigned g = (unsigned)((chunks * 32 + 255) / 256 < 148 * 16 ? (chunks * 32 + 255) / 256 : 148 * 16);
  wvc1_emit<<<g, 256, 0, st>>>(body, n_words, chunks, entry, rec_base, offsets, tokens);
  WV_LAUNCH_CHECK();
  return 0;
}

int64_t wv_vocab_tsv_workspace_bytes(int64_t rows) {
  return wv::al256((rows + 1) * 8) + wv::al256(wv::scan_tiles(rows + 1) * 8) + 512;
}

int wv_vocab_tsv(const uint8_t* lex, const int64_t* lex_off, int64_t rows, const uint8_t* roles, const int64_t* counts,
                 char* out, int64_t* total, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(rows >= 0, "bad sizes");
  WV_CHECK_ARG(ws_bytes >= wv_vocab_tsv_workspace_bytes(rows), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  int64_t* line = (int64_t*)w;
  w += al256((rows + 1) * 8);
  int64_t* sws = (int64_t*)w;
  if (rows == 0) {
    WV_CUDA(cudaMemsetAsync(total, 0, 8, st));
    return 0;
  }
  const unsigned g = (unsigned)((rows + 255) / 256 < 148 * 16 ? (rows + 255) / 256 : 148 * 16);
  vtsv_len<<<g, 256, 0, st>>>(lex, lex_off, rows, roles, counts, line);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<int64_t, int64_t>(line, rows, line, total, sws, st)));
  if (out != nullptr) {
    vtsv_emit<<<g, 256, 0, st>>>(lex, lex_off, rows, roles, counts, line, out);
    WV_LAUNCH_CHECK();
  }
  return 0;
}
}  // extern "C"
