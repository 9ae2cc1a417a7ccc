// GPU ingest: N-Triples / delimited-table parsing and first-occurrence
// interning of string keys (the step before the path).
//
// Reference (pkg/src/walkvec/ingest.py):
//   parse_ntriples     :188-229  universal-newline lines; blank and '#' lines
//                                skipped; malformed lines -> ParseError(line)
//   _scan_term         :116-164  <iri> (unescaped), _:blank, "literal" (unescaped,
//                                ^^<datatype> / @lang consumed and dropped)
//   _parse_statement   :167-185  subject not literal, predicate IRI, '.', '#' tail
//   _unescape          :72-101   \t \b \n \r \f \" \' \\ \uXXXX \UXXXXXXXX
//   parse_edge_table   :234-257  txt: whitespace split; csv/tsv: delimiter split
//   build_vocabulary   :368-396  tokens by first occurrence over the (s, p, o)
//                                stream; literal objects dropped (s, p still
//                                interned) unless include_literals
//
// Keys are compared as unescaped strings (the reference's dict keys), so a
// key's 64-bit hash runs over its unescaped UTF-8 bytes; every occurrence is
// then verified byte-for-byte against its key's first occurrence, and a hash
// collision is reported (never silently merged).
#include "common.cuh"
#include "primitives.cuh"
#include "../../include/walkvec_b200.h"

namespace wv {

enum : uint8_t { TK_IRI = 0, TK_BLANK = 1, TK_LIT = 2 };
enum : uint8_t { LN_SKIP = 0, LN_OK = 1, LN_PARSE_ERR = 2, LN_VALUE_ERR = 3 };

__device__ __forceinline__ bool is_ws(uint8_t c) { return c == ' ' || c == '\t'; }
// str.isspace() restricted to ASCII (the reference's blank-node label end)
__device__ __forceinline__ bool is_space(uint8_t c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 28 && c <= 31); }
__device__ __forceinline__ bool is_alnum(uint8_t c) {
  return (c >= '0' && c <= '9') || (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c >= 0x80;
}
__device__ __forceinline__ int hexval(uint8_t c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

// Unescaped byte stream of a raw span (escapes decoded, code points re-encoded
// as UTF-8, lone surrogates with the generic 3-byte form).
// mode: 0 raw bytes; 1 N-Triples escapes; 2 a csv.reader quoted field (opening
// quote skipped, "" -> ", characters after the closing quote kept literally)
struct KeyIter {
  const uint8_t* p;
  const uint8_t* e;
  uint8_t esc;
  uint8_t qs;  // csv: 0 before the opening quote, 1 inside the quotes, 2 after the closing quote
  uint8_t buf[4];
  int nb, ib;
  __device__ KeyIter(const uint8_t* text, int64_t s, int64_t t, uint8_t mode)
      : p(text + s), e(text + t), esc(mode), qs(0), nb(0), ib(0) {}
  __device__ bool next(uint8_t& out) {
    if (ib < nb) {
      out = buf[ib++];
      return true;
    }
    if (esc == 2) {
      while (p < e) {
        const uint8_t c = *p++;
        if (qs == 0) {  // the opening quote
          qs = 1;
          continue;
        }
        if (qs == 1 && c == '"') {
          if (p < e && *p == '"') {  // doubled quote
            ++p;
            out = '"';
            return true;
          }
          qs = 2;  // closing quote
          continue;
        }
        out = c;
        return true;
      }
      return false;
    }
    if (p >= e) return false;
    const uint8_t c = *p;
    if (!esc || c != '\\' || p + 1 >= e) {
      ++p;
      out = c;
      return true;
    }
    const uint8_t x = p[1];
    uint32_t cp;
    switch (x) {
      case 't': cp = '\t'; p += 2; break;
      case 'b': cp = '\b'; p += 2; break;
      case 'n': cp = '\n'; p += 2; break;
      case 'r': cp = '\r'; p += 2; break;
      case 'f': cp = '\f'; p += 2; break;
      case '"': cp = '"'; p += 2; break;
      case '\'': cp = '\''; p += 2; break;
      case '\\': cp = '\\'; p += 2; break;
      default: {  // u / U (validated by the parser)
        const int w = x == 'u' ? 4 : 8;
        cp = 0;
        for (int q = 0; q < w; ++q) cp = cp * 16 + (uint32_t)hexval(p[2 + q]);
        p += 2 + w;
      }
    }
    if (cp < 0x80) {
      out = (uint8_t)cp;
      return true;
    }
    if (cp < 0x800) {
      buf[0] = (uint8_t)(0xC0 | (cp >> 6));
      buf[1] = (uint8_t)(0x80 | (cp & 0x3F));
      nb = 2;
    } else if (cp < 0x10000) {
      buf[0] = (uint8_t)(0xE0 | (cp >> 12));
      buf[1] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
      buf[2] = (uint8_t)(0x80 | (cp & 0x3F));
      nb = 3;
    } else {
      buf[0] = (uint8_t)(0xF0 | (cp >> 18));
      buf[1] = (uint8_t)(0x80 | ((cp >> 12) & 0x3F));
      buf[2] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
      buf[3] = (uint8_t)(0x80 | (cp & 0x3F));
      nb = 4;
    }
    ib = 1;
    out = buf[0];
    return true;
  }
};

__device__ uint64_t key_hash(const uint8_t* text, int64_t s, int64_t t, uint8_t esc, uint64_t seed) {
  KeyIter it(text, s, t, esc);
  uint64_t h = 0xcbf29ce484222325ull ^ (seed ? splitmix64(seed) : 0ull);
  uint64_t n = 0;
  uint8_t b;
  while (it.next(b)) {
    h = (h ^ b) * 0x100000001b3ull;
    ++n;
  }
  h = splitmix64(h ^ (n * 0x9E3779B97F4A7C15ull) ^ (seed * 0xD6E8FEB86659FD93ull));
  return h ? h : 1ull;  // 0 marks an empty table slot
}

__device__ bool key_equal(const uint8_t* text, int64_t s1, int64_t t1, uint8_t e1, int64_t s2, int64_t t2,
                          uint8_t e2) {
  if (!e1 && !e2) {
    if (t1 - s1 != t2 - s2) return false;
    for (int64_t i = 0; i < t1 - s1; ++i)
      if (text[s1 + i] != text[s2 + i]) return false;
    return true;
  }
  KeyIter a(text, s1, t1, e1), b(text, s2, t2, e2);
  uint8_t x, y;
  while (true) {
    const bool ha = a.next(x), hb = b.next(y);
    if (ha != hb) return false;
    if (!ha) return true;
    if (x != y) return false;
  }
}

// Validate the escapes of a raw span (_unescape, ingest.py:72-101); returns 0 or an error code
// and the offending position.
enum : int {
  E_NONE = 0,
  E_DANGLING = 1,       // dangling escape at end of string
  E_TRUNC = 2,          // truncated \%c escape
  E_BADHEX = 3,         // bad \%c escape: %r
  E_UNKNOWN_ESC = 4,    // unknown escape \%c
  E_EOS = 5,            // unexpected end of statement
  E_UNTERM_IRI = 6,     // unterminated IRI
  E_EMPTY_BLANK = 7,    // empty blank node label
  E_UNTERM_LIT = 8,     // unterminated literal
  E_NO_DT_IRI = 9,      // expected datatype IRI after ^^
  E_UNTERM_DT = 10,     // unterminated datatype IRI
  E_EMPTY_LANG = 11,    // empty language tag
  E_UNEXPECTED = 12,    // unexpected character %r
  E_LIT_SUBJECT = 13,   // literal not allowed as subject
  E_PRED_NOT_IRI = 14,  // predicate must be an IRI
  E_NO_DOT = 15,        // expected terminating '.'
  E_TRAILING = 16,      // trailing content after '.'
  E_COLUMNS = 17,       // expected 3 columns, got %d
  E_EMPTY_SP = 18,      // subject and predicate must be non-empty (ValueError)
  E_QUOTED = 19,        // quoted csv/tsv field (csv.reader quoting): not supported on the device
};

__device__ int check_escapes(const uint8_t* text, int64_t s, int64_t t, int64_t& at) {
  for (int64_t i = s; i < t; ++i) {
    if (text[i] != '\\') continue;
    at = i;
    if (i + 1 >= t) return E_DANGLING;
    const uint8_t x = text[i + 1];
    if (x == 't' || x == 'b' || x == 'n' || x == 'r' || x == 'f' || x == '"' || x == '\'' || x == '\\') {
      ++i;
      continue;
    }
    if (x == 'u' || x == 'U') {
      const int w = x == 'u' ? 4 : 8;
      if (i + 2 + w > t) return E_TRUNC;
      uint64_t cp = 0;
      for (int q = 0; q < w; ++q) {
        const int v = hexval(text[i + 2 + q]);
        if (v < 0) return E_BADHEX;
        cp = cp * 16 + (uint64_t)v;
      }
      if (cp > 0x10FFFF) return E_BADHEX;  // chr() raises ValueError -> same message
      i += 1 + w;
      continue;
    }
    return E_UNKNOWN_ESC;
  }
  return E_NONE;
}

struct Term {
  int64_t s, t;  // key span
  uint8_t kind;
  uint8_t esc;   // span holds escapes
};

// _scan_term (ingest.py:116-164) from position i of [.., end); returns error code, sets next
__device__ int scan_term(const uint8_t* text, int64_t i, int64_t end, Term& out, int64_t& next, int64_t& at) {
  at = i;
  if (i >= end) return E_EOS;
  const uint8_t c = text[i];
  if (c == '<') {
    int64_t j = i + 1;
    while (j < end && text[j] != '>') ++j;
    if (j >= end) return E_UNTERM_IRI;
    out.s = i + 1;
    out.t = j;
    out.kind = TK_IRI;
    const int e = check_escapes(text, out.s, out.t, at);
    if (e) return e;
    out.esc = 0;
    for (int64_t q = out.s; q < out.t; ++q) out.esc |= text[q] == '\\';
    next = j + 1;
    return E_NONE;
  }
  if (c == '_' && i + 1 < end && text[i + 1] == ':') {
    int64_t j = i + 2;
    while (j < end && !is_space(text[j])) ++j;
    if (j == i + 2) return E_EMPTY_BLANK;
    out.s = i;
    out.t = j;
    out.kind = TK_BLANK;
    out.esc = 0;
    next = j;
    return E_NONE;
  }
  if (c == '"') {
    int64_t j = i + 1;
    while (j < end) {
      if (text[j] == '\\') {
        j += 2;
        continue;
      }
      if (text[j] == '"') break;
      ++j;
    }
    if (j >= end) return E_UNTERM_LIT;
    out.s = i + 1;
    out.t = j;
    out.kind = TK_LIT;
    const int e = check_escapes(text, out.s, out.t, at);
    if (e) return e;
    out.esc = 0;
    for (int64_t q = out.s; q < out.t; ++q) out.esc |= text[q] == '\\';
    j += 1;
    if (j + 2 <= end && text[j] == '^' && text[j + 1] == '^') {
      j += 2;
      at = j;
      if (j >= end || text[j] != '<') return E_NO_DT_IRI;
      int64_t q = j + 1;
      while (q < end && text[q] != '>') ++q;
      if (q >= end) return E_UNTERM_DT;
      j = q + 1;
    } else if (j < end && text[j] == '@') {
      j += 1;
      const int64_t st = j;
      while (j < end && (is_alnum(text[j]) || text[j] == '-')) ++j;
      at = j;
      if (j == st) return E_EMPTY_LANG;
    }
    next = j;
    return E_NONE;
  }
  return E_UNEXPECTED;
}

// line terminators of universal-newline text mode: '\n', '\r\n' (at the '\n'), lone '\r'
__global__ void ingest_line_ends(const uint8_t* __restrict__ text, int64_t n, uint8_t* __restrict__ term) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t c = text[i];
    term[i] = (c == '\n' || (c == '\r' && (i + 1 == n || text[i + 1] != '\n'))) ? 1 : 0;
  }
}

__global__ void ingest_line_bounds(const uint8_t* __restrict__ term, const int64_t* __restrict__ pos, int64_t n,
                                   int64_t* __restrict__ line_end) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (term[i]) line_end[pos[i]] = i;
}

// ------------------------------------------------------ csv.reader records --
// Quoted csv/tsv fields may hold delimiters and line breaks, so a record is not a
// line.  csv.reader's quoting (excel dialect, strict=False) as a per-byte state
// machine: 0 start of field, 1 unquoted field, 2 quoted field, 3 quote seen in a
// quoted field.  A '\n' / lone '\r' / the '\n' of "\r\n" ends a record unless the
// state before it is 2.  The states entering each 4 KB chunk come from composing
// per-chunk transition maps (4 states -> 4 states).
constexpr int64_t kCsvChunk = 4096;

__device__ __forceinline__ uint8_t csv_step(uint8_t st, uint8_t c, uint8_t delim) {
  if (c == '"') return st == 0 ? 2 : (st == 1 ? 1 : (st == 2 ? 3 : 2));
  if (c == delim || c == '\n' || c == '\r') return st == 2 ? 2 : 0;
  return st == 2 ? 2 : 1;
}

__global__ void csv_chunk_maps(const uint8_t* __restrict__ text, int64_t n, uint8_t delim, int64_t n_chunks,
                               uint8_t* __restrict__ maps) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_chunks * 4) return;
  const int64_t c = t >> 2;
  uint8_t st = (uint8_t)(t & 3);
  const int64_t e = min(n, (c + 1) * kCsvChunk);
  for (int64_t i = c * kCsvChunk; i < e; ++i) st = csv_step(st, text[i], delim);
  maps[t] = st;
}

// one block: the state entering every chunk (thread ranges composed, then resolved in order)
__global__ void __launch_bounds__(1024) csv_chunk_states(const uint8_t* __restrict__ maps, int64_t n_chunks,
                                                         uint8_t* __restrict__ start) {
  __shared__ uint8_t f[1024][4];
  __shared__ uint8_t entry[1024];
  const int64_t per = (n_chunks + 1023) / 1024;
  const int64_t c0 = threadIdx.x * per, c1 = min(n_chunks, c0 + per);
  uint8_t g[4] = {0, 1, 2, 3};
  for (int64_t c = c0; c < c1; ++c)
    for (int s = 0; s < 4; ++s) g[s] = maps[4 * c + g[s]];
  for (int s = 0; s < 4; ++s) f[threadIdx.x][s] = g[s];
  __syncthreads();
  if (threadIdx.x == 0) {
    uint8_t st = 0;
    for (int j = 0; j < 1024; ++j) {
      entry[j] = st;
      st = f[j][st];
    }
  }
  __syncthreads();
  uint8_t st = entry[threadIdx.x];
  for (int64_t c = c0; c < c1; ++c) {
    start[c] = st;
    st = maps[4 * c + st];
  }
}

// record terminators (rec) and universal-newline line terminators (phys)
__global__ void csv_terms(const uint8_t* __restrict__ text, int64_t n, uint8_t delim, int64_t n_chunks,
                          const uint8_t* __restrict__ start, uint8_t* __restrict__ rec, uint8_t* __restrict__ phys) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_chunks; c += (int64_t)gridDim.x * blockDim.x) {
    uint8_t st = start[c];
    const int64_t e = min(n, (c + 1) * kCsvChunk);
    for (int64_t i = c * kCsvChunk; i < e; ++i) {
      const uint8_t ch = text[i];
      const bool term = ch == '\n' || (ch == '\r' && (i + 1 == n || text[i + 1] != '\n'));
      phys[i] = term ? 1 : 0;
      rec[i] = (term && st != 2) ? 1 : 0;
      st = csv_step(st, ch, delim);
    }
  }
}

__global__ void csv_record_bounds(const uint8_t* __restrict__ rec, const int64_t* __restrict__ rpos,
                                  const int64_t* __restrict__ ppos, int64_t n, int64_t* __restrict__ rec_end,
                                  int64_t* __restrict__ rec_line) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (rec[i]) {
      rec_end[rpos[i]] = i;
      rec_line[rpos[i]] = ppos[i] + 1;  // csv.reader's line_num after the record
    }
}

// Per line: status, error (code, byte position) and the three key spans.
// mode: 0 N-Triples; 1 whitespace table; 2 delimiter table (delim)
__global__ void ingest_parse(const uint8_t* __restrict__ text, int64_t n, const int64_t* __restrict__ line_end,
                             int64_t n_lines, int mode, uint8_t delim, int has_header,
                             const int64_t* __restrict__ line_no, uint8_t* __restrict__ status,
                             int32_t* __restrict__ err, int64_t* __restrict__ err_at, Term* __restrict__ terms) {
  for (int64_t L = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; L < n_lines;
       L += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = L == 0 ? 0 : line_end[L - 1] + 1;
    int64_t e = line_end[L];  // an unterminated last line ends at n (set by the caller)
    if (e > n) e = n;
    if (e > b && text[e - 1] == '\r' && e < n && text[e] == '\n') --e;  // "\r\n"
    status[L] = LN_SKIP;
    err[L] = 0;
    Term* tm = terms + 3 * L;
    if (mode == 0) {
      // blank (after Python strip) or comment line
      int64_t q = b;
      while (q < e && is_space(text[q])) ++q;
      if (q >= e || text[q] == '#') continue;
      int code = E_NONE;
      int64_t at = b, i = b;
      while (i < e && is_ws(text[i])) ++i;
      code = scan_term(text, i, e, tm[0], i, at);
      if (!code && tm[0].kind == TK_LIT) code = E_LIT_SUBJECT;
      if (!code) {
        while (i < e && is_ws(text[i])) ++i;
        code = scan_term(text, i, e, tm[1], i, at);
        if (!code && tm[1].kind != TK_IRI) code = E_PRED_NOT_IRI;
      }
      if (!code) {
        while (i < e && is_ws(text[i])) ++i;
        code = scan_term(text, i, e, tm[2], i, at);
      }
      if (!code) {
        while (i < e && is_ws(text[i])) ++i;
        at = i;
        if (i >= e || text[i] != '.') {
          code = E_NO_DOT;
        } else {
          ++i;
          while (i < e && is_ws(text[i])) ++i;
          if (i < e && text[i] != '#') code = E_TRAILING;
        }
      }
      if (!code && (tm[0].t == tm[0].s || tm[1].t == tm[1].s)) code = E_EMPTY_SP;  // Triple.__post_init__
      status[L] = code == E_NONE ? LN_OK : (code == E_EMPTY_SP ? LN_VALUE_ERR : LN_PARSE_ERR);
      err[L] = code;
      err_at[L] = at;
      continue;
    }
    // tables: every non-empty row becomes a resource triple (exactly 3 columns);
    // the header is the row csv.reader reports at line 1
    if (has_header && (line_no ? line_no[L] == 1 : L == 0)) continue;
    int cols = 0;
    int64_t i = b;
    bool quoted = false;
    if (mode == 1) {
      while (true) {
        while (i < e && is_space(text[i])) ++i;
        if (i >= e) break;
        const int64_t s = i;
        while (i < e && !is_space(text[i])) ++i;
        if (cols < 3) tm[cols] = Term{s, i, TK_IRI, 0};
        ++cols;
      }
    } else if (mode == 2) {
      if (e == b) continue;  // csv.reader yields [] for an empty row
      int64_t s = b;
      for (i = b; i <= e; ++i) {
        if (i < e && i == s && text[i] == '"') quoted = true;
        if (i == e || text[i] == delim) {
          if (cols < 3) tm[cols] = Term{s, i, TK_IRI, 0};
          ++cols;
          s = i + 1;
        }
      }
    } else {  // mode 3: a csv.reader record with quoting (the record may span lines)
      if (e == b) continue;
      int64_t s = b;
      uint8_t st = 0;
      for (i = b; i <= e; ++i) {
        if (i == e || (text[i] == delim && st != 2)) {
          const uint8_t q = (i > s && text[s] == '"') ? 2 : 0;  // a field opened by a quote
          if (cols < 3) tm[cols] = Term{s, i, TK_IRI, q};
          ++cols;
          s = i + 1;
          st = 0;
          continue;
        }
        st = csv_step(st, text[i], delim);
      }
    }
    if (cols == 0) continue;
    int code = cols == 3 ? E_NONE : E_COLUMNS;
    if (mode == 2 && quoted) code = E_QUOTED;
    // an empty key: an empty span, or (quoted) exactly the two quotes
    auto empty_key = [&](const Term& x) {
      return x.t == x.s || (x.esc == 2 && x.t - x.s == 2 && text[x.s + 1] == '"');
    };
    if (!code && (empty_key(tm[0]) || empty_key(tm[1]))) code = E_EMPTY_SP;
    status[L] = code == E_NONE ? LN_OK : (code == E_EMPTY_SP ? LN_VALUE_ERR : LN_PARSE_ERR);
    err[L] = code == E_COLUMNS ? -cols : code;
    err_at[L] = b;
  }
}

__global__ void ingest_ok_flags(const uint8_t* __restrict__ status, int64_t n_lines, uint8_t* __restrict__ ok) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_lines; i += (int64_t)gridDim.x * blockDim.x)
    ok[i] = status[i] == LN_OK ? 1 : 0;
}

__global__ void ingest_first_bad(const uint8_t* __restrict__ status, int64_t n_lines, int64_t* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_lines; i += (int64_t)gridDim.x * blockDim.x) {
    if (status[i] >= LN_PARSE_ERR) atomicMin((unsigned long long*)bad, (unsigned long long)i);
    if (status[i] == LN_VALUE_ERR) atomicMin((unsigned long long*)(bad + 1), (unsigned long long)i);
  }
}

// statements in line order -> occurrence spans (3 per statement)
__global__ void ingest_statements(const uint8_t* __restrict__ status, const int64_t* __restrict__ stmt_of_line,
                                  int64_t n_lines, const Term* __restrict__ terms, Term* __restrict__ occ) {
  for (int64_t L = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; L < n_lines;
       L += (int64_t)gridDim.x * blockDim.x) {
    if (status[L] != LN_OK) continue;
    const int64_t j = stmt_of_line[L];
    occ[3 * j] = terms[3 * L];
    occ[3 * j + 1] = terms[3 * L + 1];
    occ[3 * j + 2] = terms[3 * L + 2];
  }
}

struct Table {
  unsigned long long* key;    // hash (0 = empty)
  unsigned long long* first;  // first occurrence position
  int64_t* token;
  uint64_t mask;
  uint64_t seed;  // hash seed: a collision (reported, never merged) is retried with another seed
};

__device__ __forceinline__ bool occ_active(const Term* occ, int64_t pos, int include_literals) {
  return (pos % 3) != 2 || include_literals || occ[pos].kind != TK_LIT;
}

__global__ void ingest_insert(const uint8_t* __restrict__ text, const Term* __restrict__ occ, int64_t n_occ,
                              int include_literals, Table T, uint32_t* __restrict__ occ_slot) {
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < n_occ;
       pos += (int64_t)gridDim.x * blockDim.x) {
    if (!occ_active(occ, pos, include_literals)) continue;
    const Term tm = occ[pos];
    const unsigned long long h = key_hash(text, tm.s, tm.t, tm.esc, T.seed);
    uint64_t slot = h & T.mask;
    while (true) {
      const unsigned long long prev = atomicCAS(T.key + slot, 0ull, h);
      if (prev == 0ull || prev == h) break;
      slot = (slot + 1) & T.mask;
    }
    atomicMin(T.first + slot, (unsigned long long)pos);
    occ_slot[pos] = (uint32_t)slot;
  }
}

// every occurrence equals its key's first occurrence (hash collisions are errors)
__global__ void ingest_verify(const uint8_t* __restrict__ text, const Term* __restrict__ occ, int64_t n_occ,
                              int include_literals, Table T, const uint32_t* __restrict__ occ_slot,
                              int* __restrict__ collision) {
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < n_occ;
       pos += (int64_t)gridDim.x * blockDim.x) {
    if (!occ_active(occ, pos, include_literals)) continue;
    const int64_t f = (int64_t)T.first[occ_slot[pos]];
    if (f == pos) continue;
    const Term a = occ[pos], b = occ[f];
    if (!key_equal(text, a.s, a.t, a.esc, b.s, b.t, b.esc)) atomicExch(collision, 1);
  }
}

__global__ void ingest_collect(Table T, int64_t cap, uint32_t* __restrict__ firsts, uint32_t* __restrict__ slots,
                               unsigned long long* __restrict__ n_unique) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cap; s += (int64_t)gridDim.x * blockDim.x) {
    if (T.key[s] == 0ull) continue;
    const unsigned long long at = atomicAdd(n_unique, 1ull);
    firsts[at] = (uint32_t)T.first[s];
    slots[at] = (uint32_t)s;
  }
}

// token r = rank of its key's first position; its lexical span = that occurrence's key span
__global__ void ingest_rank(const uint32_t* __restrict__ firsts, const uint32_t* __restrict__ slots,
                            const unsigned long long* __restrict__ n_unique, Table T, const Term* __restrict__ occ,
                            int64_t* __restrict__ tok_span) {
  const int64_t n = (int64_t)*n_unique;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    T.token[slots[r]] = r;
    const Term tm = occ[firsts[r]];
    tok_span[3 * r] = tm.s;
    tok_span[3 * r + 1] = tm.t;
    tok_span[3 * r + 2] = (int64_t)tm.esc | ((int64_t)tm.kind << 2);
  }
}

__global__ void ingest_kept_flags(const Term* __restrict__ occ, int64_t n_stmt, int include_literals,
                                  uint8_t* __restrict__ kept) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_stmt; j += (int64_t)gridDim.x * blockDim.x)
    kept[j] = (include_literals || occ[3 * j + 2].kind != TK_LIT) ? 1 : 0;
}

// edges of kept statements (literal-object statements dropped unless include_literals)
__global__ void ingest_edges(int64_t n_stmt, Table T, const uint32_t* __restrict__ occ_slot,
                             const uint8_t* __restrict__ kept, const int64_t* __restrict__ edge_of,
                             int64_t* __restrict__ edges) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_stmt; j += (int64_t)gridDim.x * blockDim.x) {
    if (!kept[j]) continue;
    int64_t* row = edges + 3 * edge_of[j];
    row[0] = T.token[occ_slot[3 * j]];
    row[1] = T.token[occ_slot[3 * j + 1]];
    row[2] = T.token[occ_slot[3 * j + 2]];
  }
}

// roles: bit 0 entity (subject, kept object), bit 1 predicate
__global__ void ingest_roles(int64_t n_stmt, Table T, const uint32_t* __restrict__ occ_slot,
                             const uint8_t* __restrict__ kept, unsigned int* __restrict__ roles32) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_stmt; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = T.token[occ_slot[3 * j]], p = T.token[occ_slot[3 * j + 1]];
    atomicOr(roles32 + s, 1u);
    atomicOr(roles32 + p, 2u);
    if (kept[j]) atomicOr(roles32 + T.token[occ_slot[3 * j + 2]], 1u);
  }
}

static inline unsigned gridn(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (unsigned)g;
}
static inline int64_t a256(int64_t b) { return (b + 255) & ~(int64_t)255; }

}  // namespace wv

extern "C" {

// Phase 1: lines.  n_lines (device int64) and line_end[n_lines] (int64; the last
// line may end at n_bytes without a terminator).
int64_t wv_ingest_lines_workspace_bytes(int64_t n_bytes) {
  using namespace wv;
  return a256(n_bytes) + a256((n_bytes + 1) * 8) + a256(scan_tiles(n_bytes + 1) * 8) + 256;
}

int wv_ingest_lines(const uint8_t* text, int64_t n_bytes, int64_t* line_end, int64_t* n_terms, void* ws,
                    int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(n_bytes >= 1, "empty input");
  WV_CHECK_ARG(ws_bytes >= wv_ingest_lines_workspace_bytes(n_bytes), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  uint8_t* term = (uint8_t*)w;
  w += a256(n_bytes);
  int64_t* pos = (int64_t*)w;
  w += a256((n_bytes + 1) * 8);
  int64_t* scan_ws = (int64_t*)w;
  ingest_line_ends<<<gridn(n_bytes, 256), 256, 0, st>>>(text, n_bytes, term);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<uint8_t, int64_t>(term, n_bytes, pos, n_terms, scan_ws, st)));
  ingest_line_bounds<<<gridn(n_bytes, 256), 256, 0, st>>>(term, pos, n_bytes, line_end);
  WV_LAUNCH_CHECK();
  return 0;
}

// Phase 2: parse + intern.  n_lines from phase 1 (terminators, +1 when the text
// does not end with one).  Outputs (device): status[n_lines], err[n_lines],
// err_at[n_lines], bad[2] (first parse-or-value error line, first value-error
// line; INT64_MAX when none), n_out[4] = {statements, edges, vocab size,
// collision flag}, edges (3 * n_lines int64 max), roles[vocab] (u32 bits:
// 1 entity, 2 predicate), tok_span[vocab] = (key start, key end, escaped flag).
int64_t wv_ingest_workspace_bytes(int64_t n_lines) {
  using namespace wv;
  int64_t cap = 1;
  while (cap < 6 * n_lines + 2) cap <<= 1;
  const int64_t occ = 3 * n_lines;
  return a256(n_lines * 3 * (int64_t)sizeof(Term)) * 2 + a256(n_lines * 8) * 2 + a256(n_lines) * 2 +
         a256(scan_tiles(n_lines + 1) * 8) + a256(cap * 8) * 2 + a256(cap * 8) + a256(occ * 4) * 3 +
         a256(radix_ws_bytes(occ, 32)) + a256(16) + 1024;
}

int64_t wv_ingest_records_workspace_bytes(int64_t n_bytes) {
  using namespace wv;
  const int64_t chunks = (n_bytes + kCsvChunk - 1) / kCsvChunk;
  return 2 * a256(n_bytes) + 2 * a256((n_bytes + 1) * 8) + 2 * a256(scan_tiles(n_bytes) * 8) + a256(chunks * 4) +
         a256(chunks) + 1024;
}

int wv_ingest_records(const uint8_t* text, int64_t n_bytes, int delim, int64_t* rec_end, int64_t* rec_line,
                      int64_t* n_records, int64_t* n_lines, void* ws, int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(n_bytes >= 1, "empty input");
  WV_CHECK_ARG(ws_bytes >= wv_ingest_records_workspace_bytes(n_bytes), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t chunks = (n_bytes + kCsvChunk - 1) / kCsvChunk;
  char* w = (char*)ws;
  uint8_t* rec = (uint8_t*)w;
  w += a256(n_bytes);
  uint8_t* phys = (uint8_t*)w;
  w += a256(n_bytes);
  int64_t* rpos = (int64_t*)w;
  w += a256((n_bytes + 1) * 8);
  int64_t* ppos = (int64_t*)w;
  w += a256((n_bytes + 1) * 8);
  int64_t* sws1 = (int64_t*)w;
  w += a256(scan_tiles(n_bytes) * 8);
  int64_t* sws2 = (int64_t*)w;
  w += a256(scan_tiles(n_bytes) * 8);
  uint8_t* maps = (uint8_t*)w;
  w += a256(chunks * 4);
  uint8_t* start = (uint8_t*)w;
  csv_chunk_maps<<<gridn(chunks * 4, 256), 256, 0, st>>>(text, n_bytes, (uint8_t)delim, chunks, maps);
  WV_LAUNCH_CHECK();
  csv_chunk_states<<<1, 1024, 0, st>>>(maps, chunks, start);
  WV_LAUNCH_CHECK();
  csv_terms<<<gridn(chunks, 128), 128, 0, st>>>(text, n_bytes, (uint8_t)delim, chunks, start, rec, phys);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<uint8_t, int64_t>(rec, n_bytes, rpos, n_records, sws1, st)));
  WV_CUDA((excl_scan<uint8_t, int64_t>(phys, n_bytes, ppos, n_lines, sws2, st)));
  csv_record_bounds<<<gridn(n_bytes, 256), 256, 0, st>>>(rec, rpos, ppos, n_bytes, rec_end, rec_line);
  WV_LAUNCH_CHECK();
  return 0;
}

int wv_ingest_parse(const uint8_t* text, int64_t n_bytes, const int64_t* line_end, int64_t n_lines, int mode,
                    const int64_t* line_no, uint64_t hash_seed,
                    int delim, int has_header, int include_literals, uint8_t* status, int32_t* err, int64_t* err_at,
                    int64_t* bad, int64_t* n_out, int64_t* edges, uint32_t* roles, int64_t* tok_span, void* ws,
                    int64_t ws_bytes, void* stream) {
  using namespace wv;
  WV_CHECK_ARG(n_lines >= 1, "empty input");
  WV_CHECK_ARG(mode >= 0 && mode <= 3, "bad mode");
  WV_CHECK_ARG(3 * n_lines < (int64_t)0xffffffffLL, "input too large for 32-bit positions");
  WV_CHECK_ARG(ws_bytes >= wv_ingest_workspace_bytes(n_lines), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t cap = 1;
  while (cap < 6 * n_lines + 2) cap <<= 1;
  const int64_t n_occ_max = 3 * n_lines;
  char* w = (char*)ws;
  auto take = [&](int64_t b) {
    char* p = w;
    w += a256(b);
    return p;
  };
  Term* terms = (Term*)take(n_lines * 3 * (int64_t)sizeof(Term));
  Term* occ = (Term*)take(n_lines * 3 * (int64_t)sizeof(Term));
  int64_t* stmt_of_line = (int64_t*)take(n_lines * 8);
  int64_t* edge_of = (int64_t*)take(n_lines * 8);
  uint8_t* okf = (uint8_t*)take(n_lines);
  uint8_t* kept = (uint8_t*)take(n_lines);
  int64_t* scan_ws = (int64_t*)take(scan_tiles(n_lines + 1) * 8);
  Table T;
  T.seed = hash_seed;
  T.key = (unsigned long long*)take(cap * 8);
  T.first = (unsigned long long*)take(cap * 8);
  T.token = (int64_t*)take(cap * 8);
  T.mask = (uint64_t)cap - 1;
  uint32_t* occ_slot = (uint32_t*)take(n_occ_max * 4);
  uint32_t* firsts = (uint32_t*)take(n_occ_max * 4);
  uint32_t* slots = (uint32_t*)take(n_occ_max * 4);
  void* rws = take(radix_ws_bytes(n_occ_max, 32));

  ingest_parse<<<gridn(n_lines, 128), 128, 0, st>>>(text, n_bytes, line_end, n_lines, mode, (uint8_t)delim,
                                                    has_header, line_no, status, err, err_at, terms);
  WV_LAUNCH_CHECK();
  const int64_t big[2] = {INT64_MAX, INT64_MAX};
  WV_CUDA(cudaMemcpyAsync(bad, big, 16, cudaMemcpyHostToDevice, st));
  ingest_first_bad<<<gridn(n_lines, 256), 256, 0, st>>>(status, n_lines, bad);
  WV_LAUNCH_CHECK();
  ingest_ok_flags<<<gridn(n_lines, 256), 256, 0, st>>>(status, n_lines, okf);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<uint8_t, int64_t>(okf, n_lines, stmt_of_line, n_out + 0, scan_ws, st)));
  ingest_statements<<<gridn(n_lines, 256), 256, 0, st>>>(status, stmt_of_line, n_lines, terms, occ);
  WV_LAUNCH_CHECK();
  // statement count is needed on the host to size the interning passes
  int64_t n_stmt = 0;
  WV_CUDA(cudaMemcpyAsync(&n_stmt, n_out + 0, 8, cudaMemcpyDeviceToHost, st));
  WV_CUDA(cudaStreamSynchronize(st));
  const int64_t n_occ = 3 * n_stmt;
  WV_CUDA(cudaMemsetAsync(T.key, 0, cap * 8, st));
  WV_CUDA(cudaMemsetAsync(T.first, 0xff, cap * 8, st));
  WV_CUDA(cudaMemsetAsync(n_out + 1, 0, 24, st));
  if (n_stmt == 0) return 0;
  ingest_insert<<<gridn(n_occ, 256), 256, 0, st>>>(text, occ, n_occ, include_literals, T, occ_slot);
  WV_LAUNCH_CHECK();
  ingest_verify<<<gridn(n_occ, 256), 256, 0, st>>>(text, occ, n_occ, include_literals, T, occ_slot,
                                                   (int*)(n_out + 3));
  WV_LAUNCH_CHECK();
  unsigned long long* n_unique = (unsigned long long*)(n_out + 2);
  ingest_collect<<<gridn(cap, 256), 256, 0, st>>>(T, cap, firsts, slots, n_unique);
  WV_LAUNCH_CHECK();
  int64_t nu = 0;
  WV_CUDA(cudaMemcpyAsync(&nu, n_out + 2, 8, cudaMemcpyDeviceToHost, st));
  WV_CUDA(cudaStreamSynchronize(st));
  // tokens = rank of the first position (distinct keys have distinct firsts)
  WV_CUDA(radix_sort_pairs(firsts, slots, nu, 32, rws, st));
  ingest_rank<<<gridn(nu, 256), 256, 0, st>>>(firsts, slots, n_unique, T, occ, tok_span);
  WV_LAUNCH_CHECK();
  ingest_kept_flags<<<gridn(n_stmt, 256), 256, 0, st>>>(occ, n_stmt, include_literals, kept);
  WV_LAUNCH_CHECK();
  WV_CUDA((excl_scan<uint8_t, int64_t>(kept, n_stmt, edge_of, n_out + 1, scan_ws, st)));
  WV_CUDA(cudaMemsetAsync(roles, 0, nu * 4, st));
  ingest_roles<<<gridn(n_stmt, 256), 256, 0, st>>>(n_stmt, T, occ_slot, kept, roles);
  WV_LAUNCH_CHECK();
  ingest_edges<<<gridn(n_stmt, 256), 256, 0, st>>>(n_stmt, T, occ_slot, kept, edge_of, edges);
  WV_LAUNCH_CHECK();
  return 0;
}

}  // extern "C"
