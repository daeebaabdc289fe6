// Batch assembler: text -> SPIR-V binary, bit-exact with the reference
// Assembler.assemble (asm.py:133-180) including the builder's serialization
// (builder.py:108-242) and the Encoder slot walk (ops.py:104-271).
//
// One warp per module (persistent warps take module tickets).  Phases:
//   A  copy the text into the warp's scratch + str.splitlines() boundaries,
//      word-parallel (asm.py:137)
//   B  tokenize_line, lane per line (asm.py:51-90); string escapes are undone
//      in place; numeric %ids are reserved (asm.py:148-153, builder.py:118-123)
//   C  leading header comments (asm.py:184-206), lane 0
//   D  symbolic result names -> ids in document order: a name table keyed by
//      the token bytes, the k-th new name gets the k-th unreserved positive
//      integer (select over the reservation bitmap; builder.py:108-116)
//   E  opname lookup, type-width and value-type scans (asm.py:215-245)
//   F  encode pass 1 (count), lane per line: Encoder.encode + coerce
//      (ops.py:120-271, asm.py:286-349) -> words per line + first error
//   G  the scope state machine (asm.py:249-284, builder.py:140-334), lane 0:
//      routing, SSA registry, functions/blocks -> placement of every line
//   H  serialization checks (builder.py:187-242) and layout: 11 section
//      buckets, then function declarations before definitions
//   I  encode pass 2 (write) at the final offsets + reference check
// Failing modules produce str(exc) of the exception the reference raises.
#include "skg_text.cuh"

namespace skg {

struct AsmTables {
  const uint32_t* info;       // 4 words / instruction: rslot | route<<8 | flags<<16, class str off, len
  const uint32_t* ophash; uint32_t ophash_cap;   // (hash, inst)
  const uint32_t* enhash; uint32_t enhash_cap;   // (hash, enum index, kind)
  const uint32_t* exhash; uint32_t exhash_cap;   // (hash, number, name off, name len)
  uint32_t storage_fn, op_label, op_fnend;
  uint32_t op_typeint, op_typefloat;   // instruction indices of those names (NONE32: absent)
};

constexpr uint32_t ROUTE_SCOPE = 11, ROUTE_VARIABLE = 12, ROUTE_KEYERROR = 13;
constexpr uint32_t AF_TERMINATOR = 1, AF_BLOCK_FORBIDDEN = 2, AF_CTXNUM = 4;
constexpr uint32_t MAX_ID = 0xFFFFFFFEu;

struct AsmArgs {
  Tables T;
  Uni U;
  AsmTables A;
  const uint8_t* text;
  const int64_t* mod_off;
  const int64_t* mod_len;
  uint32_t n_mod;
  uint32_t mod_stride;
  uint8_t* out;
  uint64_t out_cap;
  int64_t* out_span;
  int32_t* status;
  uint32_t* counters;        // [0] ticket, [2] overflow, [4..5] u64 cursor
  uint8_t* gscratch;
  uint64_t gslot_bytes;
  uint32_t default_version;   // major << 16 | minor
  const uint32_t* order;      // ticket -> module index (skg_sched.cuh)
  uint32_t group_warps;       // warps per phase-barrier group (divides the CTA's warps)
};

// token: off (text byte offset), lenf = len | TK_STR
constexpr uint32_t TK_STR = 0x80000000u, TK_ESC = 0x40000000u, TK_LEN = 0x3FFFFFFFu;

// line flags
enum : uint32_t {
  LF_TOKERR = 1, LF_RESULT = 2, LF_EMPTY = 4, LF_RESVERR = 8, LF_UNRES = 16, LF_VARFN = 32,
  LF_RESOLVE_ERR = 64, LF_PLACED = 128, LF_DROP = 256
};

// error codes (per line; E_* from the encoder, S_* from the state machine)
enum : uint32_t {
  E_OK = 0, E_NOINST, E_NEEDS_RESULT, E_NOT_PRODUCE, E_MISSING, E_EXTRA, E_STR_FOR, E_EXPECT_ID,
  E_INT_INVALID, E_INT_LIMIT, E_FLOAT_INVALID, E_NO_WIDTH, E_NEG, E_NO_ENUM_STR, E_NO_ENUM_INT,
  E_MASK_RANGE, E_LITSTR_INT, E_NUL, E_SURROGATE, E_WIDTH, E_FWIDTH, E_OVF_E, E_OVF_F, E_FIT,
  E_NO_EXT, E_NO_SPECOP, E_LIT_RANGE, E_INT_STRLIMIT, E_INTERNAL,
  S_LABEL_OUTSIDE = 64, S_LABEL_NORESULT, S_LABEL_USED, S_DUP, S_FUNC_BEFORE_END, S_OUTSIDE,
  S_PARAM_AFTER_BLOCK, S_MM_DUP, S_NEED_BLOCK, S_TERMINATED, S_VAR_FIRST, S_NOT_BLOCK, S_KEYERROR,
  S_LABEL_RESOLVE, S_VAR_NOTFN
};

// module-level outcome
enum : uint32_t {
  X_NONE = 0, X_VERSION, X_VERSION_LIMIT, X_VERSION_DEFAULT, X_RESERVE, X_OVERFLOW, X_ASSEMBLY, X_STRUCT_END,
  X_STRUCT_TERM, X_SERIAL, X_WC, X_INTERNAL
};

struct AsmMod {
  uint8_t* base;
  const uint8_t* txt; // the module text (input arena, read in place)
  uint8_t* esc;       // unescaped string tokens, at the same offsets as in txt
  uint32_t T;         // bytes
  uint32_t L;         // lines
  uint32_t* ls;       // line start
  uint32_t* le;       // line end
  uint32_t* lt0;      // first token
  uint32_t* lnt;      // token count
  uint32_t* lfl;      // flags
  uint32_t* ld;       // instruction index
  uint32_t* lec;      // error code
  uint32_t* lnw;      // operand words
  uint32_t* lrid;     // result / label id
  uint32_t* lgrp;     // placement group
  uint32_t* loff;     // offset within group, then absolute word offset
  uint32_t* lerr;     // 4 words / line: error details
  uint32_t* tok;      // 2 words / token
  uint32_t* tid;      // per token: resolved %id (0 = not an id token / not yet resolved)
  uint32_t* lwo;      // per line: offset of its encoded words in sw
  uint32_t* sw;       // encode pass 1 output words (line order)
  uint32_t* swr;      // bit per sw word: a referenced id (checked against the registry)
  uint32_t ntb;       // token slots
  uint32_t* nt;       // name table: 6 words / entry
  uint32_t ncap;
  uint32_t* rbm;      // reservation bitmap (RB bits)
  uint32_t* zpre;     // unreserved ids in [0, 32 w)
  uint32_t* reg;      // registry bitmap
  uint32_t* lab;      // label bitmap
  uint32_t RB;
  uint32_t* fn;       // functions: 4 words (result id, flags, size, base)
  uint32_t* blk;      // blocks: 3 words (fn, label, terminated)
  uint32_t* big;      // big-id lists: [0] count reg, [1] count lab, then pairs
  uint32_t big_cap;
  uint32_t* misc;     // 64 words of counters
  uint8_t* sbase;     // the warp's scratch slot (bump allocated; lane 0 may grow the name table)
  uint64_t sused, scap;
};

// misc slots
enum : uint32_t {
  MS_BIGMAX_LO = 0, MS_BIGMAX_HI, MS_NPCT, MS_RESV_LINE, MS_NSYM, MS_NFN, MS_NBLK, MS_BUCKET0 = 8,
  MS_X = 24, MS_XA, MS_XB, MS_XC, MS_NEWCOUNT, MS_GEN, MS_SCHEMA, MS_MAJOR, MS_MINOR, MS_GENSET,
  MS_HDR_LINE_V, MS_HDR_LINE_G, MS_HDR_LINE_S, MS_TOTAL, MS_NDIAG, MS_OVF_LINE, MS_SER_LINE,
  MS_WC_LINE, MS_COUNTER, MS_NTCOUNT, MS_V0 = 48
};

__device__ __forceinline__ uint32_t lane_id_a() { return threadIdx.x & 31; }
constexpr unsigned FULLM = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t wincl(uint32_t v) {
  const uint32_t l = lane_id_a();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t = __shfl_up_sync(FULLM, v, d);
    if (l >= (uint32_t)d) v += t;
  }
  return v;
}
__device__ __forceinline__ uint32_t wsum(uint32_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULLM, v, d);
  return v;
}
__device__ __forceinline__ uint32_t wmax(uint32_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = max(v, __shfl_xor_sync(FULLM, v, d));
  return v;
}
__device__ __forceinline__ uint32_t wmin(uint32_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = min(v, __shfl_xor_sync(FULLM, v, d));
  return v;
}

// one out-of-line copy each: these run at many call sites (instruction-cache footprint)
// byte loops unrolled by 4 so the four loads are in flight together (latency bound)
__device__ __noinline__ uint32_t fnv(const uint8_t* p, uint32_t n, uint32_t h = 2166136261u) {
  uint32_t i = 0;
#pragma unroll 1
  for (; i + 4 <= n; i += 4) {
    const uint32_t b0 = p[i], b1 = p[i + 1], b2 = p[i + 2], b3 = p[i + 3];
    h = (h ^ b0) * 16777619u; h = (h ^ b1) * 16777619u; h = (h ^ b2) * 16777619u; h = (h ^ b3) * 16777619u;
  }
#pragma unroll 1
  for (; i < n; ++i) h = (h ^ p[i]) * 16777619u;
  return h;
}

__device__ __noinline__ bool bytes_eq(const uint8_t* a, const uint8_t* b, uint32_t n) {
  uint32_t i = 0;
#pragma unroll 1
  for (; i + 4 <= n; i += 4) {
    const uint32_t x = a[i] | (a[i + 1] << 8) | (a[i + 2] << 16) | ((uint32_t)a[i + 3] << 24);
    const uint32_t y = b[i] | (b[i + 1] << 8) | (b[i + 2] << 16) | ((uint32_t)b[i + 3] << 24);
    if (x != y) return false;
  }
#pragma unroll 1
  for (; i < n; ++i) if (a[i] != b[i]) return false;
  return true;
}

__device__ __noinline__ bool bytes_eq_z(const uint8_t* a, uint32_t n, const char* z) {
  uint32_t i = 0;
#pragma unroll 1
  for (; i < n; ++i) if (!z[i] || (uint8_t)z[i] != a[i]) return false;
  return z[i] == 0;
}

struct Tok {
  const uint8_t* p;
  uint32_t n;
  bool str;
  uint32_t raw;   // raw byte offset of the token start (quote for strings)
};

__device__ __forceinline__ Tok tok_at(const AsmMod& m, uint32_t t) {
  const uint32_t off = m.tok[2 * t], lf = m.tok[2 * t + 1];
  Tok k;
  k.p = ((lf & TK_ESC) ? m.esc : m.txt) + off;
  k.n = lf & TK_LEN;
  k.str = (lf & TK_STR) != 0;
  k.raw = off - (k.str ? 1 : 0);
  return k;
}

// str.isdigit() of p[0..n) (non-empty)
__device__ inline bool py_isdigit(const uint8_t* p, uint32_t n, const Uni& U) {
  if (n == 0) return false;
  for (uint32_t i = 0; i < n;) {
    if (p[i] < 0x80) { if (p[i] < '0' || p[i] > '9') return false; ++i; continue; }
    uint32_t len;
    const uint32_t c = utf8_cp(p, n, i, len);
    if (!U.is_digit(c)) return false;
    i += len;
  }
  return true;
}

// Fast path of body.isdigit() + int(body): 1-9 ASCII digits (no sign, no
// underscores) -> value; false means "use the general path".
__device__ __forceinline__ bool ascii_dec9(const uint8_t* p, uint32_t n, uint32_t& v) {
  if (n == 0 || n > 9) return false;
  uint32_t x = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t d = (uint32_t)p[i] - '0';
    if (d > 9) return false;
    x = x * 10 + d;
  }
  v = x;
  return true;
}

// re.match(r"[+-]?(0[xX][0-9a-fA-F]+|\d+)$", text)  (asm.py:31)
__device__ inline bool int_token(const uint8_t* p, uint32_t n, const Uni& U) {
  uint32_t i = 0;
  if (i < n && (p[i] == '+' || p[i] == '-')) ++i;
  if (i + 2 < n + 0 && p[i] == '0' && (p[i + 1] == 'x' || p[i + 1] == 'X')) {
    uint32_t j = i + 2;
    bool hex = j < n;
    for (uint32_t k = j; k < n; ++k) {
      const uint8_t c = p[k];
      if (!((c >= '0' && c <= '9') || (c >= 'a' && c <= 'f') || (c >= 'A' && c <= 'F'))) { hex = false; break; }
    }
    if (hex) return true;
  }
  if (i >= n) return false;
  while (i < n) {
    uint32_t len = 1, c = p[i];
    if (c >= 0x80) c = utf8_cp(p, n, i, len);
    if (U.decimal(c) < 0) return false;
    i += len;
  }
  return true;
}

// Python str.strip() bounds (isspace)
__device__ inline void py_strip(const uint8_t* p, uint32_t n, const Uni& U, uint32_t& s, uint32_t& e) {
  s = 0; e = n;
  while (s < e) {
    uint32_t len, c = utf8_cp(p, n, s, len);
    if (!U.is_space(c)) break;
    s += len;
  }
  while (e > s) {
    uint32_t k = e - 1;
    while (k > s && (p[k] & 0xC0) == 0x80) --k;
    uint32_t len, c = utf8_cp(p, n, k, len);
    if (!U.is_space(c)) break;
    e = k;
  }
}

// -- name table -------------------------------------------------------------------
// entry: [0] key token (EMPTY), [1] hash, [2] first symbolic line (min), [3] id,
//        [4] last OpTypeInt/Float line + 1 (max), [5] last value-type line + 1 (max)
constexpr uint32_t NT_W = 6;
constexpr uint32_t EMPTYK = 0xFFFFFFFFu;

__device__ inline uint32_t nt_find(const AsmMod& m, const uint8_t* p, uint32_t n) {
  const uint32_t h = fnv(p, n);
  uint32_t s = (h * 0x9E3779B1u) & (m.ncap - 1);
  for (uint32_t probe = 0; probe < m.ncap; ++probe) {
    const uint32_t* e = m.nt + NT_W * s;
    const uint32_t k = e[0];
    if (k == EMPTYK) return NONE32;
    if (e[1] == h) {
      const Tok t = tok_at(m, k);
      if (t.n == n && bytes_eq(t.p, p, n)) return s;
    }
    s = (s + 1) & (m.ncap - 1);
  }
  return NONE32;
}

// insert (concurrent-safe); returns the entry slot
__device__ inline uint32_t nt_insert(const AsmMod& m, uint32_t t) {
  const Tok me = tok_at(m, t);
  const uint32_t h = fnv(me.p, me.n);
  uint32_t s = (h * 0x9E3779B1u) & (m.ncap - 1);
  for (uint32_t probe = 0; probe < m.ncap; ++probe) {
    uint32_t* e = m.nt + NT_W * s;
    uint32_t k = *(volatile uint32_t*)e;
    if (k == EMPTYK) {
      // inserting lanes compare bytes, not hashes; lookups run after the insert phase
      k = atomicCAS(e, EMPTYK, t);
      if (k == EMPTYK) { e[1] = h; return s; }
    }
    // the entry's hash, once its inserter has written it, rules out most other keys
    // without comparing bytes (0: not written yet -> compare)
    const uint32_t eh = *(volatile uint32_t*)(e + 1);
    if (eh == 0 || eh == h) {
      const Tok o = tok_at(m, k);
      if (o.n == me.n && bytes_eq(o.p, me.p, me.n)) return s;
    }
    s = (s + 1) & (m.ncap - 1);
  }
  return NONE32;
}

// lane 0: grow the name table 4x (re-hash) when unresolved operand names fill it
__device__ __noinline__ bool nt_grow(AsmMod& m) {
  const uint32_t ncap = m.ncap * 4;
  const uint64_t bytes = 4ull * NT_W * ncap;
  if (m.sused + bytes > m.scap) return false;
  uint32_t* nt = reinterpret_cast<uint32_t*>(m.sbase + m.sused);
  m.sused += (bytes + 15) & ~15ull;
  for (uint32_t k = 0; k < ncap; ++k) {
    uint32_t* e = nt + NT_W * k;
    e[0] = EMPTYK; e[1] = 0; e[2] = NONE32; e[3] = 0; e[4] = 0; e[5] = 0;
  }
  for (uint32_t k = 0; k < m.ncap; ++k) {
    const uint32_t* o = m.nt + NT_W * k;
    if (o[0] == EMPTYK) continue;
    uint32_t sl = (o[1] * 0x9E3779B1u) & (ncap - 1);
    while (nt[NT_W * sl] != EMPTYK) sl = (sl + 1) & (ncap - 1);
    for (uint32_t q = 0; q < NT_W; ++q) nt[NT_W * sl + q] = o[q];
  }
  m.nt = nt;
  m.ncap = ncap;
  return true;
}

// -- id sets ------------------------------------------------------------------------
__device__ inline bool bit_get(const uint32_t* bm, uint32_t v) { return (bm[v >> 5] >> (v & 31)) & 1; }
__device__ inline void bit_set(uint32_t* bm, uint32_t v) { bm[v >> 5] |= 1u << (v & 31); }

// registry / label sets with a small overflow list for ids >= RB (lane 0 only)
__device__ inline bool idset_has(const AsmMod& m, const uint32_t* bm, uint32_t which, uint32_t v) {
  if (v < m.RB) return bit_get(bm, v);
  const uint32_t n = m.big[which];
  const uint32_t* lst = m.big + 2 + which * m.big_cap;
  for (uint32_t i = 0; i < n; ++i) if (lst[i] == v) return true;
  return false;
}
__device__ inline bool idset_add(const AsmMod& m, uint32_t* bm, uint32_t which, uint32_t v) {
  if (v < m.RB) { bit_set(bm, v); return true; }
  const uint32_t n = m.big[which];
  if (n >= m.big_cap) return false;
  m.big[2 + which * m.big_cap + n] = v;
  m.big[which] = n + 1;
  return true;
}

// k-th (1-based) positive integer that is not reserved
__device__ inline uint32_t select_unreserved(const AsmMod& m, uint32_t k) {
  const uint32_t nw = m.RB / 32;
  uint32_t lo = 0, hi = nw;   // largest w with zpre[w] < k
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (m.zpre[mid] < k) lo = mid; else hi = mid;
  }
  const uint32_t r = k - m.zpre[lo];   // r-th zero of word lo
  uint32_t z = ~m.rbm[lo];
  for (uint32_t q = 1; q < r; ++q) z &= z - 1;
  return lo * 32 + (__ffs(z) - 1);
}

// ============================================================================
// Phase A: copy + line split.  Line separators of str.splitlines():
// \n \r \r\n \v \f \x1c \x1d \x1e \x85    .
__device__ inline uint32_t sep_len_at(const uint8_t* t, uint32_t T, uint32_t i) {
  const uint8_t b = t[i];
  if (b == '\n') return (i > 0 && t[i - 1] == '\r') ? 0 : 1;
  if (b == '\r') return (i + 1 < T && t[i + 1] == '\n') ? 2 : 1;
  if (b == 0x0B || b == 0x0C || b == 0x1C || b == 0x1D || b == 0x1E) return 1;
  if (b == 0xC2) return (i + 1 < T && t[i + 1] == 0x85) ? 2 : 0;
  if (b == 0xE2) return (i + 2 < T && t[i + 1] == 0x80 && (t[i + 2] == 0xA8 || t[i + 2] == 0xA9)) ? 3 : 0;
  return 0;
}

__device__ __forceinline__ bool word_maybe_sep(uint32_t w) {
  // any byte < 0x20 or any of 0xC2 / 0xE2
  const uint32_t lt = (w - 0x20202020u) & ~w & 0x80808080u;
  const uint32_t x2 = w ^ 0xC2C2C2C2u, x3 = w ^ 0xE2E2E2E2u;
  const uint32_t z2 = (x2 - 0x01010101u) & ~x2 & 0x80808080u;
  const uint32_t z3 = (x3 - 0x01010101u) & ~x3 & 0x80808080u;
  return (lt | z2 | z3) != 0;
}

// SWAR byte masks (0x80 in every byte of w that matches; exact, no carries)
__device__ __forceinline__ uint32_t eq_bytes(uint32_t w, uint32_t c) {
  const uint32_t t = w ^ (c * 0x01010101u);
  return ~(((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t) & 0x80808080u;
}
__device__ __forceinline__ uint32_t lt21_bytes(uint32_t w) {   // byte < 0x21
  return ~(((w & 0x7F7F7F7Fu) + 0x5F5F5F5Fu) | w) & 0x80808080u;
}

// returns L; fills ls/le (capacity cap) and lt0 = per-line token-slot bases.
// Slot bound: every token of a line starts at a "candidate" byte -- a byte
// other than ' ' whose previous byte is < 0x21 or >= 0x80 (tokenizer
// whitespace, any line separator's last byte, text start), or the byte after
// a '"' -- so counting those bytes plus one per '"' over-approximates the
// tokens.  lt0[k+1] = candidates before line k's separator; line k's slots are
// lt0[k+1] - lt0[k] (tokenize_line zero-fills the unused ones).  The text is
// read in place (the later phases read it line by line from L1/L2).
__device__ __noinline__ uint32_t split_lines(AsmMod& m, const uint8_t* src, uint32_t cap, uint32_t* lt0,
                                             uint32_t& ncand) {
  const uint32_t lane = lane_id_a();
  const uint32_t T = m.T;
  uint32_t nsep = 0, ccarry = 0, prev_last = 0;   // prev_last: byte before this chunk (0 = text start)
  const uint32_t nw = (T + 3) / 4;
  // text word w (bytes 4w..4w+3; bytes past T are masked by `valid` below): aligned
  // 32-bit loads, funnel-shifted together when the text does not start on a word
  // (texts sit at arbitrary byte offsets of the disassembler's arena); only words
  // holding text bytes are read.  Each iteration's word is loaded one iteration ahead
  // (the scan's carries make the iterations dependent; the loads need not be).
  const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(m.txt) & 3);
  const uint32_t* A = reinterpret_cast<const uint32_t*>(m.txt - sh);
  const uint32_t nA = (sh + T + 3) / 4;
  auto load_word = [&](uint32_t w) -> uint32_t {
    if (w >= nw) return 0u;
    const uint32_t lo = __ldg(A + w);
    if (sh == 0) return lo;
    const uint32_t hi = w + 1 < nA ? __ldg(A + w + 1) : 0u;
    return __funnelshift_r(lo, hi, 8 * sh);
  };
  uint32_t next_word = load_word(lane);
  for (uint32_t base = 0; base < nw; base += 32) {
    const uint32_t w = base + lane;
    uint32_t cnt = 0;
    uint32_t pos[4], len[4], cb[4];
    const uint32_t word = next_word;
    next_word = load_word(w + 32);
    uint32_t pw = __shfl_up_sync(FULLM, word, 1);
    if (lane == 0) pw = prev_last << 24;
    const uint32_t prev = (word << 8) | (pw >> 24);          // previous byte of every byte
    const uint32_t valid = w >= nw ? 0u : (4 * w + 4 <= T ? 0x80808080u : (0x80808080u >> (8 * (4 * w + 4 - T))));
    const uint32_t cm = ~eq_bytes(word, ' ') & (lt21_bytes(prev) | (prev & 0x80808080u)) & valid;
    const uint32_t qm = eq_bytes(word, '"') & valid;
    const uint32_t nc = __popc(cm) + __popc(qm);
    // common case: the word's only separator candidates are bare '\n' bytes
    const uint32_t nl = eq_bytes(word, '\n') & valid;
    const uint32_t rest = (~(((word & 0x7F7F7F7Fu) + 0x60606060u) | word) & 0x80808080u & ~nl) |
                          eq_bytes(word, 0xC2) | eq_bytes(word, 0xE2) | (eq_bytes(prev, '\r') & nl);
    if (!(rest & valid)) {
      for (uint32_t bits = nl; bits; bits &= bits - 1) {
        const uint32_t b = (__ffs(bits) - 1) >> 3;
        const uint32_t below = b ? (0xFFFFFFFFu >> (32 - 8 * b)) : 0u;
        pos[cnt] = 4 * w + b; len[cnt] = 1; cb[cnt] = __popc(cm & below) + __popc(qm & below); ++cnt;
      }
    } else if (w < nw && word_maybe_sep(word)) {
      for (uint32_t b = 0; b < 4; ++b) {
        const uint32_t i = 4 * w + b;
        if (i >= T) break;
        const uint32_t sl = sep_len_at(m.txt, T, i);
        if (sl) {
          const uint32_t below = b ? (0xFFFFFFFFu >> (32 - 8 * b)) : 0u;
          pos[cnt] = i; len[cnt] = sl; cb[cnt] = __popc(cm & below) + __popc(qm & below); ++cnt;
        }
      }
    }
    const uint32_t both = wincl((cnt << 16) | nc);   // one scan for both counts (each < 2^16 per step)
    const uint32_t incl = both >> 16, cincl = both & 0xFFFF;
    const uint32_t c0 = ccarry + cincl - nc;
    uint32_t k = nsep + incl - cnt;
    for (uint32_t q = 0; q < cnt; ++q, ++k) {
      if (k < cap) { m.le[k] = pos[q]; m.ls[k + 1] = pos[q] + len[q]; lt0[k + 1] = c0 + cb[q]; }
    }
    nsep += __shfl_sync(FULLM, incl, 31);
    ccarry += __shfl_sync(FULLM, cincl, 31);
    prev_last = __shfl_sync(FULLM, word >> 24, 31);
  }
  __syncwarp();
  if (lane == 0) { m.ls[0] = 0; lt0[0] = 0; }
  // lines: one per separator, plus a final unterminated one if non-empty
  uint32_t L = nsep;
  const uint32_t last_start = nsep ? (nsep < cap ? m.ls[nsep] : T) : 0;
  if (last_start < T) {
    if (lane == 0 && nsep < cap) m.le[nsep] = T;
    ++L;
  }
  ncand = ccarry;
  __syncwarp();
  return L;
}

// ============================================================================
// Phase B: tokenize (asm.py:51-90), lane per line, into the line's token
// slots (bound from split_lines); strings are unescaped into m.esc.

struct AsmCtx {   // one copy per CTA in shared memory (not a per-thread local copy)
  Tables T;
  Uni U;
  AsmTables A;
};

__device__ __forceinline__ bool str_stop(uint32_t d) { return d == '"' || d == '\\'; }

__device__ __noinline__ void tokenize_line(AsmMod& m, const AsmCtx& X, uint32_t li, uint32_t tb,
                                           uint32_t cap, uint32_t& npct) {
  const uint8_t* t = m.txt;
  const uint32_t s0 = m.ls[li], e0 = m.le[li];
#ifndef SKG_EXP_NO_PREFETCH
  prefetch_l1(t + s0);
  if (e0 > s0 + 64) prefetch_l1(t + e0 - 1);
#endif
  uint32_t nt = 0;
  uint32_t fl = 0;
  uint32_t i = s0;
  // indentation: whole aligned 4-byte words of spaces at a time
  while (i < e0 && (reinterpret_cast<uintptr_t>(t + i) & 3) && t[i] == ' ') ++i;
  while (i + 4 <= e0 && (reinterpret_cast<uintptr_t>(t + i) & 3) == 0 &&
         *reinterpret_cast<const uint32_t*>(t + i) == 0x20202020u) i += 4;
  while (i < e0) {
    const uint32_t c = __ldg(t + i);
    if (c <= ' ' && ((c == ' ' ? 1u : 0x2600u >> c) & 1)) { ++i; continue; }   // ' ' \t \r \n
    if (c == ';') break;
    const uint32_t start = i;
    if (c == '"') {
      ++i;
      // up to the first '"' or '\\' four bytes per step (no escape so far: w == i)
      while (i + 4 <= e0) {
        const uint32_t d0 = __ldg(t + i), d1 = __ldg(t + i + 1), d2 = __ldg(t + i + 2), d3 = __ldg(t + i + 3);
        const uint32_t k = str_stop(d0) ? 0 : str_stop(d1) ? 1 : str_stop(d2) ? 2 : str_stop(d3) ? 3 : 4;
        i += k;
        if (k < 4) break;
      }
      uint32_t w = i;
      bool esc = false;
      while (i < e0 && t[i] != '"') {
        if (t[i] == '\\' && i + 1 < e0) {
          if (!esc) {   // first escape: the unescaped copy starts with the bytes so far
            for (uint32_t q = start + 1; q < w; ++q) m.esc[q] = t[q];
            esc = true;
          }
          ++i;
        }
        if (esc) m.esc[w] = t[i];
        ++w; ++i;
      }
      if (i >= e0) {
        fl |= LF_TOKERR;
        m.lerr[4 * li] = start;   // raw position of the quote
        nt = 0;
        break;
      }
      ++i;
      if (nt < cap) {
        m.tok[2 * (tb + nt)] = start + 1;
        m.tok[2 * (tb + nt) + 1] = (w - start - 1) | TK_STR | (esc ? TK_ESC : 0);
      }
      ++nt;
      continue;
    }
    // token end: the first \t \n \r ' ' '"' ';' -- four independent loads per step
    auto delim = [](uint32_t d) -> bool {   // bit d of 0x0800000500002600 (d < 64), in 32-bit halves
      const uint32_t h = d < 32 ? 0x00002600u : (d < 64 ? 0x08000005u : 0u);
      return __funnelshift_r(h, h, d) & 1;
    };
    while (i + 4 <= e0) {
      const uint32_t d0 = __ldg(t + i), d1 = __ldg(t + i + 1), d2 = __ldg(t + i + 2), d3 = __ldg(t + i + 3);
      const uint32_t k = delim(d0) ? 0 : delim(d1) ? 1 : delim(d2) ? 2 : delim(d3) ? 3 : 4;
      i += k;
      if (k < 4) goto token_end;
    }
    while (i < e0 && !delim(__ldg(t + i))) ++i;
  token_end:
    if (nt < cap) {   // cap = candidate bound of this line (split_lines)
      m.tok[2 * (tb + nt)] = start;
      m.tok[2 * (tb + nt) + 1] = i - start;
    }
    ++nt;
  }
  for (uint32_t q = min(nt, cap); q < cap; ++q) { m.tok[2 * (tb + q)] = 0; m.tok[2 * (tb + q) + 1] = 0; }
  if (!(fl & LF_TOKERR) && nt == 0) fl |= LF_EMPTY;
  if (!(fl & (LF_TOKERR | LF_EMPTY)) && nt >= 3) {
    const Tok a = tok_at(m, tb), b = tok_at(m, tb + 1);
    if (a.n >= 1 && a.p[0] == '%' && b.n == 1 && b.p[0] == '=') fl |= LF_RESULT;
  }
  m.lt0[li] = tb;
  m.lnt[li] = (fl & LF_TOKERR) ? 0 : nt;
  m.lfl[li] = fl;
  // reservations: result + non-string operand tokens starting with '%' (asm.py:148-153)
  uint32_t bad = NONE32;
  if (!(fl & (LF_TOKERR | LF_EMPTY))) {
    const uint32_t first_op = (fl & LF_RESULT) ? 3 : 1;
    for (uint32_t k = 0; k < nt; ++k) {
      const bool is_res = (fl & LF_RESULT) && k == 0;
      if (!is_res && k < first_op) continue;
      const Tok tk = tok_at(m, tb + k);
      if (!(tk.n >= 1 && tk.p[0] == '%')) continue;
      if (!is_res && tk.str) continue;
      ++npct;
      uint32_t id;
      if (!ascii_dec9(tk.p + 1, tk.n - 1, id)) {
        if (!py_isdigit(tk.p + 1, tk.n - 1, X.U)) continue;
        const IntVal v = parse_int(tk.p + 1, tk.n - 1, 10, X.U);
        if (v.status != INT_OK || v.big || v.mag == 0 || v.mag > MAX_ID) { bad = k; break; }
        id = (uint32_t)v.mag;
      }
      if (id == 0) { bad = k; break; }
      if (id < m.RB) atomicOr(&m.rbm[id >> 5], 1u << (id & 31));
      else atomicMax(&m.misc[MS_BIGMAX_LO], id);
    }
  }
  if (bad != NONE32) {
    m.lfl[li] = fl | LF_RESVERR;
    m.lerr[4 * li + 1] = tb + bad;
  }
}

// ============================================================================
// literal info (asm.py:351-362): width / signed / floating of the governing type
struct LitInfo {
  bool ok;
  uint32_t wtok;     // token holding the width (int(text, 0))
  bool sgn, flt;
  IntVal w;
};

__device__ inline uint32_t op_tok(const AsmMod& m, uint32_t li, uint32_t k) {
  // k-th operand token of line li (after result '=' opname), NONE32 if absent
  const uint32_t first = (m.lfl[li] & LF_RESULT) ? 3 : 1;
  return first + k < m.lnt[li] ? m.lt0[li] + first + k : NONE32;
}

__device__ inline LitInfo width_of_entry(const AsmMod& m, const AsmCtx& X, uint32_t ent) {
  LitInfo r{};
  r.ok = false;
  if (ent == NONE32) return r;
  const uint32_t wl = m.nt[NT_W * ent + 4];
  if (wl == 0) return r;
  const uint32_t li = wl - 1;
  const uint32_t t0 = op_tok(m, li, 0);
  const Tok w = tok_at(m, t0);
  const uint32_t opn = m.lt0[li] + 2;   // opname token (result line)
  const Tok on = tok_at(m, opn);
  r.ok = true;
  r.wtok = t0;
  r.w = parse_int(w.p, w.n, 0, X.U);
  if (bytes_eq_z(on.p, on.n, "OpTypeInt")) {
    const Tok s = tok_at(m, op_tok(m, li, 1));
    const IntVal sv = parse_int(s.p, s.n, 0, X.U);
    r.sgn = !sv.big && !sv.neg && sv.mag == 1;
    r.flt = false;
  } else {
    r.sgn = false;
    r.flt = true;
  }
  return r;
}

// ============================================================================
// The encoder (ops.py:104-271 with the assembler's coerce, asm.py:286-332)
enum : uint32_t { M_COUNT = 0, M_WRITE = 1, M_RESOLVE = 2 };

struct EncOut {
  uint32_t nw;
  uint32_t ecode, etok, eaux, eaux2, eaux3;
  uint32_t result_id;
  uint32_t word2;         // third operand word (OpVariable storage class)
  bool unres;
  uint32_t bad_ref;       // M_WRITE: first referenced id not in the registry
};

struct EncCtx {
  const AsmMod& m;
  const AsmCtx& X;
  uint32_t li, d, mode;
  uint32_t* out;          // M_WRITE: operand words
  uint32_t ops0, nops;    // operand tokens
  uint32_t rtok, ridx;    // result token, insertion index (NONE32 = none)
  uint32_t nitems, pos;
  EncOut r;
  LitInfo info;
  bool is_switch;
  uint32_t* rbits;        // pass 1: bit per scratch word, set for referenced ids
  uint32_t rbase;         // bit index of operand word 0
};

__device__ __forceinline__ Tok tok_of(const EncCtx& c, uint32_t t) {
  const uint32_t off = c.m.tok[2 * t], lf = c.m.tok[2 * t + 1];
  Tok k;
  k.p = ((lf & TK_ESC) ? c.m.esc : c.m.txt) + off;
  k.n = lf & TK_LEN;
  k.str = (lf & TK_STR) != 0;
  k.raw = off - (k.str ? 1 : 0);
  return k;
}

__device__ __forceinline__ uint32_t enc_item(const EncCtx& c, uint32_t k) {
  if (c.ridx == NONE32) return c.ops0 + k;
  if (k < c.ridx) return c.ops0 + k;
  if (k == c.ridx) return c.rtok;
  return c.ops0 + k - 1;
}

__device__ __forceinline__ void emit_word(EncCtx& c, uint32_t w) {
  if (c.r.nw == 2) c.r.word2 = w;
  if (c.out) c.out[c.r.nw] = w;
  ++c.r.nw;
}

__device__ inline bool enc_fail(EncCtx& c, uint32_t code, uint32_t tok = 0, uint32_t a = 0, uint32_t b = 0,
                                uint32_t c3 = 0) {
  c.r.ecode = code; c.r.etok = tok; c.r.eaux = a; c.r.eaux2 = b; c.r.eaux3 = c3;
  return false;
}

// enumerant of kind k by name
__device__ inline uint32_t enum_by_name(const AsmCtx& X, uint32_t k, const uint8_t* p, uint32_t n) {
  const uint32_t h = fnv(p, n) ^ (k * 0x9E3779B1u);
  const uint32_t cap = X.A.enhash_cap;
  uint32_t s = h & (cap - 1);
  for (uint32_t probe = 0; probe < cap; ++probe) {
    const uint32_t* e = X.A.enhash + 3 * s;
    const uint32_t eh = __ldg(e), ei = __ldg(e + 1), ek = __ldg(e + 2);
    if (eh == 0 && ei == 0 && ek == 0) return NONE32;
    if (eh == h && ek == k && X.T.ename_len(ei) == n && bytes_eq(X.T.str + X.T.ename_off(ei), p, n)) return ei;
    s = (s + 1) & (cap - 1);
  }
  return NONE32;
}

__device__ inline uint32_t inst_by_name(const AsmCtx& X, const uint8_t* p, uint32_t n, const uint8_t* pre = nullptr,
                                        uint32_t npre = 0) {
  uint32_t h = 2166136261u;
  if (pre) h = fnv(pre, npre, h);
  h = fnv(p, n, h);
  const uint32_t cap = X.A.ophash_cap;
  uint32_t s = h & (cap - 1);
  for (uint32_t probe = 0; probe < cap; ++probe) {
    const uint32_t* e = X.A.ophash + 2 * s;
    const uint32_t eh = __ldg(e), ei = __ldg(e + 1);
    if (eh == 0 && ei == 0) return NONE32;
    if (eh == h && X.T.iname_len(ei) == n + npre) {
      const uint8_t* nm = X.T.str + X.T.iname_off(ei);
      if ((!pre || bytes_eq(nm, pre, npre)) && bytes_eq(nm + npre, p, n)) return ei;
    }
    s = (s + 1) & (cap - 1);
  }
  return NONE32;
}

__device__ inline bool ext_by_name(const AsmCtx& X, const uint8_t* p, uint32_t n, uint32_t& num) {
  const uint32_t h = fnv(p, n);
  const uint32_t cap = X.A.exhash_cap;
  uint32_t s = h & (cap - 1);
  for (uint32_t probe = 0; probe < cap; ++probe) {
    const uint32_t* e = X.A.exhash + 4 * s;
    const uint32_t eh = __ldg(e), en = __ldg(e + 1), eo = __ldg(e + 2), el = __ldg(e + 3);
    if (eh == 0 && en == 0 && eo == 0 && el == 0) return false;
    if (eh == h && el == n && bytes_eq(X.T.str + eo, p, n)) { num = en; return true; }
    s = (s + 1) & (cap - 1);
  }
  return false;
}

// id of an %name token for coerce (asm.py:106-120); false on error
__device__ inline bool enc_id(EncCtx& c, uint32_t t, const Tok& k, uint32_t& id) {
  if (c.mode != M_RESOLVE) {   // resolved once per token after the result names are bound
    const uint32_t cached = c.m.tid[t];
    if (cached) { id = cached; return true; }
  }
  if (!(k.n >= 2 && k.p[0] == '%')) return enc_fail(c, E_EXPECT_ID, t);
  if (ascii_dec9(k.p + 1, k.n - 1, id)) return true;
  if (py_isdigit(k.p + 1, k.n - 1, c.X.U)) {
    const IntVal v = parse_int(k.p + 1, k.n - 1, 10, c.X.U);
    id = (uint32_t)v.mag;   // validated by the reservation pass
    return true;
  }
  const uint32_t e = nt_find(c.m, k.p, k.n);
  if (e != NONE32 && c.m.nt[NT_W * e + 3] != 0) { id = c.m.nt[NT_W * e + 3]; return true; }
  if (c.mode == M_RESOLVE) {
    AsmMod& mm = const_cast<AsmMod&>(c.m);
    if (4 * (mm.misc[MS_NTCOUNT] + 1) > 3 * mm.ncap && !nt_grow(mm)) return enc_fail(c, E_INTERNAL, t);
    ++mm.misc[MS_NTCOUNT];
    const uint32_t s = nt_insert(c.m, t);
    uint32_t* ent = c.m.nt + NT_W * s;
    if (ent[3] == 0) {
      const uint32_t kk = ++c.m.misc[MS_NEWCOUNT];
      ent[3] = select_unreserved(c.m, kk);
    }
    id = ent[3];
    return true;
  }
  c.r.unres = true;
  id = 0;
  return true;
}

// encode_string (codec.py:104-114) of a string token
__device__ inline bool enc_string(EncCtx& c, uint32_t t, const Tok& k) {
  // text.encode("utf-8"): surrogates raise UnicodeEncodeError, then embedded NULs
  bool nul = false;
  uint32_t cpi = 0;
  for (uint32_t i = 0; i < k.n;) {
    const uint8_t b = k.p[i];
    nul |= b == 0;
    if (b == 0xED && i + 1 < k.n && k.p[i + 1] >= 0xA0) {
      uint32_t j = i, cpe = cpi;   // surrogate run [cpi, cpe)
      while (j + 3 <= k.n && k.p[j] == 0xED && k.p[j + 1] >= 0xA0) { j += 3; ++cpe; }
      return enc_fail(c, E_SURROGATE, t, cpi, cpe);
    }
    i += b < 0x80 ? 1 : b < 0xE0 ? 2 : b < 0xF0 ? 3 : 4;
    ++cpi;
  }
  if (nul) return enc_fail(c, E_NUL, t);
  const uint32_t nw = k.n / 4 + 1;
  if (c.out) {
    for (uint32_t q = 0; q < nw; ++q) {
      uint32_t w = 0;
      for (uint32_t b = 0; b < 4; ++b) {
        const uint32_t i = 4 * q + b;
        if (i < k.n) w |= (uint32_t)k.p[i] << (8 * b);
      }
      emit_word(c, w);
    }
  } else {
    if (c.r.nw <= 2 && c.r.nw + nw > 2) c.r.word2 = 0;
    c.r.nw += nw;
  }
  return true;
}

// encode_context_dependent_literal, integer flavour (codec.py:132-168)
__device__ inline bool enc_typed_int(EncCtx& c, uint32_t t, const IntVal& v, const LitInfo& inf) {
  const IntVal& w = inf.w;
  if (w.status != INT_OK || w.big || w.neg ||
      !(w.mag == 8 || w.mag == 16 || w.mag == 32 || w.mag == 64))
    return enc_fail(c, E_WIDTH, inf.wtok);
  const uint32_t width = (uint32_t)w.mag;
  bool fits;
  if (inf.sgn) {
    const uint64_t lim = 1ull << (width - 1);
    fits = !v.big && (v.neg ? v.mag <= lim : v.mag < lim);
  } else {
    fits = !v.big && (!v.neg || v.mag == 0) && (width == 64 || v.mag < (1ull << width));
  }
  if (!fits) return enc_fail(c, E_FIT, t, inf.sgn ? 1 : 0, width);
  uint64_t bits = v.neg ? (uint64_t)0 - v.mag : v.mag;
  if (width == 64) { emit_word(c, (uint32_t)bits); emit_word(c, (uint32_t)(bits >> 32)); return true; }
  uint32_t b = (uint32_t)bits & (width == 32 ? 0xFFFFFFFFu : ((1u << width) - 1));
  if (inf.sgn && v.neg && v.mag != 0 && width < 32) b |= 0xFFFFFFFFu << width;
  emit_word(c, b);
  return true;
}

__device__ inline bool enc_typed_float(EncCtx& c, uint32_t t, const Tok& k, const LitInfo& inf) {
  uint64_t bits;
  if (parse_float(k.p, k.n, c.X.U, bits) != FLT_OK) return enc_fail(c, E_FLOAT_INVALID, t);
  const IntVal& w = inf.w;
  if (w.status != INT_OK || w.big || w.neg ||
      !(w.mag == 8 || w.mag == 16 || w.mag == 32 || w.mag == 64))
    return enc_fail(c, E_WIDTH, inf.wtok);
  if (w.mag == 8) return enc_fail(c, E_FWIDTH, inf.wtok);
  if (w.mag == 64) { emit_word(c, (uint32_t)bits); emit_word(c, (uint32_t)(bits >> 32)); return true; }
  uint32_t o;
  if (w.mag == 32) { if (!pack_f32(bits, o)) return enc_fail(c, E_OVF_F, t); }
  else if (!pack_f16(bits, o)) return enc_fail(c, E_OVF_E, t);
  emit_word(c, o);
  return true;
}

constexpr int ESTACK = 48;
constexpr uint32_t KP_PARAM = 0x10000u;   // stack entry flag: take() with the "enumerant parameter" message

// value(kind, item) for one stack entry; pushes follow-ups
__device__ __forceinline__ bool enc_one(EncCtx& c, uint32_t entry, uint32_t* st, int& sp) {
  const Tables& T = c.X.T;
  const uint32_t k = entry & 0xFFFF;
  if (c.pos >= c.nitems) return enc_fail(c, E_MISSING, 0, k, (entry & KP_PARAM) ? 1 : 0);
  const uint32_t t = enc_item(c, c.pos++);
  const Tok tk = tok_of(c, t);
  uint32_t kk = k;
  // coerce(kind, token) sees the composite kind itself first: a string token there is
  // reported under the composite's name (reference asm.py:293-295, ops.py:160-164)
  if (tk.str && T.kcat(kk) == CAT_COMPOSITE) return enc_fail(c, E_STR_FOR, t, kk);
  // composite: value(bases[0], tok) then param(b) for the rest
  while (T.kcat(kk) == CAT_COMPOSITE) {
    const uint32_t nb = T.knbases(kk), bo = T.kbase_off(kk);
    if (sp + (int)nb > ESTACK) return enc_fail(c, E_MISSING, 0, kk, 1);
    for (int j = (int)nb - 1; j >= 1; --j) st[sp++] = (__ldg(T.slot + bo + j) & 0xFFFF) | KP_PARAM;
    kk = __ldg(T.slot + bo) & 0xFFFF;
  }
  const uint32_t cat = T.kcat(kk), sub = T.ksub(kk);
  if (tk.str && !(cat == CAT_LITERAL && sub == LIT_STRING)) return enc_fail(c, E_STR_FOR, t, kk);
  if (cat == CAT_ID) {
    uint32_t id;
    if (!enc_id(c, t, tk, id)) return false;
    if (sub == IDR_RESULT) c.r.result_id = id;
    else if (c.rbits) {
      const uint32_t b = c.rbase + c.r.nw;
      atomicOr(&c.rbits[b >> 5], 1u << (b & 31));
    } else if (c.mode == M_WRITE && c.r.bad_ref == NONE32) {
      if (!idset_has(c.m, c.m.reg, 0, id)) c.r.bad_ref = id;
    }
    emit_word(c, id);
    return true;
  }
  if (cat == CAT_VALUEENUM) {
    uint32_t e;
    if (int_token(tk.p, tk.n, c.X.U)) {
      const IntVal v = parse_int(tk.p, tk.n, 0, c.X.U);
      if (v.status == INT_INVALID) return enc_fail(c, E_INT_INVALID, t);
      if (v.status == INT_LIMIT) return enc_fail(c, E_INT_LIMIT, t, v.ndig);
      e = (!v.big && !(v.neg && v.mag) && v.mag <= 0xFFFFFFFFull) ? T.venum_lookup(kk, (uint32_t)v.mag) : NONE32;
      if (e == NONE32) return enc_fail(c, E_NO_ENUM_INT, t, kk);
    } else {
      e = enum_by_name(c.X, kk, tk.p, tk.n);
      if (e == NONE32) return enc_fail(c, E_NO_ENUM_STR, t, kk, 0, tk.n);
    }
    emit_word(c, T.evalue(e));
    const uint32_t np = T.enparams(e), po = T.eparam_off(e);
    if (sp + (int)np > ESTACK) return enc_fail(c, E_MISSING, 0, kk, 1);
    for (int j = (int)np - 1; j >= 0; --j) st[sp++] = T.slot_kind(po + j) | KP_PARAM;
    return true;
  }
  if (cat == CAT_BITENUM) {
    const uint32_t eo = T.kenum_off(kk), ne = T.knenum(kk);
    uint64_t parts = 0;
    uint32_t mask = 0;
    if (int_token(tk.p, tk.n, c.X.U)) {
      const IntVal v = parse_int(tk.p, tk.n, 0, c.X.U);
      if (v.status == INT_INVALID) return enc_fail(c, E_INT_INVALID, t);
      if (v.status == INT_LIMIT) return enc_fail(c, E_INT_LIMIT, t, v.ndig);
      if (v.big || (v.neg && v.mag) || v.mag > 0xFFFFFFFFull) return enc_fail(c, E_MASK_RANGE, t, kk);
      mask = (uint32_t)v.mag;
      if (mask) {   // bit_components: all-or-nothing cover in file order (ops.py:77-89)
        uint32_t covered = 0;
        uint64_t p = 0;
        for (uint32_t j = 0; j < ne && j < 64; ++j) {
          const uint32_t ev = T.evalue(eo + j);
          if (ev && (mask & ev) == ev && (covered & ev) != ev) { covered |= ev; p |= 1ull << j; }
        }
        if (covered == mask) parts = p;
      }
    } else {
      // "A|B" names (ops.py:189-201)
      uint32_t s = 0;
      while (s <= tk.n) {
        uint32_t e = s;
        while (e < tk.n && tk.p[e] != '|') ++e;
        uint32_t a, b;
        py_strip(tk.p + s, e - s, c.X.U, a, b);
        if (b > a) {
          const uint32_t en = enum_by_name(c.X, kk, tk.p + s + a, b - a);
          if (en == NONE32) return enc_fail(c, E_NO_ENUM_STR, t, kk, s + a, b - a);
          const uint32_t ev = T.evalue(en);
          if (ev && (mask & ev) != ev) parts |= 1ull << ((en - eo) & 63);
          mask |= ev;
        }
        s = e + 1;
      }
    }
    emit_word(c, mask);
    // parameters of the parts in file order: push in reverse
    for (int j = 63; j >= 0; --j) {
      if (!((parts >> j) & 1)) continue;
      const uint32_t e = eo + (uint32_t)j;
      const uint32_t np = T.enparams(e), po = T.eparam_off(e);
      if (sp + (int)np > ESTACK) return enc_fail(c, E_MISSING, 0, kk, 1);
      for (int q = (int)np - 1; q >= 0; --q) st[sp++] = T.slot_kind(po + q) | KP_PARAM;
    }
    return true;
  }
  // literals
  if (sub == LIT_STRING) {
    if (tk.str) return enc_string(c, t, tk);
    const IntVal v = parse_int(tk.p, tk.n, 0, c.X.U);
    if (v.status == INT_INVALID) return enc_fail(c, E_INT_INVALID, t);
    if (v.status == INT_LIMIT) return enc_fail(c, E_INT_LIMIT, t, v.ndig);
    if (v.neg && (v.mag || v.big)) return enc_fail(c, E_NEG, t, kk);
    return enc_fail(c, E_LITSTR_INT, t);
  }
  if (sub == LIT_CTXNUM) {
    if (!c.info.ok) return enc_fail(c, E_NO_WIDTH, t);
    if (c.info.flt) return enc_typed_float(c, t, tk, c.info);
    const IntVal v = parse_int(tk.p, tk.n, 0, c.X.U);
    if (v.status == INT_INVALID) return enc_fail(c, E_INT_INVALID, t);
    if (v.status == INT_LIMIT) return enc_fail(c, E_INT_LIMIT, t, v.ndig);
    return enc_typed_int(c, t, v, c.info);
  }
  if (sub == LIT_INTEGER && c.is_switch && c.info.ok) {
    const IntVal v = parse_int(tk.p, tk.n, 0, c.X.U);
    if (v.status == INT_INVALID) return enc_fail(c, E_INT_INVALID, t);
    if (v.status == INT_LIMIT) return enc_fail(c, E_INT_LIMIT, t, v.ndig);
    return enc_typed_int(c, t, v, c.info);
  }
  if ((sub == LIT_EXTINST || sub == LIT_SPECOP) && !int_token(tk.p, tk.n, c.X.U)) {
    if (sub == LIT_EXTINST) {
      uint32_t num;
      if (!ext_by_name(c.X, tk.p, tk.n, num)) return enc_fail(c, E_NO_EXT, t);
      emit_word(c, num);
      return true;
    }
    const bool has_op = tk.n >= 2 && tk.p[0] == 'O' && tk.p[1] == 'p';
    const uint32_t d = has_op ? inst_by_name(c.X, tk.p, tk.n)
                              : inst_by_name(c.X, tk.p, tk.n, (const uint8_t*)"Op", 2);
    if (d == NONE32) return enc_fail(c, E_NO_SPECOP, t, has_op ? 0 : 1);
    emit_word(c, __ldg(T.irec(d) + 5));
    return true;
  }
  const IntVal v = parse_int(tk.p, tk.n, 0, c.X.U);
  if (v.status == INT_INVALID) return enc_fail(c, E_INT_INVALID, t);
  if (v.status == INT_LIMIT) return enc_fail(c, E_INT_LIMIT, t, v.ndig);
  const bool negative = v.neg && (v.mag || v.big);
  if (negative && sub != LIT_EXTINST && sub != LIT_SPECOP) return enc_fail(c, E_NEG, t, kk);
  if (negative || v.big || v.mag > 0xFFFFFFFFull) return enc_fail(c, E_LIT_RANGE, t, kk);
  emit_word(c, (uint32_t)v.mag);
  return true;
}

// Encoder.encode (ops.py:120-155) over the instruction's slots.  The context
// is copied into registers for the walk (the caller's copy lives in local
// memory) and enc_one is inlined at a single call site: the slot sequence
// ('*' repeats to the end, '?' skipped when no tokens remain, the
// SpecConstantOp IdRef tail) is generated by a small state machine.
__device__ inline bool enc_setup(EncCtx& c, const AsmMod& m, uint32_t li);

__device__ __forceinline__ void encode_walk(EncCtx& c) {
  const Tables& T = c.X.T;
  c.pos = 0;
  uint32_t st[ESTACK];
  int sp = 0;
  const uint32_t ns = T.inslots(c.d), so = T.islot_off(c.d);
  uint32_t s = 0, repk = 0;
  bool rep = false, stop_after = false, pending_tail = false;
#pragma unroll 1
  for (;;) {
    if (sp == 0) {
      if (pending_tail) { pending_tail = false; rep = true; stop_after = false; repk = T.idref; }
      if (rep) {
        if (c.pos >= c.nitems) {
          if (stop_after) break;
          rep = false;
          continue;
        }
        st[sp++] = repk;
      } else {
        if (s >= ns) break;
        const uint32_t q = T.slot_quant(so + s), k = T.slot_kind(so + s);
        const bool tail = T.slot_spec_tail(so + s);
        ++s;
        if (q == Q_VAR) { rep = true; stop_after = true; repk = k; continue; }
        if (q == Q_OPT && c.pos >= c.nitems) continue;
        st[sp++] = k;
        pending_tail = tail;
      }
    }
    const uint32_t e = st[--sp];
    if (!enc_one(c, e, st, sp)) return;
  }
  if (c.pos < c.nitems) enc_fail(c, E_EXTRA, 0, c.nitems - c.pos);
}

// One line through the encoder, the context built here in registers rather
// than passed in through (per-lane) local memory.  Pass 1 (M_COUNT) stores the
// line's results itself; the other modes return them through *ro.
__device__ __noinline__ void encode_line(const AsmMod& m, const AsmCtx& X, uint32_t li, uint32_t d, uint32_t mode,
                                         uint32_t* out, uint32_t* rbits, uint32_t rbase, EncOut* ro) {
  EncCtx c{m, X, li, d, mode, out};
  c.rbits = rbits;
  c.rbase = rbase;
  c.r.nw = 0; c.r.ecode = E_OK; c.r.result_id = 0; c.r.word2 = NONE32; c.r.unres = false;
  c.r.bad_ref = NONE32;
  const bool setup = enc_setup(c, m, li);
  if (setup) encode_walk(c);   // one inlined copy of the walk
  if (ro) { *ro = c.r; return; }
  m.lec[li] = c.r.ecode;
  if (!setup) return;
  if (c.r.ecode != E_OK) {
    uint32_t* e = m.lerr + 4 * li;
    e[0] = c.r.etok; e[1] = c.r.eaux; e[2] = c.r.eaux2; e[3] = c.r.eaux3;
  }
  m.lnw[li] = c.r.nw;
  m.lrid[li] = c.r.result_id;
  uint32_t f2 = m.lfl[li];
  if (c.r.unres) f2 |= LF_UNRES;
  if (X.T.special(d) == SP_VARIABLE && c.r.word2 == X.A.storage_fn) f2 |= LF_VARFN;
  m.lfl[li] = f2;
}

// set up an encoder context for line li (d known, not OpLabel); false = pre-encode error
__device__ inline bool enc_setup(EncCtx& c, const AsmMod& m, uint32_t li) {
  const Tables& T = c.X.T;
  const uint32_t fl = m.lfl[li];
  const bool has_res = fl & LF_RESULT;
  c.rtok = has_res ? m.lt0[li] : NONE32;
  const uint32_t first = has_res ? 3 : 1;
  c.ops0 = m.lt0[li] + first;
  c.nops = m.lnt[li] - first;
  const uint32_t info = __ldg(c.X.A.info + 4 * c.d);
  if (T.has_result(c.d)) {
    if (!has_res) { c.r.ecode = E_NEEDS_RESULT; return false; }
    const uint32_t rs = info & 0xFF;
    c.ridx = rs < c.nops ? rs : c.nops;
    c.nitems = c.nops + 1;
  } else {
    if (has_res) { c.r.ecode = E_NOT_PRODUCE; return false; }
    c.ridx = NONE32;
    c.nitems = c.nops;
  }
  c.is_switch = T.special(c.d) == SP_SWITCH;
  c.info.ok = false;
  if (c.is_switch) {
    if (c.nops > 0) {
      const Tok sel = tok_at(m, c.ops0);
      const uint32_t e = nt_find(m, sel.p, sel.n);
      const uint32_t vl = e != NONE32 ? m.nt[NT_W * e + 5] : 0;
      if (vl) {
        const Tok vt = tok_at(m, op_tok(m, vl - 1, 0));
        c.info = width_of_entry(m, c.X, nt_find(m, vt.p, vt.n));
      }
    }
  } else if (((info >> 16) & AF_CTXNUM) && T.has_rtype(c.d) && c.nops > 0) {
    const Tok rt = tok_at(m, c.ops0);
    c.info = width_of_entry(m, c.X, nt_find(m, rt.p, rt.n));
  }
  return true;
}

// ============================================================================
// Header comments (asm.py:184-206): returns X_NONE or a ValueError outcome.
// Groups are matched on the stripped line with Unicode \s and \d.
struct Dec {   // a \d+ group: value mod 2^32, ==1 test, small (< 2^32) value
  uint32_t mod32;
  uint32_t ndig;
  bool fits;       // value < 2^32
  uint32_t s, e;   // byte range
};

__device__ inline uint32_t skip_ws(const uint8_t* p, uint32_t n, uint32_t i, const Uni& U) {
  while (i < n) { uint32_t len, c = utf8_cp(p, n, i, len); if (!U.is_space(c)) break; i += len; }
  return i;
}
__device__ inline bool match_dec(const uint8_t* p, uint32_t n, uint32_t& i, const Uni& U, Dec& d) {
  d.mod32 = 0; d.ndig = 0; d.fits = true; d.s = i;
  uint64_t v = 0;
  while (i < n) {
    uint32_t len, c = utf8_cp(p, n, i, len);
    const int x = U.decimal(c);
    if (x < 0) break;
    d.mod32 = d.mod32 * 10 + (uint32_t)x;
    if (d.fits) { v = v * 10 + (uint64_t)x; if (v > 0xFFFFFFFFull) d.fits = false; }
    ++d.ndig;
    i += len;
  }
  d.e = i;
  return d.ndig > 0;
}
__device__ inline bool match_lit(const uint8_t* p, uint32_t n, uint32_t& i, const char* z) {
  uint32_t j = i;
  for (; *z; ++z, ++j) if (j >= n || p[j] != (uint8_t)*z) return false;
  i = j;
  return true;
}


// ============================================================================
// Message formatting (lane 0): str(exc) of the exceptions the reference raises.
struct FmtCtx {
  const AsmMod& m;
  const AsmCtx& X;
  const uint32_t* knames;   // per kind: (string offset, length)
  uint32_t* scratch;        // big-integer limbs
  uint32_t scratch_limbs;
};

__device__ const char* const STR_LIMIT_MSG =
    "Exceeds the limit (4300 digits) for integer string conversion; use sys.set_int_max_str_digits() "
    "to increase the limit";

template <class S>
__device__ void put_tab(S& s, const Tables& T, uint32_t off, uint32_t len) {
  for (uint32_t i = 0; i < len; ++i) s.put(__ldg(T.str + off + i));
}
template <class S>
__device__ void put_dname(S& s, const FmtCtx& F, uint32_t d) {
  put_tab(s, F.X.T, F.X.T.iname_off(d), F.X.T.iname_len(d));
}
template <class S>
__device__ void put_kname(S& s, const FmtCtx& F, uint32_t k) {
  put_tab(s, F.X.T, __ldg(F.knames + 2 * k), __ldg(F.knames + 2 * k + 1));
}
template <class S>
__device__ void put_id(S& s, uint32_t id) {   // Id.__repr__ inside "%{id}" -> "%%N"
  s.put('%'); s.put('%'); put_u64(s, id);
}

// does str(int(text, 0)) succeed (<= 4300 digits)?
__device__ inline bool int_prints(const FmtCtx& F, const Tok& k, const IntVal& v) {
  Sink cnt;
  return put_int_decimal(cnt, k.p, v, F.X.U, F.scratch, F.scratch_limbs / 2);
}
template <class S>
__device__ void put_int_of(S& s, const FmtCtx& F, const Tok& k, const IntVal& v) {
  put_int_decimal(s, k.p, v, F.X.U, F.scratch, F.scratch_limbs / 2);
}

template <class S>
__device__ void put_col(S& s, const FmtCtx& F, uint32_t li, uint32_t raw) {
  put_u64(s, li + 1);
  s.put(':');
  put_u64(s, cp_count(F.m.txt + F.m.ls[li], raw - F.m.ls[li]) + 1);
  s.put(':'); s.put(' ');
}

// message of an emit-phase diagnostic of line li
template <class S>
__device__ __noinline__ void put_emit_msg(S& s, const FmtCtx& F, uint32_t li) {
  const AsmMod& m = F.m;
  const uint32_t code = m.lec[li];
  const uint32_t* e = m.lerr + 4 * li;
  const uint32_t d = m.ld[li];
  const Uni& U = F.X.U;
  auto tokrepr = [&](uint32_t t, uint32_t limit) { const Tok k = tok_at(m, t); put_py_repr(s, k.p, k.n, U, limit); };
  switch (code) {
    case E_NOINST: {
      put_cstr(s, "no instruction ");
      tokrepr(m.lt0[li] + ((m.lfl[li] & LF_RESULT) ? 2 : 0), 0);
      put_cstr(s, " in grammar");
      break;
    }
    case E_NEEDS_RESULT: put_dname(s, F, d); put_cstr(s, " needs a result name"); break;
    case E_NOT_PRODUCE: put_dname(s, F, d); put_cstr(s, " does not produce a result"); break;
    case E_MISSING:
      put_cstr(s, "missing operand: expected "); put_dname(s, F, d);
      put_cstr(s, e[2] ? " enumerant parameter of kind " : " operand of kind "); put_kname(s, F, e[1]);
      break;
    case E_EXTRA: put_dname(s, F, d); put_cstr(s, ": "); put_u64(s, e[1]); put_cstr(s, " unexpected extra operand(s)"); break;
    case E_STR_FOR: put_cstr(s, "string literal given for a "); put_kname(s, F, e[1]); put_cstr(s, " operand"); break;
    case E_EXPECT_ID: put_cstr(s, "expected an id like %name, got "); tokrepr(e[0], 0); break;
    case E_INT_INVALID: put_cstr(s, "invalid literal for int() with base 0: "); tokrepr(e[0], 200); break;
    case E_INT_LIMIT:
      put_cstr(s, "Exceeds the limit (4300 digits) for integer string conversion: value has ");
      put_u64(s, e[1]);
      put_cstr(s, " digits; use sys.set_int_max_str_digits() to increase the limit");
      break;
    case E_FLOAT_INVALID: put_cstr(s, "could not convert string to float: "); tokrepr(e[0], 0); break;
    case E_NO_WIDTH: put_cstr(s, "cannot resolve the literal width (unknown governing type)"); break;
    case E_NEG: put_kname(s, F, e[1]); put_cstr(s, " cannot be negative"); break;
    case E_NO_ENUM_STR: {
      const Tok k = tok_at(m, e[0]);
      put_cstr(s, "no enumerant ");
      put_py_repr(s, k.p + e[2], e[3], U);
      put_cstr(s, " in operand kind "); put_kname(s, F, e[1]);
      break;
    }
    case E_NO_ENUM_INT: case E_LITSTR_INT: case E_FIT: case E_LIT_RANGE: case E_WIDTH: case E_FWIDTH: {
      const Tok k = tok_at(m, e[0]);
      const IntVal v = parse_int(k.p, k.n, 0, U);
      if (!int_prints(F, k, v)) { put_cstr(s, STR_LIMIT_MSG); break; }
      if (code == E_NO_ENUM_INT) {
        put_cstr(s, "no enumerant "); put_int_of(s, F, k, v); put_cstr(s, " in operand kind "); put_kname(s, F, e[1]);
      } else if (code == E_LITSTR_INT) {
        put_dname(s, F, d); put_cstr(s, ": literal string expected, got "); put_int_of(s, F, k, v);
      } else if (code == E_FIT) {
        put_cstr(s, "value "); put_int_of(s, F, k, v);
        put_cstr(s, e[1] ? " does not fit a signed " : " does not fit an unsigned "); put_u64(s, e[2]);
        put_cstr(s, "-bit literal");
      } else if (code == E_LIT_RANGE) {
        put_dname(s, F, d); put_cstr(s, ": "); put_kname(s, F, e[1]); put_cstr(s, " value ");
        put_int_of(s, F, k, v); put_cstr(s, " out of range");
      } else {
        put_cstr(s, code == E_WIDTH ? "unsupported literal width " : "unsupported float width ");
        put_int_of(s, F, k, v);
      }
      break;
    }
    case E_MASK_RANGE: {
      const Tok k = tok_at(m, e[0]);
      const IntVal v = parse_int(k.p, k.n, 0, U);
      put_dname(s, F, d); put_cstr(s, ": "); put_kname(s, F, e[1]); put_cstr(s, " mask ");
      put_int_hex(s, k.p, v, U, F.scratch, F.scratch_limbs);
      put_cstr(s, " out of range");
      break;
    }
    case E_NUL: put_cstr(s, "string literal contains an embedded NUL byte"); break;
    case E_SURROGATE: {
      const Tok k = tok_at(m, e[0]);
      put_cstr(s, "'utf-8' codec can't encode ");
      if (e[2] - e[1] == 1) {
        uint32_t cp = 0;   // the surrogate code point at index e[1]
        for (uint32_t i = 0, q = 0; i < k.n; ++q) {
          uint32_t len, c = utf8_cp(k.p, k.n, i, len);
          if (q == e[1]) { cp = c; break; }
          i += len;
        }
        put_cstr(s, "character '\\u");
        for (int sh = 12; sh >= 0; sh -= 4) s.put((uint8_t)"0123456789abcdef"[(cp >> sh) & 0xF]);
        put_cstr(s, "' in position "); put_u64(s, e[1]);
      } else {
        put_cstr(s, "characters in position "); put_u64(s, e[1]); s.put('-'); put_u64(s, e[2] - 1);
      }
      put_cstr(s, ": surrogates not allowed");
      break;
    }
    case E_NO_EXT: put_cstr(s, "no extended instruction "); tokrepr(e[0], 0); break;
    case E_NO_SPECOP: {
      const Tok k = tok_at(m, e[0]);
      put_cstr(s, "no instruction ");
      put_py_repr_prefixed(s, e[1] ? "Op" : "", k.p, k.n, U);
      put_cstr(s, " in grammar");
      break;
    }
    case S_LABEL_OUTSIDE: put_cstr(s, "OpLabel outside a function"); break;
    case S_LABEL_NORESULT: put_cstr(s, "OpLabel needs a result name"); break;
    case S_LABEL_RESOLVE: put_cstr(s, "expected an id like %name, got "); tokrepr(m.lt0[li], 0); break;
    case S_LABEL_USED: put_id(s, e[0]); put_cstr(s, " is already used as a block label"); break;
    case S_DUP: put_id(s, e[0]); put_cstr(s, " is defined by more than one instruction"); break;
    case S_FUNC_BEFORE_END: put_cstr(s, "OpFunction before the previous OpFunctionEnd"); break;
    case S_OUTSIDE: put_dname(s, F, d); put_cstr(s, " outside a function"); break;
    case S_PARAM_AFTER_BLOCK: put_cstr(s, "function parameters must precede all blocks"); break;
    case S_MM_DUP: put_cstr(s, "module already has a memory model"); break;
    case S_NEED_BLOCK: put_dname(s, F, d); put_cstr(s, " must appear inside a block"); break;
    case S_TERMINATED: put_cstr(s, "block already has its terminator"); break;
    case S_VAR_FIRST: put_cstr(s, "Function-storage OpVariable must open the first block"); break;
    case S_VAR_NOTFN: put_cstr(s, "only Function-storage OpVariable belongs in a block"); break;
    case S_NOT_BLOCK: {
      put_dname(s, F, d); put_cstr(s, " (");
      const uint32_t* inf = F.X.A.info + 4 * d;
      put_tab(s, F.X.T, __ldg(inf + 1), __ldg(inf + 2));
      put_cstr(s, ") is not a block instruction");
      break;
    }
    case S_KEYERROR: {   // str(KeyError(name)) = repr(name)
      const Tables& T = F.X.T;
      put_py_repr(s, T.str + T.iname_off(d), T.iname_len(d), U);
      break;
    }
    default: put_cstr(s, "internal: unknown diagnostic"); break;
  }
}

// AssemblyError text: "{n} error(s):\n" + "line:col: msg" lines (errors.py:73-94)
template <class S>
__device__ __noinline__ void put_assembly_error(S& s, const FmtCtx& F, uint32_t ndiag) {
  const AsmMod& m = F.m;
  put_u64(s, ndiag);
  put_cstr(s, " error(s):");
  for (uint32_t li = 0; li < m.L; ++li) {          // tokenizer diagnostics
    if (!(m.lfl[li] & LF_TOKERR)) continue;
    s.put('\n'); put_col(s, F, li, m.lerr[4 * li]); put_cstr(s, "unterminated string literal");
  }
  for (uint32_t li = 0; li < m.L; ++li) {          // result-name diagnostics
    if (!(m.lfl[li] & LF_RESOLVE_ERR)) continue;
    s.put('\n'); put_col(s, F, li, tok_at(m, m.lt0[li]).raw);
    put_cstr(s, "expected an id like %name, got ");
    const Tok k = tok_at(m, m.lt0[li]);
    put_py_repr(s, k.p, k.n, F.X.U);
  }
  for (uint32_t li = 0; li < m.L; ++li) {          // emit diagnostics
    if ((m.lfl[li] & (LF_TOKERR | LF_EMPTY)) || m.lec[li] == E_OK) continue;
    s.put('\n');
    put_col(s, F, li, tok_at(m, m.lt0[li] + ((m.lfl[li] & LF_RESULT) ? 2 : 0)).raw);
    put_emit_msg(s, F, li);
  }
}

// module-level exception text
template <class S>
__device__ __noinline__ void put_module_error(S& s, const FmtCtx& F, uint32_t x, uint32_t ndiag) {
  const AsmMod& m = F.m;
  const uint32_t* ms = m.misc;
  switch (x) {
    case X_VERSION: {
      put_cstr(s, "unsupported SPIR-V version ");
      // normalised decimals of the last Version: groups (byte ranges in misc)
      for (int g = 0; g < 2; ++g) {
        if (g) s.put('.');
        const uint32_t a = ms[MS_V0 + 2 * g], b = ms[MS_V0 + 2 * g + 1];
        bool lead = true, any = false;
        for (uint32_t i = a; i < b;) {
          uint32_t len, c = utf8_cp(m.txt, b, i, len);
          i += len;
          const int dv = F.X.U.decimal(c);
          if (lead && dv == 0) continue;
          lead = false; any = true;
          s.put((uint8_t)('0' + dv));
        }
        if (!any) s.put('0');
      }
      break;
    }
    case X_VERSION_DEFAULT:
      put_cstr(s, "unsupported SPIR-V version "); put_u64(s, ms[MS_V0]); s.put('.'); put_u64(s, ms[MS_V0 + 1]);
      break;
    case X_VERSION_LIMIT:
      put_cstr(s, "Exceeds the limit (4300 digits) for integer string conversion: value has ");
      put_u64(s, ms[MS_XA]);
      put_cstr(s, " digits; use sys.set_int_max_str_digits() to increase the limit");
      break;
    case X_RESERVE: {
      const uint32_t li = ms[MS_RESV_LINE];
      const Tok k = tok_at(m, m.lerr[4 * li + 1]);
      const IntVal v = parse_int(k.p + 1, k.n - 1, 10, F.X.U);
      if (v.status == INT_INVALID) {
        put_cstr(s, "invalid literal for int() with base 10: ");
        put_py_repr(s, k.p + 1, k.n - 1, F.X.U, 200);
      } else if (v.status == INT_LIMIT) {
        put_cstr(s, "Exceeds the limit (4300 digits) for integer string conversion: value has ");
        put_u64(s, v.ndig);
        put_cstr(s, " digits; use sys.set_int_max_str_digits() to increase the limit");
      } else {
        put_cstr(s, "id ");
        put_int_decimal(s, k.p + 1, v, F.X.U, F.scratch, F.scratch_limbs / 2);
        put_cstr(s, " out of range");
      }
      break;
    }
    case X_OVERFLOW:
      put_cstr(s, m.lec[ms[MS_OVF_LINE]] == E_OVF_E ? "float too large to pack with e format"
                                                     : "float too large to pack with f format");
      break;
    case X_ASSEMBLY: put_assembly_error(s, F, ndiag); break;
    case X_STRUCT_END: put_cstr(s, "function "); put_id(s, ms[MS_XA]); put_cstr(s, " has no OpFunctionEnd"); break;
    case X_STRUCT_TERM:
      put_cstr(s, "block "); put_id(s, ms[MS_XB]); put_cstr(s, " in function "); put_id(s, ms[MS_XA]);
      put_cstr(s, " has no terminator");
      break;
    case X_SERIAL:
      put_id(s, ms[MS_XA]); put_cstr(s, " is referenced by "); put_dname(s, F, ms[MS_XB]);
      put_cstr(s, " but never defined");
      break;
    case X_WC:
      put_cstr(s, "instruction length "); put_u64(s, ms[MS_XA]);
      put_cstr(s, " words overflows the 16-bit count");
      break;
    default: put_cstr(s, "internal: module exceeds the per-warp assembler scratch"); break;
  }
}

// ============================================================================
// Phase C: header comments (asm.py:184-206), one line per lane in rounds of 32
// lines; the outcome is the reference's sequential loop: lines up to the first
// non-comment line, the first int() digit-limit error stops the scan, and a later
// match of a pattern overrides an earlier one.  Returns X_NONE / X_VERSION_LIMIT /
// X_VERSION / X_VERSION_DEFAULT and fills major/minor validity, generator, schema.
struct HdrLine {
  uint32_t key;        // 0 none, 1 version, 2 generator, 3 schema, 4 digit-limit error, 5 stop
  uint32_t a, b, c, d; // version: d1.s, d1.e, d2.s, d2.e (line-relative) | generator word | schema
  uint32_t f;          // version: major/minor validity (major ok << 16 | minor + 1) | limit: digits
};

__device__ __forceinline__ HdrLine header_line(const AsmMod& m, const AsmCtx& X, uint32_t li) {
  const Uni& U = X.U;
  HdrLine r{0, 0, 0, 0, 0, 0};
  const uint8_t* p = m.txt + m.ls[li];
  const uint32_t n = m.le[li] - m.ls[li];
  // an instruction line (the common case): after ASCII blanks, a printable ASCII byte
  // other than ';' -- str.strip() then leaves it non-empty and not a comment
  {
    uint32_t i = 0;
    while (i < n && (p[i] == ' ' || p[i] == '\t')) ++i;
    if (i < n && p[i] > 0x20 && p[i] < 0x7F && p[i] != ';') { r.key = 5; return r; }
  }
  uint32_t a, b;
  py_strip(p, n, U, a, b);
  if (b > a && p[a] != ';') { r.key = 5; return r; }
  if (b == a) return r;
  // the three patterns, anchored at a, must consume up to b
  for (int key = 0; key < 3; ++key) {
    uint32_t i = a;
    if (!match_lit(p, b, i, ";")) break;
    i = skip_ws(p, b, i, U);
    const char* kw = key == 0 ? "Version:" : key == 1 ? "Generator:" : "Schema:";
    if (!match_lit(p, b, i, kw)) continue;
    i = skip_ws(p, b, i, U);
    Dec d1, d2;
    if (!match_dec(p, b, i, U, d1)) continue;
    if (key == 0) {
      if (!match_lit(p, b, i, ".")) continue;
      if (!match_dec(p, b, i, U, d2)) continue;
    } else if (key == 1) {
      if (!match_lit(p, b, i, ";")) continue;
      i = skip_ws(p, b, i, U);
      if (!match_dec(p, b, i, U, d2)) continue;
    }
    i = skip_ws(p, b, i, U);
    if (i != b) continue;
    // int() of each group, in order (the 4300-digit limit raises here)
    if (d1.ndig > PY_MAX_STR_DIGITS) { r.key = 4; r.f = d1.ndig; return r; }
    if (key != 2 && d2.ndig > PY_MAX_STR_DIGITS) { r.key = 4; r.f = d2.ndig; return r; }
    if (key == 0) {
      r.key = 1;
      r.a = d1.s; r.b = d1.e; r.c = d2.s; r.d = d2.e;
      r.f = ((d1.fits && d1.mod32 == 1) ? 1u << 16 : 0u) | ((d2.fits && d2.mod32 <= 6) ? d2.mod32 + 1 : 0u);
    } else if (key == 1) {
      r.key = 2;
      r.a = ((d1.mod32 & 0xFFFFu) << 16) | d2.mod32;
    } else {
      r.key = 3;
      r.a = d1.mod32;
    }
    break;
  }
  return r;
}

__device__ __noinline__ uint32_t scan_header(AsmMod& m, const AsmCtx& X, uint32_t dv) {
  const uint32_t lane = lane_id_a();
  uint32_t* ms = m.misc;
  bool vset = false;
  for (uint32_t base = 0; base < m.L; base += 32) {
    const uint32_t li = base + lane;
    const HdrLine h = li < m.L ? header_line(m, X, li) : HdrLine{0, 0, 0, 0, 0, 0};
    const uint32_t stop = __ballot_sync(FULLM, h.key == 5);
    const uint32_t upto = stop ? (1u << (__ffs(stop) - 1)) - 1 : FULLM;   // lanes before the stop line
    const uint32_t lim = __ballot_sync(FULLM, h.key == 4) & upto;
    // the last match of each key among lanes [0, first limit error) wins
    const uint32_t valid = lim ? (1u << (__ffs(lim) - 1)) - 1 : upto;
    const uint32_t kv = __ballot_sync(FULLM, h.key == 1) & valid;
    const uint32_t kg = __ballot_sync(FULLM, h.key == 2) & valid;
    const uint32_t ks = __ballot_sync(FULLM, h.key == 3) & valid;
    if (kv && lane == 31 - __clz(kv)) {
      const uint32_t lb = m.ls[li];
      ms[MS_MAJOR] = h.f >> 16;
      ms[MS_MINOR] = h.f & 0xFFFF;
      ms[MS_V0] = lb + h.a; ms[MS_V0 + 1] = lb + h.b;
      ms[MS_V0 + 2] = lb + h.c; ms[MS_V0 + 3] = lb + h.d;
    }
    if (kg && lane == 31 - __clz(kg)) { ms[MS_GEN] = h.a; ms[MS_GENSET] = 1; }
    if (ks && lane == 31 - __clz(ks)) ms[MS_SCHEMA] = h.a;
    vset |= kv != 0;
    if (lim) {
      if (lane == __ffs(lim) - 1) ms[MS_XA] = h.f;
      __syncwarp();
      return X_VERSION_LIMIT;
    }
    if (stop) break;
  }
  __syncwarp();
  if (!vset) {   // Assembler.default_version
    const uint32_t mj = dv >> 16, mn = dv & 0xFFFF;
    if (!(mj == 1 && mn <= 6)) {
      if (lane == 0) { ms[MS_V0] = mj; ms[MS_V0 + 1] = mn; }
      __syncwarp();
      return X_VERSION_DEFAULT;
    }
    if (lane == 0) { ms[MS_MAJOR] = 1; ms[MS_MINOR] = mn + 1; }
    __syncwarp();
    return X_NONE;
  }
  if (!(ms[MS_MAJOR] == 1 && ms[MS_MINOR] != 0)) return X_VERSION;
  return X_NONE;
}

// label id / result id of a result token without encoding (lane-local)
__device__ inline uint32_t result_id_of(const AsmMod& m, const AsmCtx& X, uint32_t t) {
  if (m.tid[t]) return m.tid[t];
  const Tok k = tok_at(m, t);
  if (k.n < 2) return 0;
  if (py_isdigit(k.p + 1, k.n - 1, X.U)) return (uint32_t)parse_int(k.p + 1, k.n - 1, 10, X.U).mag;
  const uint32_t e = nt_find(m, k.p, k.n);
  return e != NONE32 ? m.nt[NT_W * e + 3] : 0;
}

// lane 0: re-run the encoder of line li assigning ids to unseen names in order
__device__ __noinline__ bool resolve_line(AsmMod& m, const AsmCtx& X, uint32_t li) {
  EncOut r;
  encode_line(m, X, li, m.ld[li], M_RESOLVE, nullptr, nullptr, 0, &r);
  return r.ecode != E_INTERNAL;
}

// Phase G (lane 0): the scope state machine of Assembler._emit / builder scopes.
constexpr uint32_t FN_ENDED = 1, FN_BLOCKS = 2;
__device__ __noinline__ uint32_t state_machine(AsmMod& m, const AsmCtx& X) {
  const Tables& T = X.T;
  int32_t fn = -1, blk = -1;
  uint32_t nfn = 0, nblk = 0, ndiag = 0;
  bool mm = false, blk_term = false, blk_nonvar = false;
  uint32_t* bucket = m.misc + MS_BUCKET0;
  auto diag = [&](uint32_t li, uint32_t code, uint32_t a = 0) {
    m.lec[li] = code;
    m.lerr[4 * li] = a;
    ++ndiag;
  };
  auto place_fn = [&](uint32_t li, uint32_t words) {
    m.lgrp[li] = 16 + (uint32_t)fn;
    m.loff[li] = m.fn[4 * fn + 2];
    m.fn[4 * fn + 2] += words;
    m.lfl[li] |= LF_PLACED;
  };
  for (uint32_t li = 0; li < m.L; ++li) {
    const uint32_t fl = m.lfl[li];
    if (fl & (LF_TOKERR | LF_EMPTY)) continue;
    const uint32_t d = m.ld[li];
    if (d == NONE32) { ++ndiag; continue; }
    const uint32_t sp = T.special(d);
    if (sp == SP_LABEL) {
      if (fn < 0) { diag(li, S_LABEL_OUTSIDE); continue; }
      if (!(fl & LF_RESULT)) { diag(li, S_LABEL_NORESULT); continue; }
      if (fl & LF_RESOLVE_ERR) { diag(li, S_LABEL_RESOLVE); continue; }
      const uint32_t L = m.lrid[li];
      if (idset_has(m, m.lab, 1, L)) { diag(li, S_LABEL_USED, L); continue; }
      if (idset_has(m, m.reg, 0, L)) { diag(li, S_DUP, L); continue; }
      if (!idset_add(m, m.lab, 1, L) || !idset_add(m, m.reg, 0, L)) return NONE32;
      blk = (int32_t)nblk++;
      m.blk[3 * blk] = (uint32_t)fn; m.blk[3 * blk + 1] = L; m.blk[3 * blk + 2] = 0;
      m.fn[4 * fn + 1] |= FN_BLOCKS;
      blk_term = false; blk_nonvar = false;
      m.lnw[li] = 1;
      place_fn(li, 2);
      continue;
    }
    if ((fl & LF_UNRES) && !resolve_line(m, X, li)) return NONE32;
    if (m.lec[li] != E_OK) { ++ndiag; continue; }
    const uint32_t info = __ldg(X.A.info + 4 * d);
    const uint32_t words = 1 + m.lnw[li];
    const bool has_res = T.has_result(d);
    const uint32_t rid = m.lrid[li];
    if (sp == SP_FUNCTION) {
      if (fn >= 0 && !(m.fn[4 * fn + 1] & FN_ENDED)) { diag(li, S_FUNC_BEFORE_END); continue; }
      if (idset_has(m, m.reg, 0, rid)) { diag(li, S_DUP, rid); continue; }
      if (!idset_add(m, m.reg, 0, rid)) return NONE32;
      fn = (int32_t)nfn++;
      m.fn[4 * fn] = rid; m.fn[4 * fn + 1] = 0; m.fn[4 * fn + 2] = 0; m.fn[4 * fn + 3] = 0;
      blk = -1;
      place_fn(li, words);
      continue;
    }
    if (sp == SP_FUNCTIONPARAM || sp == SP_FUNCTIONEND) {
      if (fn < 0) { diag(li, S_OUTSIDE); continue; }
      if (sp == SP_FUNCTIONPARAM) {
        if (m.fn[4 * fn + 1] & FN_BLOCKS) { diag(li, S_PARAM_AFTER_BLOCK); continue; }
        if (has_res) {
          if (idset_has(m, m.reg, 0, rid)) { diag(li, S_DUP, rid); continue; }
          if (!idset_add(m, m.reg, 0, rid)) return NONE32;
        }
        place_fn(li, words);
        continue;
      }
      m.fn[4 * fn + 1] |= FN_ENDED;
      m.lfl[li] |= LF_DROP;
      fn = -1; blk = -1;
      continue;
    }
    uint32_t route = (info >> 8) & 0xFF;
    if (route == ROUTE_VARIABLE) route = (fl & LF_VARFN) ? ROUTE_SCOPE : 10;
    if (route == ROUTE_KEYERROR) { diag(li, S_KEYERROR); continue; }
    if (route != ROUTE_SCOPE) {   // ModuleScope.add
      if (route == 3 && mm) { diag(li, S_MM_DUP); continue; }
      if (has_res) {
        if (idset_has(m, m.reg, 0, rid)) { diag(li, S_DUP, rid); continue; }
        if (!idset_add(m, m.reg, 0, rid)) return NONE32;
      }
      if (route == 3) mm = true;
      m.lgrp[li] = route;
      m.loff[li] = bucket[route];
      bucket[route] += words;
      m.lfl[li] |= LF_PLACED;
      continue;
    }
    // BlockScope.add
    if (blk < 0) { diag(li, S_NEED_BLOCK); continue; }
    if (blk_term) { diag(li, S_TERMINATED); continue; }
    if (sp == SP_VARIABLE) {
      if (!(fl & LF_VARFN)) { diag(li, S_VAR_NOTFN); continue; }
      if (blk_nonvar) { diag(li, S_VAR_FIRST); continue; }
    } else if ((info >> 16) & AF_BLOCK_FORBIDDEN) {
      diag(li, S_NOT_BLOCK);
      continue;
    }
    if (has_res) {
      if (idset_has(m, m.reg, 0, rid)) { diag(li, S_DUP, rid); continue; }
      if (!idset_add(m, m.reg, 0, rid)) return NONE32;
    }
    place_fn(li, words);
    if ((info >> 16) & AF_TERMINATOR) { blk_term = true; m.blk[3 * blk + 2] = 1; }
    if (sp != SP_VARIABLE) blk_nonvar = true;
  }
  m.misc[MS_NFN] = nfn;
  m.misc[MS_NBLK] = nblk;
  return ndiag;
}


// Warp-parallel form of the state machine for modules without diagnostics
// (the common case).  Every rule the sequential machine enforces is checked as
// a per-line predicate over prefix scans (function nesting, block membership,
// terminators, parameter placement, one memory model, SSA uniqueness via
// atomic test-and-set on the registry bitmaps); the first violated rule makes
// it return false, and the caller resets and runs the exact sequential
// machine, which produces the diagnostics.  On success the placement (group,
// offset within group) of every line, the bucket sizes and the function
// records equal the sequential machine's.
enum : uint32_t { K_SKIP = 0, K_MOD, K_FUNC, K_PARAM, K_END, K_LABEL, K_BLOCK, K_BLOCKVAR };

__device__ __noinline__ bool state_fast(AsmMod& m, const AsmCtx& X) {
  const Tables& T = X.T;
  const uint32_t lane = lane_id_a();
  const uint32_t below = (1u << lane) - 1;
  uint32_t nF = 0, nE = 0, nMM = 0;          // running counts
  uint32_t last_struct_kind = K_SKIP;         // kind of the previous structural line
  uint32_t last_struct_term = 0;
  uint32_t last_func_line = NONE32, last_label_line = NONE32;
  uint32_t brun = 0;   // lane b < 11: words placed so far in bucket b
  uint32_t P = 0;                             // words of function-group lines so far
  bool ok = true;
  for (uint32_t base = 0; base < m.L && ok; base += 32) {
    const uint32_t li = base + lane;
    uint32_t kind = K_SKIP, words = 0, route = 0, term = 0, rid = 0;
    bool has_res = false, bad = false;
    if (li < m.L) {
      const uint32_t fl = m.lfl[li];
      if (!(fl & (LF_TOKERR | LF_EMPTY))) {
        const uint32_t d = m.ld[li];
        if (d == NONE32 || m.lec[li] != E_OK || (fl & (LF_UNRES | LF_RESOLVE_ERR))) bad = true;
        else {
          const uint32_t sp = T.special(d), info = __ldg(X.A.info + 4 * d);
          rid = m.lrid[li];
          has_res = T.has_result(d);
          words = 1 + m.lnw[li];
          if (sp == SP_LABEL) { kind = K_LABEL; words = 2; has_res = (fl & LF_RESULT) != 0; bad |= !has_res; }
          else if (sp == SP_FUNCTION) kind = K_FUNC;
          else if (sp == SP_FUNCTIONPARAM) kind = K_PARAM;
          else if (sp == SP_FUNCTIONEND) { kind = K_END; words = 0; }
          else {
            route = (info >> 8) & 0xFF;
            if (route == ROUTE_VARIABLE) route = (fl & LF_VARFN) ? ROUTE_SCOPE : 10;
            if (route == ROUTE_KEYERROR) bad = true;
            else if (route != ROUTE_SCOPE) kind = K_MOD;
            else {
              kind = sp == SP_VARIABLE ? K_BLOCKVAR : K_BLOCK;
              if (kind == K_BLOCK && ((info >> 16) & AF_BLOCK_FORBIDDEN)) bad = true;
              term = ((info >> 16) & AF_TERMINATOR) ? 1 : 0;
            }
          }
        }
      }
    }
    // function nesting: F = OpFunction lines <= li, E = OpFunctionEnd lines < li
    const unsigned bF = __ballot_sync(FULLM, kind == K_FUNC), bE = __ballot_sync(FULLM, kind == K_END);
    const uint32_t F = nF + __popc(bF & (below | (1u << lane))), E = nE + __popc(bE & below);
    const bool inside = F > E;
    if (kind == K_FUNC && F - 1 != E) bad = true;                       // previous function not ended
    if ((kind == K_PARAM || kind == K_END || kind == K_LABEL || kind == K_BLOCK || kind == K_BLOCKVAR) && !inside)
      bad = true;
    // previous structural line (function-scope lines) and its kind
    const bool structural = kind == K_FUNC || kind == K_PARAM || kind == K_END || kind == K_LABEL ||
                            kind == K_BLOCK || kind == K_BLOCKVAR;
    const unsigned bS = __ballot_sync(FULLM, structural);
    const unsigned prevS = bS & below;
    const uint32_t my_kind_term = kind | (term << 8);
    uint32_t pk = last_struct_kind, pt = last_struct_term;
    {
      const int src = prevS ? 31 - __clz(prevS) : 0;
      const uint32_t v = __shfl_sync(FULLM, my_kind_term, src);
      if (prevS) { pk = v & 0xFF; pt = v >> 8; }
    }
    const bool open_block = pk == K_LABEL || pk == K_BLOCK || pk == K_BLOCKVAR;
    if ((kind == K_LABEL || kind == K_END) && open_block && !(pk == K_BLOCK && pt)) bad = true;  // unterminated block
    if (kind == K_BLOCK && (!open_block || (pk == K_BLOCK && pt))) bad = true;
    if (kind == K_BLOCKVAR && !(pk == K_LABEL || pk == K_BLOCKVAR)) bad = true;
    // parameters precede all blocks of their function
    const unsigned bL = __ballot_sync(FULLM, kind == K_LABEL), bFn = bF;
    uint32_t lastL = last_label_line, lastF = last_func_line;
    {
      const unsigned pl = bL & below, pf = bFn & (below | (1u << lane));
      if (pl) lastL = base + 31 - __clz(pl);
      if (pf) lastF = base + 31 - __clz(pf);
    }
    if (kind == K_PARAM && lastL != NONE32 && lastF != NONE32 && lastL > lastF) bad = true;
    // one memory model
    const unsigned bMM = __ballot_sync(FULLM, kind == K_MOD && route == 3);
    if (kind == K_MOD && route == 3 && nMM + __popc(bMM & below) > 0) bad = true;
    // SSA registry / labels: atomic test-and-set (any collision -> exact path)
    if (!bad && has_res && kind != K_SKIP) {
      if (rid >= m.RB || rid == 0) bad = true;
      else {
        const uint32_t bit = 1u << (rid & 31);
        if (atomicOr(&m.reg[rid >> 5], bit) & bit) bad = true;
        if (kind == K_LABEL && (atomicOr(&m.lab[rid >> 5], bit) & bit)) bad = true;
      }
    }
    if (__any_sync(FULLM, bad)) { ok = false; break; }
    // placement: buckets
    uint32_t off = 0;
    // one scan per bucket present in this group of lines (usually one or two)
    const bool placed = kind == K_MOD && route < 11;
    for (uint32_t pend = __ballot_sync(FULLM, placed && words); pend;) {
      const uint32_t r = __shfl_sync(FULLM, route, __ffs(pend) - 1);
      const bool mine = placed && route == r;
      const uint32_t v = mine ? words : 0;
      const uint32_t incl = wincl(v);
      const uint32_t base = __shfl_sync(FULLM, brun, r);
      const uint32_t tot = __shfl_sync(FULLM, incl, 31);
      if (mine) off = base + incl - v;
      if (lane == r) brun += tot;
      pend &= ~__ballot_sync(FULLM, mine);
    }
    // placement: function lines, offset from the function's first line
    const bool fline = kind == K_FUNC || kind == K_PARAM || kind == K_LABEL || kind == K_BLOCK || kind == K_BLOCKVAR;
    const uint32_t fv = fline ? words : 0;
    const uint32_t fincl = wincl(fv);
    const uint32_t Pexcl = P + fincl - fv;
    const uint32_t f = F - 1;
    if (kind == K_FUNC) { m.fn[4 * f] = rid; m.fn[4 * f + 1] = 0; m.fn[4 * f + 3] = Pexcl; }
    __syncwarp();
    if (kind == K_LABEL) m.fn[4 * f + 1] |= FN_BLOCKS;   // same value from every lane: benign
    __syncwarp();
    if (fline) off = Pexcl - m.fn[4 * f + 3];
    if (kind == K_END) { m.fn[4 * f + 2] = Pexcl - m.fn[4 * f + 3]; m.fn[4 * f + 1] |= FN_ENDED; }
    if (kind == K_MOD) { m.lgrp[li] = route; m.loff[li] = off; m.lfl[li] |= LF_PLACED; }
    else if (fline) { m.lgrp[li] = 16 + f; m.loff[li] = off; m.lfl[li] |= LF_PLACED; }
    else if (kind == K_END) m.lfl[li] |= LF_DROP;
    if (kind == K_LABEL) m.lnw[li] = 1;
    P += __shfl_sync(FULLM, fincl, 31);
    nF += __popc(bF); nE += __popc(bE); nMM += __popc(bMM);
    if (bS) {
      const uint32_t v = __shfl_sync(FULLM, my_kind_term, 31 - __clz(bS));
      last_struct_kind = v & 0xFF; last_struct_term = v >> 8;
    }
    if (bL) last_label_line = base + 31 - __clz(bL);
    if (bF) last_func_line = base + 31 - __clz(bF);
    __syncwarp();
  }
  if (ok && nF != nE) ok = false;                 // a function without OpFunctionEnd
  if (!ok) return false;
  if (lane < 11) m.misc[MS_BUCKET0 + lane] = brun;
  if (lane == 0) {
    m.misc[MS_NFN] = nF;
    m.misc[MS_NBLK] = 0;                          // every block was checked terminated above
  }
  __syncwarp();
  return true;
}

// reset what state_fast may have touched before the exact machine runs
__device__ __noinline__ void state_reset(AsmMod& m) {
  const uint32_t lane = lane_id_a();
  for (uint32_t k = lane; k < m.RB / 32; k += 32) { m.reg[k] = 0; m.lab[k] = 0; }
  for (uint32_t li = lane; li < m.L; li += 32) m.lfl[li] &= ~(LF_PLACED | LF_DROP);
  if (lane < 11) m.misc[MS_BUCKET0 + lane] = 0;
  if (lane < 2) m.big[lane] = 0;
  __syncwarp();
}

// ============================================================================
// Optional per-phase cycle counters (build with -DSKG_PHASE_TIMING; profiling only)
#ifdef SKG_PHASE_TIMING
__device__ unsigned long long g_asm_phase[16];
#define PHASE_MARK(k)                                                   \
  do {                                                                  \
    __syncwarp();                                                       \
    const long long now_ = clock64();                                   \
    if (lane_id_a() == 0) atomicAdd(&g_asm_phase[k], (unsigned long long)(now_ - ph_t0_)); \
    ph_t0_ = now_;                                                      \
  } while (0)
#define PHASE_START() long long ph_t0_ = clock64()
#else
#define PHASE_MARK(k) do {} while (0)
#define PHASE_START() do {} while (0)
#endif

// ============================================================================
// Module driver
constexpr uint32_t BIG_CAP = 64;

__device__ __forceinline__ uint64_t al16(uint64_t x) { return (x + 15) & ~15ull; }

// reserve output bytes (bump allocator, 16-byte aligned)
__device__ inline uint64_t asm_alloc(const AsmArgs& a, uint64_t bytes, bool& fits) {
  uint64_t off = 0;
  if (lane_id_a() == 0 && bytes) {
    off = atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 4), (unsigned long long)al16(bytes));
    if (off + bytes > a.out_cap) atomicExch(a.counters + 2, 1u);
  }
  off = __shfl_sync(FULLM, off, 0);
  fits = off + bytes <= a.out_cap;
  return off;
}

// status codes (skgpu.h)
enum : int32_t { AST_OK = 0, AST_CODEC = 4, AST_VALUE = 7, AST_OVERFLOW = 8, AST_ASSEMBLY = 9,
                 AST_STRUCTURE = 10, AST_SERIALIZATION = 11, AST_INTERNAL = 99 };

__device__ inline int32_t outcome_status(uint32_t x) {
  switch (x) {
    case X_VERSION: case X_VERSION_LIMIT: case X_VERSION_DEFAULT: case X_RESERVE: return AST_VALUE;
    case X_OVERFLOW: return AST_OVERFLOW;
    case X_ASSEMBLY: return AST_ASSEMBLY;
    case X_STRUCT_END: case X_STRUCT_TERM: return AST_STRUCTURE;
    case X_SERIAL: return AST_SERIALIZATION;
    case X_WC: return AST_CODEC;
    default: return AST_INTERNAL;
  }
}

__device__ __noinline__ void finish_error(const AsmArgs& a, AsmMod& m, const AsmCtx& X, uint32_t t, uint32_t x,
                                          uint32_t ndiag, uint32_t* fscratch, uint32_t flimbs) {
  const uint32_t lane = lane_id_a();
  FmtCtx F{m, X, X.T.blob + __ldg(X.T.blob + 52), fscratch, flimbs};
  uint32_t n = 0;
  if (lane == 0) {
    Sink cnt;
    if (x == X_INTERNAL) put_cstr(cnt, "internal: module exceeds the per-warp assembler scratch");
    else put_module_error(cnt, F, x, ndiag);
    n = cnt.n;
  }
  n = __shfl_sync(FULLM, n, 0);
  bool fits;
  const uint64_t off = asm_alloc(a, n, fits);
  if (lane == 0) {
    if (fits) {
      Sink w(a.out + off);
      if (x == X_INTERNAL) put_cstr(w, "internal: module exceeds the per-warp assembler scratch");
      else put_module_error(w, F, x, ndiag);
    }
    a.out_span[2 * t] = (int64_t)off;
    a.out_span[2 * t + 1] = (int64_t)n;
    a.status[t] = outcome_status(x);
  }
  __syncwarp();
}

// All warps of the CTA run this together, one module per warp, with a CTA
// barrier between phases: every warp of an SM then executes the same phase's
// code at the same time, which keeps the instruction working set to one phase
// (the per-warp independent schedule thrashed the instruction cache).  A warp
// whose module is finished (error exit) or absent (t >= n_mod) idles through
// the remaining phases.
#define CTA_SYNC() group_sync(gid, gw)
// Line order grouped by instruction (counting sort over a hash of the
// instruction index; order within a bucket is arbitrary): perm[0..L).
constexpr uint32_t OPG_BUCKETS = 64;
template <class K>
__device__ __forceinline__ void group_lines(AsmMod& m, uint32_t* perm, K&& key) {
  const uint32_t lane = lane_id_a();
  const uint32_t L = m.L;
  uint32_t* cnt = perm + L;
  uint32_t* cur = cnt + OPG_BUCKETS;
  for (uint32_t b = lane; b < OPG_BUCKETS; b += 32) cnt[b] = 0;
  __syncwarp();
  for (uint32_t li = lane; li < L; li += 32) atomicAdd(&cnt[key(li)], 1u);
  __syncwarp();
  const uint32_t c0 = __ldcg(cnt + lane), c1 = __ldcg(cnt + 32 + lane);
  const uint32_t i0 = wincl(c0);
  const uint32_t t0 = __shfl_sync(FULLM, i0, 31);
  const uint32_t i1 = wincl(c1);
  cur[lane] = i0 - c0;
  cur[32 + lane] = t0 + i1 - c1;
  __syncwarp();
  for (uint32_t li = lane; li < L; li += 32) perm[atomicAdd(&cur[key(li)], 1u)] = li;
  __syncwarp();
}

__device__ __noinline__ void group_lines_by_opcode(AsmMod& m, uint32_t* perm) {
  group_lines(m, perm, [&](uint32_t li) -> uint32_t {
    const uint32_t d = (m.lfl[li] & (LF_TOKERR | LF_EMPTY)) ? 0xFFFFu : m.ld[li];
    return (d * 0x9E3779B1u) >> 26;
  });
}

__device__ __noinline__ void assemble_module(const AsmArgs& a, const AsmCtx& X, uint32_t t, uint8_t* slot,
                                             uint32_t gid, uint32_t gw, AsmMod& m, AsmMod* all, CtaSort& cs) {
  const uint32_t lane = lane_id_a();
  PHASE_START();
  bool done = t >= a.n_mod;
  const int64_t len64 = done ? 0 : a.mod_len[(size_t)t * a.mod_stride];
  const uint8_t* src = done ? a.text : a.text + a.mod_off[(size_t)t * a.mod_stride];
  m = AsmMod{};   // every lane writes the same (zero) values
  uint64_t used = 0;
  auto take = [&](uint64_t bytes) -> uint8_t* { uint8_t* r = slot + used; used += al16(bytes); return r; };
  uint32_t* fscratch = nullptr;
  uint32_t flimbs = 0;
  auto fail_internal = [&]() { finish_error(a, m, X, t, X_INTERNAL, 0, nullptr, 0); };
  const uint32_t T = (uint32_t)len64;
  uint32_t L = 0, npct = 0, x = X_NONE, ndiag = 0, total = 0, ntb0 = 0;
  uint32_t* lperm = nullptr;
  bool fits = false;
  uint64_t off = 0;
  uint32_t* ow = nullptr;
  if (done) goto end_a;
  m.T = T;
  m.misc = reinterpret_cast<uint32_t*>(take(64 * 4));
  m.txt = src;
  m.esc = take((uint64_t)T + 16);   // touched only by strings with escapes
  m.ls = reinterpret_cast<uint32_t*>(take(4ull * (T + 2)));
  m.le = reinterpret_cast<uint32_t*>(take(4ull * (T + 2)));
  m.lt0 = reinterpret_cast<uint32_t*>(take(4ull * (T + 2)));
  if (used > a.gslot_bytes || len64 < 0 || len64 > 0x3FFFFFFF) { fail_internal(); done = true; goto end_a; }
  for (uint32_t k = lane; k < 64; k += 32) m.misc[k] = 0;
  __syncwarp();
#ifndef SKG_EXP_NO_PREFETCH
  prefetch_l2(src, T);
#endif
  L = split_lines(m, src, T + 1, m.lt0, ntb0);
  m.L = L;
end_a:
  PHASE_MARK(0);
  CTA_SYNC();
  {
  bool bready = false;
  if (!done) {
  // per-line arrays (lt0: token-slot bases from split_lines)
  m.lnt = reinterpret_cast<uint32_t*>(take(4ull * L));
  m.lfl = reinterpret_cast<uint32_t*>(take(4ull * L));
  m.ld = reinterpret_cast<uint32_t*>(take(4ull * L));
  m.lec = reinterpret_cast<uint32_t*>(take(4ull * L));
  m.lnw = reinterpret_cast<uint32_t*>(take(4ull * L));
  m.lrid = reinterpret_cast<uint32_t*>(take(4ull * L));
  m.lgrp = reinterpret_cast<uint32_t*>(take(4ull * L));
  m.loff = reinterpret_cast<uint32_t*>(take(4ull * L));
  m.lerr = reinterpret_cast<uint32_t*>(take(16ull * L));
  lperm = reinterpret_cast<uint32_t*>(take(4ull * L + 4 * 2 * OPG_BUCKETS));
  const uint32_t ntb = ntb0;   // token slots: candidate bound (split_lines)
  m.ntb = ntb;
  m.tok = reinterpret_cast<uint32_t*>(take(8ull * ntb + 8));
  m.tid = reinterpret_cast<uint32_t*>(take(4ull * ntb + 4));
  m.RB = (ntb + 64 + 31) & ~31u;   // ids to select among: <= tokens + reserved
  m.rbm = reinterpret_cast<uint32_t*>(take(m.RB / 8));
  m.zpre = reinterpret_cast<uint32_t*>(take(m.RB / 8 + 4));
  m.reg = reinterpret_cast<uint32_t*>(take(m.RB / 8));
  m.lab = reinterpret_cast<uint32_t*>(take(m.RB / 8));
  m.fn = reinterpret_cast<uint32_t*>(take(16ull * L + 16));
  m.blk = reinterpret_cast<uint32_t*>(take(12ull * L + 16));
  m.big_cap = BIG_CAP;
  m.big = reinterpret_cast<uint32_t*>(take(4ull * (2 + 2 * BIG_CAP)));
  if (used > a.gslot_bytes || L >= (1u << 27)) {
    fail_internal();
    done = true;
  } else {
    for (uint32_t k = lane; k < m.RB / 32; k += 32) { m.rbm[k] = 0; m.reg[k] = 0; m.lab[k] = 0; }
    if (lane < 2) m.big[lane] = 0;
    __syncwarp();
    if (lane == 0) m.rbm[0] = 1;   // id 0 is never allocated
    __syncwarp();
    bready = true;
  }
  }

  PHASE_MARK(1);
  // -- B: tokenize + reservations ------------------------------------------------
  uint32_t nres = 0;
  // (lane per line within the module: a cross-module assignment of the lines measured
  //  5% slower unsorted and 10% sorted by length on the bench batch -- the module's text
  //  and token arrays stay in L1 when one warp tokenizes them)
  if (bready) {
    for (uint32_t base = 0; base < L; base += 32) {
      const uint32_t li = base + lane;
      if (li < L) {
        m.lec[li] = E_OK;
        const uint32_t cap = (li + 1 < L ? m.lt0[li + 1] : m.ntb) - m.lt0[li];
        tokenize_line(m, X, li, m.lt0[li], cap, npct);
        nres += (m.lfl[li] & LF_RESULT) ? 1 : 0;
      }
    }
    npct = wsum(npct);
    nres = wsum(nres);
  }
  if (bready) {
  m.ncap = 32;   // result names at load <= 2/3 (+ unresolved operand names: lane 0 grows the table)
  while (2 * m.ncap < 3 * nres + 48) m.ncap <<= 1;
  if (lane == 0) m.misc[MS_NTCOUNT] = nres;
  m.nt = reinterpret_cast<uint32_t*>(take(4ull * NT_W * m.ncap));
  // formatting scratch (lane 0, error paths): big integers of the longest token
  flimbs = T / 2 + 64;
  fscratch = reinterpret_cast<uint32_t*>(take(4ull * flimbs));
  m.sbase = slot; m.sused = used; m.scap = a.gslot_bytes;
  if (used > a.gslot_bytes) {
    fail_internal();
    done = true;
  } else {
    for (uint32_t k = lane; k < m.ncap; k += 32) {
      uint32_t* e = m.nt + NT_W * k;
      e[0] = EMPTYK; e[1] = 0; e[2] = NONE32; e[3] = 0; e[4] = 0; e[5] = 0;
    }
    __syncwarp();
  }
  }
  }
  PHASE_MARK(2);
  CTA_SYNC();
  if (done) goto end_c;
  // -- C: header comments; then the first reservation failure --------------------
  x = scan_header(m, X, a.default_version);
  if (x != X_NONE) { finish_error(a, m, X, t, x, 0, fscratch, flimbs); done = true; goto end_c; }
  for (uint32_t base = 0; base < L; base += 32) {
    const uint32_t li = base + lane;
    const unsigned bad = __ballot_sync(FULLM, li < L && (m.lfl[li] & LF_RESVERR));
    if (bad) {
      if (lane == 0) m.misc[MS_RESV_LINE] = base + __ffs(bad) - 1;
      __syncwarp();
      finish_error(a, m, X, t, X_RESERVE, 0, fscratch, flimbs);
      done = true;
      goto end_c;
    }
  }
end_c:
  PHASE_MARK(3);
  CTA_SYNC();
  if (done) goto end_d;
  // -- D: unreserved prefix counts; symbolic result names in document order -------
  {
    uint32_t carry = 0;
    const uint32_t nw = m.RB / 32;
    for (uint32_t base = 0; base < nw; base += 32) {
      const uint32_t w = base + lane;
      const uint32_t z = w < nw ? 32 - __popc(m.rbm[w]) : 0;
      const uint32_t incl = wincl(z);
      if (w < nw) m.zpre[w] = carry + incl - z;
      carry += __shfl_sync(FULLM, incl, 31);
    }
  }
  for (uint32_t base = 0; base < L; base += 32) {
    const uint32_t li = base + lane;
    if (li < L && (m.lfl[li] & LF_RESULT)) {
      const uint32_t rt = m.lt0[li];
      const Tok k = tok_at(m, rt);
      const uint32_t e = nt_insert(m, rt);
      m.lgrp[li] = e;   // the line's result entry, for the binding pass and phase E (lgrp is free until G)
      if (!py_isdigit(k.p + 1, k.n - 1, X.U)) {
        if (k.n == 1) m.lfl[li] |= LF_RESOLVE_ERR;
        else if (e != NONE32) atomicMin(&m.nt[NT_W * e + 2], li);
      }
    }
  }
  __syncwarp();
  {
    uint32_t carry = 0;
    for (uint32_t base = 0; base < L; base += 32) {
      const uint32_t li = base + lane;
      uint32_t e = NONE32;
      bool first = false;
      if (li < L && (m.lfl[li] & LF_RESULT) && !(m.lfl[li] & LF_RESOLVE_ERR)) {
        const Tok k = tok_at(m, m.lt0[li]);
        if (!py_isdigit(k.p + 1, k.n - 1, X.U)) {
          e = m.lgrp[li];
          first = e != NONE32 && m.nt[NT_W * e + 2] == li;
        }
      }
      const unsigned b = __ballot_sync(FULLM, first);
      if (first) m.nt[NT_W * e + 3] = select_unreserved(m, carry + __popc(b & ((1u << lane) - 1)) + 1);
      carry += __popc(b);
    }
    if (lane == 0) m.misc[MS_NEWCOUNT] = carry;
  }
  __syncwarp();
  // every %name token resolved once, token-parallel (load-balanced across lanes)
  for (uint32_t k = lane; k < m.ntb; k += 32) {
    const Tok tk = tok_at(m, k);
    uint32_t id = 0;
    if (tk.n >= 2 && tk.p[0] == '%') {
      if (!ascii_dec9(tk.p + 1, tk.n - 1, id)) {
        id = 0;
        if (py_isdigit(tk.p + 1, tk.n - 1, X.U)) {
          const IntVal v = parse_int(tk.p + 1, tk.n - 1, 10, X.U);
          if (v.status == INT_OK && !v.big && v.mag && v.mag <= MAX_ID) id = (uint32_t)v.mag;
        } else {
          const uint32_t e = nt_find(m, tk.p, tk.n);
          if (e != NONE32) id = m.nt[NT_W * e + 3];
        }
      }
    }
    m.tid[k] = id;
  }
end_d:
  PHASE_MARK(4);
  CTA_SYNC();
  // -- E: opname lookup, width / value-type scans ---------------------------------
  {
    auto e_line = [&](AsmMod& mm, uint32_t li) {
      const uint32_t fl = mm.lfl[li];
      const bool res = fl & LF_RESULT;
      const Tok on = tok_at(mm, mm.lt0[li] + (res ? 2 : 0));
      const uint32_t d = inst_by_name(X, on.p, on.n);
      mm.ld[li] = d;
      if (!res || mm.lnt[li] < 4) return;
      const uint32_t e = mm.lgrp[li];   // the result token's entry (phase D's insert)
      if (e == NONE32) return;
      const Tok o0 = tok_at(mm, mm.lt0[li] + 3);
      const bool ti = d != NONE32 ? d == X.A.op_typeint : bytes_eq_z(on.p, on.n, "OpTypeInt");
      const bool tf = d != NONE32 ? d == X.A.op_typefloat : bytes_eq_z(on.p, on.n, "OpTypeFloat");
      if (ti || tf) {
        bool ok = parse_int(o0.p, o0.n, 0, X.U).status == INT_OK;
        if (ok && ti) {
          if (mm.lnt[li] < 5) ok = false;
          else { const Tok o1 = tok_at(mm, mm.lt0[li] + 4); ok = parse_int(o1.p, o1.n, 0, X.U).status == INT_OK; }
        }
        if (ok) atomicMax(&mm.nt[NT_W * e + 4], li + 1);
      }
      if (d != NONE32 && X.T.has_rtype(d) && o0.n >= 1 && o0.p[0] == '%') atomicMax(&mm.nt[NT_W * e + 5], li + 1);
    };
    if (gw == (blockDim.x >> 5)) {
      const uint32_t wib = threadIdx.x >> 5;
      uint32_t ne = 0;
      if (!done) {
        for (uint32_t base = 0; base < L; base += 32) {
          const uint32_t li = base + lane;
          bool want = false;
          if (li < L) {
            if (m.lfl[li] & (LF_TOKERR | LF_EMPTY)) m.ld[li] = NONE32;
            else want = true;
          }
          const unsigned bm = __ballot_sync(FULLM, want);
          if (want) lperm[ne + __popc(bm & ((1u << lane) - 1))] = (wib << 27) | li;
          ne += __popc(bm);
        }
      }
      // the sorted share: m.loff (free until phase H)
      cta_dispatch(cs, lperm, m.loff, ne,
                   [&](uint32_t e) {
                     const uint32_t li = e & CTA_ITEM;
                     const Tok on = tok_at(m, m.lt0[li] + ((m.lfl[li] & LF_RESULT) ? 2 : 0));
                     const uint32_t b2 = on.n > 2 ? on.p[2] : 0, b3 = on.n > 3 ? on.p[3] : 0;
                     return ((b2 & 31) << 5 | (b3 & 31)) ^ (min(on.n, 31u) << 5);
                   },
                   [&](uint32_t e) { e_line(all[e >> 27], e & CTA_ITEM); });
    } else if (!done) {
      for (uint32_t base = 0; base < L; base += 32) {
        const uint32_t li = base + lane;
        if (li >= L) continue;
        if (m.lfl[li] & (LF_TOKERR | LF_EMPTY)) { m.ld[li] = NONE32; continue; }
        e_line(m, li);
      }
    }
  }
  if (done) goto end_e;
end_e:
  PHASE_MARK(5);
  CTA_SYNC();
  // -- F: encode pass 1 -------------------------------------------------------------
  // When the barrier group is the whole CTA, the lines of all its modules are encoded
  // together: every warp lists its lines that need the Encoder walk, the CTA sorts
  // them by instruction (shared-memory counting sort), and each warp then encodes 32
  // consecutive lines of that order -- lanes of one warp run the same instruction's
  // walk, mostly for different modules, and warps whose module is finished (or
  // smaller) take their share of the others' lines.  Results go to each line's own
  // module scratch, exactly as in the per-module loop (kept for other group sizes).
  {
    const uint32_t nwb = blockDim.x >> 5, wib = threadIdx.x >> 5;
    const bool fcross = gw == nwb;
    uint32_t nent = 0;
    uint32_t* fin = nullptr;
    uint32_t* fout = nullptr;
    bool local = !fcross;
    if (!done) {   // words of a line are bounded by 2 per token (4 string bytes per word)
      uint32_t carry = 0;
      m.lwo = reinterpret_cast<uint32_t*>(take(4ull * L + 4));
      for (uint32_t base = 0; base < L; base += 32) {
        const uint32_t li = base + lane;
        uint32_t ub = 0;
        if (li < L) {
          ub = 1;
          for (uint32_t k = 0; k < m.lnt[li]; ++k) {
            const uint32_t lf = m.tok[2 * (m.lt0[li] + k) + 1];
            ub += (lf & TK_STR) ? (lf & TK_LEN) / 4 + 1 : 2;
          }
        }
        const uint32_t incl = wincl(ub);
        if (li < L) m.lwo[li] = carry + incl - ub;
        carry += __shfl_sync(FULLM, incl, 31);
      }
      m.sw = reinterpret_cast<uint32_t*>(take(4ull * carry + 4));
      m.swr = reinterpret_cast<uint32_t*>(take(carry / 8 + 8));
      if (used > a.gslot_bytes) {
        fail_internal();
        done = true;
      } else {
        m.sused = used;
        for (uint32_t k = lane; k <= carry / 32; k += 32) m.swr[k] = 0;
        if (fcross) {   // the line lists (input, sorted share) fit the slot, else this module stays local
          const uint64_t used0 = used;
          fin = reinterpret_cast<uint32_t*>(take(4ull * L + 16));
          fout = reinterpret_cast<uint32_t*>(take(4ull * L + 16));
          if (used > a.gslot_bytes || L >= (1u << 27)) { used = used0; local = true; fin = fout = nullptr; }
          m.sused = used;
        }
        if (fcross && !local) {
          for (uint32_t base = 0; base < L; base += 32) {
            const uint32_t li = base + lane;
            bool enc = false;
            uint32_t d = NONE32;
            if (li < L) {
              const uint32_t fl = m.lfl[li];
              m.lnw[li] = 0; m.lrid[li] = 0;
              if (!(fl & (LF_TOKERR | LF_EMPTY))) {
                d = m.ld[li];
                if (d == NONE32) m.lec[li] = E_NOINST;
                else if (X.T.special(d) == SP_LABEL) {
                  if ((fl & LF_RESULT) && !(fl & LF_RESOLVE_ERR)) m.lrid[li] = result_id_of(m, X, m.lt0[li]);
                } else {
                  enc = true;
                }
              }
            }
            const unsigned bm = __ballot_sync(FULLM, enc);
            if (enc) {
              fin[nent + __popc(bm & ((1u << lane) - 1))] = (wib << 27) | li;
            }
            nent += __popc(bm);
          }
        } else {
          group_lines_by_opcode(m, lperm);
        }
      }
    }
    if (fcross) {
      cta_dispatch(cs, fin, fout, nent,
                   [&](uint32_t e) { return m.ld[e & CTA_ITEM]; },   // own entries only
                   [&](uint32_t e) {
                     const AsmMod& mm = all[e >> 27];
                     const uint32_t li = e & CTA_ITEM;
                     const uint32_t w0 = mm.lwo[li] + 1;
                     encode_line(mm, X, li, mm.ld[li], M_COUNT, mm.sw + w0, mm.swr, w0, nullptr);
                   });
    }
    if (!done && local) {
      // lanes take lines grouped by instruction (one code path per group instead of
      // the union of 32 different encoders); results are stored per line
      for (uint32_t base = 0; base < L; base += 32) {
        if (base + lane >= L) continue;
        const uint32_t li = lperm[base + lane];
        const uint32_t fl = m.lfl[li];
        m.lnw[li] = 0; m.lrid[li] = 0;
        if (fl & (LF_TOKERR | LF_EMPTY)) continue;
        const uint32_t d = m.ld[li];
        if (d == NONE32) { m.lec[li] = E_NOINST; continue; }
        if (X.T.special(d) == SP_LABEL) {
          if ((fl & LF_RESULT) && !(fl & LF_RESOLVE_ERR)) m.lrid[li] = result_id_of(m, X, m.lt0[li]);
          continue;
        }
        const uint32_t w0 = m.lwo[li] + 1;
        encode_line(m, X, li, d, M_COUNT, m.sw + w0, m.swr, w0, nullptr);
      }
    }
  }
  if (done) goto end_f;
  __syncwarp();
  // first OverflowError (escapes the emit loop's except clause)
  for (uint32_t base = 0; base < L; base += 32) {
    const uint32_t li = base + lane;
    const unsigned b = __ballot_sync(FULLM, li < L && !(m.lfl[li] & (LF_TOKERR | LF_EMPTY)) &&
                                                (m.lec[li] == E_OVF_E || m.lec[li] == E_OVF_F));
    if (b) {
      if (lane == 0) m.misc[MS_OVF_LINE] = base + __ffs(b) - 1;
      __syncwarp();
      finish_error(a, m, X, t, X_OVERFLOW, 0, fscratch, flimbs);
      done = true;
      goto end_f;
    }
  }
end_f:
  PHASE_MARK(6);
  CTA_SYNC();
  if (done) goto end_g;
  // -- G: state machine ------------------------------------------------------------
  if (state_fast(m, X)) {
    ndiag = 0;
  } else {
    state_reset(m);
    if (lane == 0) ndiag = state_machine(m, X);
    __syncwarp();   // lane 0 may have grown the name table (m.nt / m.ncap, shared by the warp)
  }
  if (lane == 0 && ndiag != NONE32) {
    for (uint32_t li = 0; li < L; ++li) {
      const uint32_t fl = m.lfl[li];
      ndiag += (fl & LF_TOKERR) ? 1 : 0;
      ndiag += (fl & LF_RESOLVE_ERR) ? 1 : 0;
    }
  }
  ndiag = __shfl_sync(FULLM, ndiag, 0);
  if (ndiag == NONE32) { fail_internal(); done = true; goto end_g; }
  if (ndiag) { finish_error(a, m, X, t, X_ASSEMBLY, ndiag, fscratch, flimbs); done = true; goto end_g; }
end_g:
  PHASE_MARK(7);
  CTA_SYNC();
  if (done) goto end_h;
  // -- H: structure checks + layout (lane 0) ----------------------------------------
  if (lane == 0) {
    const uint32_t nfn = m.misc[MS_NFN], nblk = m.misc[MS_NBLK];
    uint32_t bi = 0;
    x = X_NONE;
    for (uint32_t f = 0; f < nfn && x == X_NONE; ++f) {
      if (!(m.fn[4 * f + 1] & FN_ENDED)) { x = X_STRUCT_END; m.misc[MS_XA] = m.fn[4 * f]; break; }
      for (; bi < nblk && m.blk[3 * bi] == f; ++bi) {
        if (!m.blk[3 * bi + 2]) {
          x = X_STRUCT_TERM; m.misc[MS_XA] = m.fn[4 * f]; m.misc[MS_XB] = m.blk[3 * bi + 1];
          break;
        }
      }
    }
    uint32_t pos = 5;
    for (uint32_t b = 0; b < 11; ++b) {
      const uint32_t sz = m.misc[MS_BUCKET0 + b];
      m.misc[MS_BUCKET0 + b] = pos;
      pos += sz;
    }
    for (int pass = 0; pass < 2; ++pass)
      for (uint32_t f = 0; f < nfn; ++f) {
        const bool has_blocks = m.fn[4 * f + 1] & FN_BLOCKS;
        if (has_blocks != (pass == 1)) continue;
        m.fn[4 * f + 3] = pos;
        pos += m.fn[4 * f + 2] + 1;
      }
    m.misc[MS_TOTAL] = pos;
  }
  x = __shfl_sync(FULLM, x, 0);
  if (x != X_NONE) { finish_error(a, m, X, t, x, 0, fscratch, flimbs); done = true; goto end_h; }
  __syncwarp();
  total = m.misc[MS_TOTAL];
end_h:
  PHASE_MARK(8);
  CTA_SYNC();
  if (done) goto end_i;
  {
  // -- I: output ---------------------------------------------------------------------
  off = asm_alloc(a, 4ull * total, fits);
  ow = reinterpret_cast<uint32_t*>(a.out + off);
  if (fits && lane == 0) {
    ow[0] = 0x07230203u;
    ow[1] = (m.misc[MS_MAJOR] << 16) | ((m.misc[MS_MINOR] - 1) << 8);
    ow[2] = m.misc[MS_GENSET] ? m.misc[MS_GEN] : (32u << 16);
    ow[4] = m.misc[MS_SCHEMA];
  }
  if (lane == 0) {   // bound = max(counter, max reserved) + 1
    const uint32_t nnew = m.misc[MS_NEWCOUNT];
    uint32_t mx = nnew ? select_unreserved(m, nnew) : 0;
    mx = max(mx, m.misc[MS_BIGMAX_LO]);
    for (int w = (int)m.RB / 32 - 1; w >= 0; --w) {
      const uint32_t bits = m.rbm[w] & (w == 0 ? ~1u : ~0u);
      if (bits) { mx = max(mx, (uint32_t)w * 32 + 31 - __clz(bits)); break; }
    }
    if (fits) ow[3] = mx + 1;
  }
  // function ends
  {
    const uint32_t nfn = m.misc[MS_NFN];
    const uint32_t endw = (1u << 16) | __ldg(X.T.irec(X.A.op_fnend) + 5);
    for (uint32_t f = lane; f < nfn; f += 32)
      if (fits) ow[m.fn[4 * f + 3] + m.fn[4 * f + 2]] = endw;
  }
  uint32_t ser_off = NONE32, wc_off = NONE32;
  const uint32_t label_word = (2u << 16) | __ldg(X.T.irec(X.A.op_label) + 5);
  for (uint32_t base = 0; base < L; base += 32) {
    const uint32_t li = base + lane;
    if (li >= L || !(m.lfl[li] & LF_PLACED)) continue;
    const uint32_t g = m.lgrp[li];
    const uint32_t at = m.loff[li] + (g < 16 ? m.misc[MS_BUCKET0 + g] : m.fn[4 * (g - 16) + 3]);
    m.loff[li] = at;
    const uint32_t d = m.ld[li];
    if (X.T.special(d) == SP_LABEL) {
      if (fits) { ow[at] = label_word; ow[at + 1] = m.lrid[li]; }
      continue;
    }
    if (1 + m.lnw[li] > 0xFFFF) wc_off = min(wc_off, at);
    uint32_t bad_ref = NONE32;
    if (m.lfl[li] & LF_UNRES) {   // ids of names first seen in the state machine: re-encode
      EncOut r;   // M_WRITE also checks references
      encode_line(m, X, li, d, M_WRITE, fits ? ow + at + 1 : nullptr, nullptr, 0, &r);
      bad_ref = r.bad_ref;
    } else {                      // copy pass-1 words; check the referenced ids
      const uint32_t w0 = m.lwo[li] + 1, nw = m.lnw[li];
      for (uint32_t k = 0; k < nw; ++k) {
        const uint32_t w = m.sw[w0 + k];
        if (fits) ow[at + 1 + k] = w;
        const uint32_t b = w0 + k;
        if (bad_ref == NONE32 && ((m.swr[b >> 5] >> (b & 31)) & 1) && !idset_has(m, m.reg, 0, w)) bad_ref = w;
      }
    }
    if (fits) ow[at] = ((1 + m.lnw[li]) << 16) | __ldg(X.T.irec(d) + 5);
    if (bad_ref != NONE32) { m.lerr[4 * li + 3] = bad_ref; ser_off = min(ser_off, at); }
  }
  ser_off = wmin(ser_off);
  wc_off = wmin(wc_off);
  if (ser_off != NONE32 || wc_off != NONE32) {
    const uint32_t target = ser_off != NONE32 ? ser_off : wc_off;
    for (uint32_t base = 0; base < L; base += 32) {
      const uint32_t li = base + lane;
      const bool hit = li < L && (m.lfl[li] & LF_PLACED) && m.loff[li] == target;
      if (hit) {
        if (ser_off != NONE32) { m.misc[MS_XA] = m.lerr[4 * li + 3]; m.misc[MS_XB] = m.ld[li]; }
        else m.misc[MS_XA] = 1 + m.lnw[li];
      }
    }
    __syncwarp();
    finish_error(a, m, X, t, ser_off != NONE32 ? X_SERIAL : X_WC, 0, fscratch, flimbs);
    done = true;
    goto end_i;
  }
  }
  if (lane == 0) {
    a.out_span[2 * t] = (int64_t)off;
    a.out_span[2 * t + 1] = (int64_t)(4ull * total);
    a.status[t] = AST_OK;
  }
end_i:
  PHASE_MARK(9);
  CTA_SYNC();
}

#ifndef SKG_ASM_MAXT
#define SKG_ASM_MAXT 1024
#define SKG_ASM_MINB 1
#endif
__global__ void __launch_bounds__(SKG_ASM_MAXT, SKG_ASM_MINB) asm_kernel(const __grid_constant__ AsmArgs a) {
  __shared__ uint32_t s_base[16];
  __shared__ AsmMod s_amod[32];   // the module descriptor, one per warp (not a per-thread local copy)
  __shared__ CtaSort s_cs;        // cross-module work assignment (phases B, F)
  const uint32_t warps = blockDim.x >> 5;
  const uint32_t warp_in_block = threadIdx.x >> 5;
  const uint32_t gw = a.group_warps;                 // warps per barrier group
  const uint32_t gid = warp_in_block / gw, gwarp_in = warp_in_block % gw;
  const uint32_t gwarp = blockIdx.x * warps + warp_in_block;
  uint8_t* slot = a.gscratch + (size_t)gwarp * a.gslot_bytes;
  __shared__ AsmCtx s_ctx;
  __shared__ AsmArgs s_args;   // one copy per CTA: field reads are shared loads
  if (threadIdx.x == 0) { s_ctx.T = a.T; s_ctx.U = a.U; s_ctx.A = a.A; s_args = a; }
  __syncthreads();
  const AsmCtx& X = s_ctx;
  while (true) {
    if (gwarp_in == 0 && (threadIdx.x & 31) == 0) s_base[gid] = atomicAdd(a.counters, gw);
    group_sync(gid, gw);
    const uint32_t base = s_base[gid];
    group_sync(gid, gw);
    if (base >= a.n_mod) break;
    const uint32_t tk = base + gwarp_in;
    assemble_module(s_args, X, tk < a.n_mod ? a.order[tk] : a.n_mod, slot, gid, gw, s_amod[warp_in_block], s_amod, s_cs);
  }
}

}  // namespace skg
