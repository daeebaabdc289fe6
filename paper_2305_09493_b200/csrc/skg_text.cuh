// Text-side primitives of the assembler: the CPython string and number
// semantics that reference asm.py inherits from the interpreter.
//
//  * Unicode predicates the reference reaches through str methods and re:
//    str.isprintable (repr), str.isspace (strip, re \s), str.isdecimal
//    (int()/float() digit transform, re \d) and str.isdigit (asm.py:113) --
//    code-point tables generated from the same CPython (tables.py).
//  * repr(str), including the %.200R truncation of int()'s error message.
//  * int(text, 0) / int(text) (Objects/longobject.c PyLong_FromString: digit
//    transform, prefixes, underscores, the 4300-digit limit).
//  * float(text) (Objects/floatobject.c + Python/pystrtod.c): syntax, then a
//    correctly rounded decimal -> double (Clinger fast path, Eisel-Lemire with
//    128-bit powers of five, big-integer comparison fallback).
//  * struct.pack('<e' / '<f') with CPython's rounding and OverflowError
//    (PyFloat_Pack2 / PyFloat_Pack4), used by codec.encode_context_dependent_literal
//    (codec.py:132-168).
//
// Everything is __host__ __device__ so tests/native/text_check.cpp can run the
// exact same code on the host against CPython.
#pragma once
#include "skg_fmt.cuh"
#include "skg_pow5_parse.cuh"
#include <cstring>

namespace skg {

SKG_HD inline uint32_t ldg32(const uint32_t* p) {
#if defined(__CUDA_ARCH__)
  return __ldg(p);
#else
  return *p;
#endif
}

struct Uni {
  const uint32_t* printable; uint32_t n_printable;   // [lo, hi) pairs, sorted
  const uint32_t* space; uint32_t n_space;           // sorted code points
  const uint32_t* dec; uint32_t n_dec;               // starts of 10-digit runs, sorted
  const uint32_t* digit; uint32_t n_digit;           // isdigit() but not isdecimal(), sorted

  // ASCII answers inline; the table searches are out of line (one copy of code)
  SKG_HD bool is_space(uint32_t c) const {
    if (c < 0x80) return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1C && c <= 0x1F);
    return is_space_slow(c);
  }
  SKG_HD int decimal(uint32_t c) const {   // decimal value 0..9 or -1 (str.isdecimal)
    if (c < 0x80) return (c >= '0' && c <= '9') ? (int)(c - '0') : -1;
    return decimal_slow(c);
  }
  SKG_HD bool is_digit(uint32_t c) const {
    if (c < 0x80) return c >= '0' && c <= '9';
    return is_digit_slow(c);
  }
  SKG_HD bool is_printable(uint32_t c) const {
    if (c >= 0x20 && c < 0x7F) return true;
    if (c < 0xA0) return false;
    return is_printable_slow(c);
  }
  SKG_HD SKG_NOINLINE bool is_space_slow(uint32_t c) const {
    for (uint32_t i = 0; i < n_space; ++i) if (ldg32(space + i) == c) return true;
    return false;
  }
  SKG_HD SKG_NOINLINE int decimal_slow(uint32_t c) const {
    uint32_t lo = 0, hi = n_dec;
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      if (ldg32(dec + mid) <= c) lo = mid + 1; else hi = mid;
    }
    if (lo == 0) return -1;
    uint32_t s = ldg32(dec + lo - 1);
    return c - s < 10 ? (int)(c - s) : -1;
  }
  SKG_HD SKG_NOINLINE bool is_digit_slow(uint32_t c) const {
    if (decimal_slow(c) >= 0) return true;
    uint32_t lo = 0, hi = n_digit;
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      uint32_t v = ldg32(digit + mid);
      if (v == c) return true;
      if (v < c) lo = mid + 1; else hi = mid;
    }
    return false;
  }
  SKG_HD SKG_NOINLINE bool is_printable_slow(uint32_t c) const {
    uint32_t lo = 0, hi = n_printable;
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      if (ldg32(printable + 2 * mid) <= c) lo = mid + 1; else hi = mid;
    }
    return lo > 0 && c < ldg32(printable + 2 * (lo - 1) + 1);
  }
};

SKG_HD SKG_NOINLINE uint32_t utf8_cp_multi(const uint8_t* p, uint32_t n, uint32_t i, uint32_t& len);

// One code point of (valid, surrogatepass) UTF-8 at p[i]; sets its byte length.
SKG_HD inline uint32_t utf8_cp(const uint8_t* p, uint32_t n, uint32_t i, uint32_t& len) {
  const uint32_t c = p[i];
  if (c < 0x80) { len = 1; return c; }
  return utf8_cp_multi(p, n, i, len);
}

SKG_HD SKG_NOINLINE uint32_t utf8_cp_multi(const uint8_t* p, uint32_t n, uint32_t i, uint32_t& len) {
  uint32_t c = p[i];
  if (c < 0x80 || i + 1 >= n) { len = 1; return c; }
  if (c < 0xE0) { len = 2; return ((c & 0x1F) << 6) | (p[i + 1] & 0x3F); }
  if (c < 0xF0 || i + 3 > n) {
    len = i + 2 < n ? 3 : 2;
    return ((c & 0x0F) << 12) | ((p[i + 1] & 0x3F) << 6) | (len == 3 ? (p[i + 2] & 0x3F) : 0);
  }
  len = i + 3 < n ? 4 : 3;
  return ((c & 0x07) << 18) | ((p[i + 1] & 0x3F) << 12) | ((p[i + 2] & 0x3F) << 6) |
         (len == 4 ? (p[i + 3] & 0x3F) : 0);
}

SKG_HD inline uint32_t cp_count(const uint8_t* p, uint32_t n) {
  uint32_t k = 0;
  for (uint32_t i = 0; i < n; ++i) k += (p[i] & 0xC0) != 0x80;
  return k;
}

// -- repr(str) ------------------------------------------------------------------
// Objects/unicodeobject.c unicode_repr.  `limit` > 0 truncates the produced repr
// to that many code points (PyUnicode_FromFormat "%.200R").
struct ReprLimit {
  uint32_t limit, n = 0;
};

template <class S>
SKG_HD SKG_NOINLINE void put_py_repr_prefixed(S& s, const char* pre, const uint8_t* p, uint32_t n, const Uni& U,
                                          uint32_t limit = 0);

template <class S>
SKG_HD inline void put_py_repr(S& s, const uint8_t* p, uint32_t n, const Uni& U, uint32_t limit = 0) {
  put_py_repr_prefixed(s, "", p, n, U, limit);
}

// repr(pre + text); `pre` is plain ASCII without quotes or backslashes
template <class S>
SKG_HD SKG_NOINLINE void put_py_repr_prefixed(S& s, const char* pre, const uint8_t* p, uint32_t n, const Uni& U,
                                          uint32_t limit) {
  bool has_sq = false, has_dq = false;
  for (uint32_t i = 0; i < n; ++i) { has_sq |= p[i] == '\''; has_dq |= p[i] == '"'; }
  const uint8_t q = (has_sq && !has_dq) ? '"' : '\'';
  uint32_t out = 0;   // code points emitted
  auto emit = [&](uint8_t c) -> bool {
    if (limit && out >= limit) return false;
    s.put(c);
    ++out;
    return true;
  };
  auto emit_hex = [&](uint32_t v, int digits) {
    for (int k = digits - 1; k >= 0; --k) emit((uint8_t)"0123456789abcdef"[(v >> (4 * k)) & 0xF]);
  };
  emit(q);
  for (const char* z = pre; *z; ++z) emit((uint8_t)*z);
  for (uint32_t i = 0; i < n;) {
    if (limit && out >= limit) return;
    uint32_t len;
    const uint32_t c = utf8_cp(p, n, i, len);
    if (c == q || c == '\\') { emit('\\'); emit((uint8_t)c); }
    else if (c == '\t') { emit('\\'); emit('t'); }
    else if (c == '\n') { emit('\\'); emit('n'); }
    else if (c == '\r') { emit('\\'); emit('r'); }
    else if (c < 0x20 || c == 0x7F) { emit('\\'); emit('x'); emit_hex(c, 2); }
    else if (c < 0x7F) emit((uint8_t)c);
    else if (U.is_printable(c)) {
      if (limit && out >= limit) return;
      for (uint32_t k = 0; k < len; ++k) s.put(p[i + k]);
      ++out;
    } else if (c < 0x100) { emit('\\'); emit('x'); emit_hex(c, 2); }
    else if (c < 0x10000) { emit('\\'); emit('u'); emit_hex(c, 4); }
    else { emit('\\'); emit('U'); emit_hex(c, 8); }
    i += len;
  }
  emit(q);
}

// -- int() ----------------------------------------------------------------------
enum : uint32_t { INT_OK = 0, INT_INVALID = 1, INT_LIMIT = 2 };
constexpr uint32_t PY_MAX_STR_DIGITS = 4300;

struct IntVal {
  uint32_t status;
  bool neg;
  bool big;          // |value| >= 2^64
  uint64_t mag;
  uint32_t base;     // digit base actually used (2, 8, 10, 16)
  uint32_t ndig;     // digit characters (4300-digit limit, base 10)
  uint32_t ds, de;   // byte range of the digit run (underscores included)
};

// The interpreter's view of a character in int()/float(): ASCII as is, other
// white space -> ' ', other decimal digits -> '0'..'9', anything else -> '?'
// (_PyUnicode_TransformDecimalAndSpaceToASCII).
SKG_HD SKG_NOINLINE uint32_t xform_multi(const uint8_t* p, uint32_t n, uint32_t i, uint32_t& len, const Uni& U);
SKG_HD inline uint32_t xform(const uint8_t* p, uint32_t n, uint32_t i, uint32_t& len, const Uni& U) {
  if (p[i] < 0x80) { len = 1; return p[i] ? p[i] : '?'; }   // embedded NUL: invalid in both parsers
  return xform_multi(p, n, i, len, U);
}
SKG_HD SKG_NOINLINE uint32_t xform_multi(const uint8_t* p, uint32_t n, uint32_t i, uint32_t& len, const Uni& U) {
  const uint32_t c = utf8_cp(p, n, i, len);
  if (U.is_space(c)) return ' ';
  const int d = U.decimal(c);
  return d >= 0 ? (uint32_t)('0' + d) : '?';
}

SKG_HD inline bool ascii_space(uint32_t c) { return c == ' ' || (c >= 9 && c <= 13); }

SKG_HD inline int digit_value(uint32_t c) {
  if (c >= '0' && c <= '9') return (int)(c - '0');
  if (c >= 'a' && c <= 'z') return (int)(c - 'a' + 10);
  if (c >= 'A' && c <= 'Z') return (int)(c - 'A' + 10);
  return 99;
}

// PyLong_FromString(text, base) for base 0 (int(t, 0)) or 10 (int(t)).
SKG_HD SKG_NOINLINE IntVal parse_int(const uint8_t* p, uint32_t n, uint32_t base, const Uni& U) {
  IntVal r{};
  r.status = INT_INVALID;
  if ((base == 0 || base == 10) && n >= 1 && n <= 19) {   // fast path: [+-]?[1-9][0-9]* | [+-]?0
    const uint32_t s0 = (p[0] == '-' || p[0] == '+') ? 1u : 0u;
    const uint32_t nd = n - s0;
    if (nd >= 1 && nd <= 18 && (p[s0] != '0' || nd == 1)) {
      uint64_t v = 0;
      uint32_t i = s0;
      for (; i < n; ++i) {
        const uint32_t d = (uint32_t)p[i] - '0';
        if (d > 9) break;
        v = v * 10 + d;
      }
      if (i == n) {
        r.status = INT_OK; r.neg = p[0] == '-'; r.big = false; r.mag = v; r.base = 10;
        r.ndig = nd; r.ds = s0; r.de = n;
        return r;
      }
    }
  }
  uint32_t i = 0, len = 1, c = 0;
  auto peek = [&](uint32_t at, uint32_t& l) -> uint32_t { return at < n ? xform(p, n, at, l, U) : 0u; };
  c = peek(i, len);
  while (i < n && ascii_space(c)) { i += len; c = peek(i, len); }
  if (c == '+' || c == '-') { r.neg = c == '-'; i += len; c = peek(i, len); }
  bool nonzero_is_error = false;
  uint32_t l2;
  if (base == 0) {
    if (c != '0') base = 10;
    else {
      const uint32_t c2 = peek(i + len, l2);
      if (c2 == 'x' || c2 == 'X') base = 16;
      else if (c2 == 'o' || c2 == 'O') base = 8;
      else if (c2 == 'b' || c2 == 'B') base = 2;
      else { nonzero_is_error = true; base = 10; }
      if (base != 10) {
        i += len + l2;
        c = peek(i, len);
        if (c == '_') { i += len; c = peek(i, len); }
      }
    }
  }
  r.base = base;
  if (c == '_') return r;
  r.ds = i;
  uint32_t prev = 0, nd = 0;
  uint64_t mag = 0;
  bool big = false, any_nonzero = false;
  while (i < n) {
    c = peek(i, len);
    if (c == '_') {
      if (prev == '_') return r;
    } else {
      const int d = digit_value(c);
      if (d >= (int)base) break;
      ++nd;
      any_nonzero |= d != 0;
      if (!big) {
        const uint64_t hi = mag >> 32;
        uint64_t t_hi = hi * base, t_lo = (mag & 0xFFFFFFFFull) * base + (uint64_t)d;
        t_hi += t_lo >> 32;
        if (t_hi >> 32) big = true;
        else mag = (t_hi << 32) | (t_lo & 0xFFFFFFFFull);
      }
    }
    prev = c;
    i += len;
  }
  r.de = i;
  if (prev == '_' || nd == 0) return r;
  c = peek(i, len);
  while (i < n && ascii_space(c)) { i += len; c = peek(i, len); }
  if (i < n) return r;
  r.ndig = nd;
  if (base == 10 && nd > PY_MAX_STR_DIGITS) { r.status = INT_LIMIT; return r; }
  if (nonzero_is_error && any_nonzero) return r;
  r.status = INT_OK;
  r.big = big;
  r.mag = big ? 0 : mag;
  return r;
}

// -- big integers (message formatting of out-of-range values, float fallback) -----
// Little-endian base-2^32 limbs; capacity supplied by the caller.
struct Big {
  uint32_t* d;
  uint32_t n;     // used limbs
  uint32_t cap;
  bool ovf = false;
  SKG_HD void set_small(uint64_t v) {
    n = 0;
    if (v) { d[n++] = (uint32_t)v; if (v >> 32) d[n++] = (uint32_t)(v >> 32); }
  }
  SKG_HD void mul_add(uint32_t m, uint32_t a) {
    uint64_t carry = a;
    for (uint32_t k = 0; k < n; ++k) {
      const uint64_t t = (uint64_t)d[k] * m + carry;
      d[k] = (uint32_t)t;
      carry = t >> 32;
    }
    if (carry) { if (n < cap) d[n++] = (uint32_t)carry; else ovf = true; }
  }
  SKG_HD void shl(uint32_t bits) {
    const uint32_t w = bits / 32, b = bits % 32;
    if (n == 0) return;
    if (n + w + 1 > cap) { ovf = true; return; }
    uint32_t top = 0;
    if (b) top = d[n - 1] >> (32 - b);
    for (int k = (int)n - 1; k >= 0; --k) {
      const uint32_t lo = (b && k > 0) ? (d[k - 1] >> (32 - b)) : 0;
      d[k + w] = (b ? (d[k] << b) : d[k]) | lo;
    }
    for (uint32_t k = 0; k < w; ++k) d[k] = 0;
    n += w;
    if (top) d[n++] = top;
  }
  SKG_HD void mul_pow5(uint32_t e) {
    while (e >= 13) { mul_add(1220703125u, 0); e -= 13; }
    uint32_t m = 1;
    while (e--) m *= 5;
    if (m != 1) mul_add(m, 0);
  }
  // divide in place by v (< 2^32), returns remainder
  SKG_HD uint32_t divmod(uint32_t v) {
    uint64_t rem = 0;
    for (int k = (int)n - 1; k >= 0; --k) {
      const uint64_t cur = (rem << 32) | d[k];
      d[k] = (uint32_t)(cur / v);
      rem = cur % v;
    }
    while (n && d[n - 1] == 0) --n;
    return (uint32_t)rem;
  }
};

SKG_HD inline int big_cmp(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int k = (int)a.n - 1; k >= 0; --k)
    if (a.d[k] != b.d[k]) return a.d[k] < b.d[k] ? -1 : 1;
  return 0;
}

// Load the digits of a validated int() token into `b` (binary value).
SKG_HD inline void big_from_token(Big& b, const uint8_t* p, const IntVal& v, const Uni& U) {
  b.n = 0;
  for (uint32_t i = v.ds; i < v.de;) {
    uint32_t len;
    const uint32_t c = xform(p, v.de, i, len, U);
    i += len;
    if (c == '_') continue;
    b.mul_add(v.base, (uint32_t)digit_value(c));
  }
}

// str(int) of a validated token: decimal with sign; the digits of a base-10
// token are copied (normalised), other bases are converted.  Returns false
// (writes nothing) when CPython's str() would raise the 4300-digit ValueError.
// `scratch` must hold (de - ds) / 2 + 8 limbs.
template <class S>
SKG_HD SKG_NOINLINE bool put_int_decimal(S& s, const uint8_t* p, const IntVal& v, const Uni& U, uint32_t* scratch,
                                     uint32_t scratch_limbs) {
  if (!v.big) {
    if (v.neg && v.mag) s.put('-');
    put_u64(s, v.mag);
    return true;
  }
  if (v.base == 10) {   // > 4300 digits was rejected at parse time
    if (v.neg) s.put('-');
    bool lead = true;
    for (uint32_t i = v.ds; i < v.de;) {
      uint32_t len;
      const uint32_t c = xform(p, v.de, i, len, U);
      i += len;
      if (c == '_' || (lead && c == '0')) continue;
      lead = false;
      s.put((uint8_t)c);
    }
    return true;
  }
  Big b{scratch, 0, scratch_limbs};
  big_from_token(b, p, v, U);
  // decimal digits: chunks of 9 by repeated division
  const uint32_t nchunks_max = b.n * 32 / 29 + 2;
  uint32_t* chunks = scratch + b.n;   // caller sized scratch for 2x limbs
  uint32_t k = 0;
  while (b.n && k < nchunks_max) chunks[k++] = b.divmod(1000000000u);
  // digit count
  uint32_t top = chunks[k - 1], td = 1;
  while (top >= 10) { top /= 10; ++td; }
  if ((k - 1) * 9 + td > PY_MAX_STR_DIGITS) return false;
  if (v.neg) s.put('-');
  put_u64(s, chunks[k - 1]);
  for (int j = (int)k - 2; j >= 0; --j) {
    uint32_t c = chunks[j];
    char buf[9];
    for (int q = 8; q >= 0; --q) { buf[q] = (char)('0' + c % 10); c /= 10; }
    for (int q = 0; q < 9; ++q) s.put((uint8_t)buf[q]);
  }
  return true;
}

// format(value, '#x') of a validated token (-0x... for negatives)
template <class S>
SKG_HD SKG_NOINLINE void put_int_hex(S& s, const uint8_t* p, const IntVal& v, const Uni& U, uint32_t* scratch,
                                 uint32_t scratch_limbs) {
  if (v.neg && (v.big || v.mag)) s.put('-');
  s.put('0'); s.put('x');
  if (!v.big) {
    int sh = 60;
    while (sh > 0 && ((v.mag >> sh) & 0xF) == 0) sh -= 4;
    for (; sh >= 0; sh -= 4) s.put((uint8_t)"0123456789abcdef"[(v.mag >> sh) & 0xF]);
    return;
  }
  Big b{scratch, 0, scratch_limbs};
  big_from_token(b, p, v, U);
  bool lead = true;
  for (int k = (int)b.n - 1; k >= 0; --k)
    for (int sh = 28; sh >= 0; sh -= 4) {
      const uint32_t h = (b.d[k] >> sh) & 0xF;
      if (lead && h == 0) continue;
      lead = false;
      s.put((uint8_t)"0123456789abcdef"[h]);
    }
}

// -- float() --------------------------------------------------------------------
struct Am { uint64_t m; int32_t p2; };   // fast_float adjusted mantissa (biased exponent)

SKG_HD inline int clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
  return __clzll((long long)x);
#else
  return x ? __builtin_clzll(x) : 64;
#endif
}

// Eisel-Lemire (w != 0, exact w): the proof of Mushtak & Lemire shows the
// 128-bit product always decides binary64.
SKG_HD inline Am lemire(int64_t q, uint64_t w) {
  Am a{0, 0};
  if (w == 0 || q < -342) return a;
  if (q > 308) { a.p2 = 0x7FF; return a; }
  const int lz = clz64(w);
  w <<= lz;
  const uint64_t* e = POW5_128[q + 342];
  uint64_t lo, hi = umul128_hi(w, e[0], &lo);
  if ((hi & 0x1FF) == 0x1FF) {   // precision mask for 55 bits
    uint64_t lo2, hi2 = umul128_hi(w, e[1], &lo2);
    lo += hi2;
    if (hi2 > lo) ++hi;
  }
  const int upper = (int)(hi >> 63);
  const int shift = upper + 64 - 52 - 3;
  a.m = hi >> shift;
  a.p2 = (int32_t)((((152170 + 65536) * q) >> 16) + 63) + upper - lz + 1023;
  if (a.p2 <= 0) {
    if (-a.p2 + 1 >= 64) { a.m = 0; a.p2 = 0; return a; }
    a.m >>= -a.p2 + 1;
    a.m += a.m & 1;
    a.m >>= 1;
    a.p2 = a.m < (1ull << 52) ? 0 : 1;
    return a;
  }
  if (lo <= 1 && q >= -4 && q <= 23 && (a.m & 3) == 1 && (a.m << shift) == hi) a.m &= ~1ull;
  a.m += a.m & 1;
  a.m >>= 1;
  if (a.m >= (2ull << 52)) { a.m = 1ull << 52; a.p2++; }
  a.m &= ~(1ull << 52);
  if (a.p2 >= 0x7FF) { a.p2 = 0x7FF; a.m = 0; }
  return a;
}

SKG_HD inline uint64_t am_bits(const Am& a) { return ((uint64_t)a.p2 << 52) | a.m; }

constexpr uint32_t FLT_MAXDIG = 800;   // beyond 768 significant digits only "nonzero" matters
constexpr uint32_t BIG_LIMBS = 160;

// Exact comparison of digits[0..nd) * 10^e10 (+ sticky) with the halfway point
// above the double `bits` (positive, finite): returns -1/0/+1.
SKG_HD SKG_NOINLINE int cmp_halfway(const uint8_t* digits, uint32_t nd, int32_t e10, bool sticky, uint64_t bits) {
  uint32_t da[BIG_LIMBS], db[BIG_LIMBS];
  Big A{da, 0, BIG_LIMBS}, B{db, 0, BIG_LIMBS};
  for (uint32_t i = 0; i < nd;) {   // 9 digits at a time
    uint32_t chunk = 0, mul = 1, k = 0;
    for (; k < 9 && i < nd; ++k, ++i) { chunk = chunk * 10 + digits[i]; mul *= 10; }
    A.mul_add(mul, chunk);
  }
  const uint32_t be = (uint32_t)(bits >> 52);
  uint64_t m = bits & ((1ull << 52) - 1);
  int32_t e2;
  if (be == 0) e2 = 1 - 1075; else { m |= 1ull << 52; e2 = (int32_t)be - 1075; }
  B.set_small(2 * m + 1);               // halfway = (2m + 1) * 2^(e2 - 1)
  int32_t ea = 0, eb = e2 - 1;          // A * 2^ea * 5^e10 (after folding 2^e10) vs B * 2^eb
  if (e10 >= 0) { A.mul_pow5((uint32_t)e10); ea += e10; }
  else { B.mul_pow5((uint32_t)-e10); eb -= e10; }
  if (ea > eb) { A.shl((uint32_t)(ea - eb)); } else if (eb > ea) { B.shl((uint32_t)(eb - ea)); }
  int c = big_cmp(A, B);
  if (c == 0 && sticky) c = 1;
  return c;
}

enum : uint32_t { FLT_OK = 0, FLT_INVALID = 1 };

// float(text) -> double bits (Python semantics).  Returns FLT_INVALID for a
// ValueError("could not convert string to float: ...").
SKG_HD SKG_NOINLINE uint32_t parse_float(const uint8_t* p, uint32_t n, const Uni& U, uint64_t& out) {
  // transformed characters, stripped
  uint32_t i = 0, len = 1, c;
  auto peek = [&](uint32_t at, uint32_t& l) -> uint32_t { return at < n ? xform(p, n, at, l, U) : 0u; };
  c = peek(i, len);
  while (i < n && ascii_space(c)) { i += len; c = peek(i, len); }
  uint32_t end = n;   // strip trailing spaces: find the last non-space character
  {
    uint32_t j = i, last_ns = i;
    while (j < n) { uint32_t l; uint32_t cc = xform(p, n, j, l, U); j += l; if (!ascii_space(cc)) last_ns = j; }
    end = last_ns;
  }
  if (i >= end) return FLT_INVALID;
  // underscores: only between digits (_Py_string_to_number_with_underscores)
  {
    uint32_t prev = 0;
    for (uint32_t j = i; j < end;) {
      uint32_t l; const uint32_t cc = xform(p, n, j, l, U);
      if (cc == '_') { if (!(prev >= '0' && prev <= '9')) return FLT_INVALID; }
      else if (prev == '_' && !(cc >= '0' && cc <= '9')) return FLT_INVALID;
      prev = cc; j += l;
    }
    if (prev == '_') return FLT_INVALID;
  }
  auto nextc = [&](uint32_t& j) -> uint32_t {   // next non-underscore char in [j, end)
    while (j < end) { uint32_t l; const uint32_t cc = xform(p, n, j, l, U); j += l; if (cc != '_') return cc; }
    return 0;
  };
  uint32_t j = i;
  uint32_t save = j;
  c = nextc(j);
  bool neg = false;
  if (c == '+' || c == '-') { neg = c == '-'; save = j; c = nextc(j); }
  const uint64_t sign = neg ? (1ull << 63) : 0;
  auto lower = [](uint32_t x) { return (x >= 'A' && x <= 'Z') ? x + 32 : x; };
  if (!((c >= '0' && c <= '9') || c == '.')) {
    // inf / infinity / nan (case-insensitive)
    uint32_t k = save;
    char buf[8]; uint32_t nb = 0;
    while (k < end && nb < 8) { buf[nb++] = (char)lower(nextc(k)); }
    if (k < end) return FLT_INVALID;
    auto is = [&](const char* z) { uint32_t q = 0; while (z[q]) { if (q >= nb || buf[q] != z[q]) return false; ++q; } return q == nb; };
    if (is("inf") || is("infinity")) { out = sign | (0x7FFull << 52); return FLT_OK; }
    if (is("nan")) { out = sign | (0x7FF8ull << 48); return FLT_OK; }
    return FLT_INVALID;
  }
  // mantissa digits
  uint64_t w = 0;
  uint32_t nsig = 0, nint = 0, nfrac = 0;
  int64_t drop = 0;      // significant digits not held in w (position count)
  bool seen_nonzero = false, trunc_nonzero = false, any_digit = false, dot = false;
  uint32_t dstart = save;
  while (true) {
    if (c >= '0' && c <= '9') {
      any_digit = true;
      if (dot) ++nfrac; else ++nint;
      const uint32_t d = c - '0';
      if (seen_nonzero || d != 0) {
        seen_nonzero = true;
        if (nsig < 19) { w = w * 10 + d; ++nsig; }
        else { ++drop; trunc_nonzero |= d != 0; }
      }
    } else if (c == '.' && !dot) {
      dot = true;
    } else break;
    if (j >= end) { c = 0; break; }
    c = nextc(j);
  }
  if (!any_digit) return FLT_INVALID;
  int64_t exp10 = 0;
  if (c == 'e' || c == 'E') {
    uint32_t c2 = j < end ? nextc(j) : 0;
    bool eneg = false;
    if (c2 == '+' || c2 == '-') { eneg = c2 == '-'; c2 = j < end ? nextc(j) : 0; }
    if (!(c2 >= '0' && c2 <= '9')) return FLT_INVALID;
    while (true) {
      if (c2 >= '0' && c2 <= '9') { if (exp10 < 100000000) exp10 = exp10 * 10 + (c2 - '0'); }
      else return FLT_INVALID;
      if (j >= end) break;
      c2 = nextc(j);
    }
    if (eneg) exp10 = -exp10;
  } else if (c != 0) {
    return FLT_INVALID;
  }
  if (!seen_nonzero) { out = sign; return FLT_OK; }
  // value = w * 10^q (+ truncated digits)
  const int64_t q = exp10 - (int64_t)nfrac + drop;
  if (q + (int64_t)nsig > 310) { out = sign | (0x7FFull << 52); return FLT_OK; }
  if (q + (int64_t)nsig < -345) { out = sign; return FLT_OK; }
  // Clinger fast path
  if (!drop && w <= (1ull << 53) && q >= -22 && q <= 22) {
    const double p10[23] = {1e0, 1e1, 1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8, 1e9, 1e10, 1e11,
                            1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
    double d = (double)w;
    d = q < 0 ? d / p10[-q] : d * p10[q];
    uint64_t b;
    memcpy(&b, &d, 8);
    out = sign | b;
    return FLT_OK;
  }
  Am a = lemire(q, w);
  if (drop == 0 || !trunc_nonzero) {   // w * 10^q is exact
    out = sign | am_bits(a);
    return FLT_OK;
  }
  Am a2 = lemire(q, w + 1);
  if (a.m == a2.m && a.p2 == a2.p2) { out = sign | am_bits(a); return FLT_OK; }
  // big-number decision between a and its successor: collect all digits
  uint8_t digs[FLT_MAXDIG];
  uint32_t nd = 0;
  bool sticky = false;
  for (uint32_t k = dstart, sn = 0; k < end;) {
    const uint32_t cc = nextc(k);
    if (cc == '.') continue;
    if (!(cc >= '0' && cc <= '9')) break;
    if (!sn && cc == '0') continue;
    sn = 1;
    if (nd < FLT_MAXDIG) digs[nd++] = (uint8_t)(cc - '0');
    else sticky |= cc != '0';
  }
  // all significant digits * 10^(exp10 - nfrac); the kept prefix ends (nsig + drop - nd) places higher
  const int64_t kept_pos_exp = exp10 - (int64_t)nfrac + ((int64_t)nsig + drop - (int64_t)nd);
  const uint64_t lo_bits = am_bits(a);
  const int c3 = cmp_halfway(digs, nd, (int32_t)kept_pos_exp, sticky, lo_bits);
  uint64_t r = lo_bits;
  if (c3 > 0 || (c3 == 0 && (lo_bits & 1))) r = lo_bits + 1;
  out = sign | r;
  return FLT_OK;
}

// struct.pack('<f', x) (PyFloat_Pack4): false on OverflowError
SKG_HD inline bool pack_f32(uint64_t bits, uint32_t& out) {
  const uint32_t sign = (uint32_t)(bits >> 63) << 31;
  const uint64_t ab = bits & ~(1ull << 63);
  if (ab > (0x7FFull << 52)) { out = sign | 0x7FC00000u | (uint32_t)((ab >> 29) & 0x3FFFFF); return true; }
  if (ab == (0x7FFull << 52)) { out = sign | 0x7F800000u; return true; }
  double x;
  memcpy(&x, &bits, 8);
#if defined(__CUDA_ARCH__)
  const float y = __double2float_rn(x);
#else
  const float y = (float)x;
#endif
  uint32_t yb;
  memcpy(&yb, &y, 4);
  if ((yb & 0x7FFFFFFFu) == 0x7F800000u) return false;
  out = yb;
  return true;
}

// struct.pack('<e', x) (PyFloat_Pack2): false on OverflowError
SKG_HD inline bool pack_f16(uint64_t bits, uint32_t& out) {
  const uint32_t sign = (uint32_t)(bits >> 63);
  const uint64_t ab = bits & ~(1ull << 63);
  uint32_t e, h;
  if (ab == 0) { e = 0; h = 0; }
  else if (ab == (0x7FFull << 52)) { e = 0x1F; h = 0; }
  else if (ab > (0x7FFull << 52)) { e = 0x1F; h = 512; }
  else {
    double x;
    memcpy(&x, &ab, 8);
    // frexp: x = f * 2^ex with f in [0.5, 1); then f *= 2, ex-- (f in [1, 2))
    int ex;
    uint32_t be = (uint32_t)(ab >> 52);
    uint64_t mant = ab & ((1ull << 52) - 1);
    if (be == 0) {   // subnormal double: normalise
      int sh = clz64(mant) - 11;
      mant <<= sh;
      mant &= (1ull << 52) - 1;
      ex = 1 - 1023 - sh;
    } else {
      ex = (int)be - 1023;
    }
    uint64_t fb = (1023ull << 52) | mant;   // f in [1, 2)
    double f;
    memcpy(&f, &fb, 8);
    if (ex >= 16) return false;
    int ee;
    if (ex < -25) { f = 0.0; ee = 0; }
    else if (ex < -14) {   // f = ldexp(f, 14 + ex): exact scaling by a power of two
      double scale = 1.0;
      for (int k = 0; k < -(14 + ex); ++k) scale *= 0.5;
      f *= scale;
      ee = 0;
    } else { ee = ex + 15; f -= 1.0; }
    f *= 1024.0;
    uint32_t b = (uint32_t)f;
    const double frac = f - (double)b;
    if (frac > 0.5 || (frac == 0.5 && (b & 1))) {
      ++b;
      if (b == 1024) { b = 0; ++ee; if (ee == 31) return false; }
    }
    e = (uint32_t)ee;
    h = b;
  }
  out = h | (e << 10) | (sign << 15);
  return true;
}

}  // namespace skg
