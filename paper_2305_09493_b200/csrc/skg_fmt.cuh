// Text primitives shared by the codec kernels: output sinks, CPython-exact
// integer / float formatting, strict UTF-8 validation with CPython's error
// positions.  Everything is __host__ __device__ so the exhaustive float tests
// can also run the same code on the host (tests/test_fmt_host.py).
#pragma once
#include <cstdint>

#ifndef SKG_HD
#define SKG_HD __host__ __device__
#endif
#ifndef SKG_NOINLINE
#define SKG_NOINLINE __noinline__
#endif

#include "skg_pow5.cuh"

namespace skg {

// ---------------------------------------------------------------------------
// Sinks.  Every renderer is templated on a sink so the size pass and the write
// pass run the same code (disasm size-then-write).
// One sink type for both passes keeps a single instantiation of every
// renderer (code size matters: the kernels are instruction-fetch bound when
// each visitor/sink pair is inlined separately).  p == nullptr counts only.
struct Sink {
  uint8_t* p;
  uint32_t n = 0;
  SKG_HD explicit Sink(uint8_t* dst = nullptr) : p(dst) {}
  SKG_HD void put(uint8_t c) { if (p) p[n] = c; ++n; }
  SKG_HD void putn(const uint8_t* s, uint32_t len) {
    if (p) for (uint32_t i = 0; i < len; ++i) p[n + i] = s[i];
    n += len;
  }
  SKG_HD void fill(uint8_t c, uint32_t k) {
    if (p) for (uint32_t i = 0; i < k; ++i) p[n + i] = c;
    n += k;
  }
};
using CountSink = Sink;
using MemSink = Sink;

template <class S>
SKG_HD SKG_NOINLINE void put_cstr(S& s, const char* z) {
#pragma unroll 1
  while (*z) s.put((uint8_t)*z++);
}

SKG_HD inline uint32_t dec_len_u64(uint64_t v) {
  uint32_t n = 1;
  while (v >= 10) { v /= 10; ++n; }
  return n;
}

template <class S>
SKG_HD SKG_NOINLINE void put_u64(S& s, uint64_t v) {
  char buf[20];
  int n = 0;
#pragma unroll 1
  do { buf[n++] = (char)('0' + v % 10); v /= 10; } while (v);
#pragma unroll 1
  while (n) s.put((uint8_t)buf[--n]);
}

template <class S>
SKG_HD inline void put_i64(S& s, int64_t v) {
  if (v < 0) { s.put('-'); put_u64(s, (uint64_t)0 - (uint64_t)v); }
  else put_u64(s, (uint64_t)v);
}

// "0x%x" lowercase, unpadded (disasm.py:350)
template <class S>
SKG_HD inline void put_hex_lower(S& s, uint32_t v) {
  s.put('0'); s.put('x');
  int sh = 28;
  while (sh > 0 && ((v >> sh) & 0xF) == 0) sh -= 4;
  for (; sh >= 0; sh -= 4) s.put((uint8_t)"0123456789abcdef"[(v >> sh) & 0xF]);
}

// "0x%08X" uppercase (disasm.py:276, codec.py:215)
template <class S>
SKG_HD inline void put_hex8_upper(S& s, uint32_t v) {
  for (int sh = 28; sh >= 0; sh -= 4) s.put((uint8_t)"0123456789ABCDEF"[(v >> sh) & 0xF]);
}

template <class S>
SKG_HD inline void put_hex2_lower(S& s, uint32_t v) {
  s.put((uint8_t)"0123456789abcdef"[(v >> 4) & 0xF]);
  s.put((uint8_t)"0123456789abcdef"[v & 0xF]);
}

// ---------------------------------------------------------------------------
// Shortest round-trip decimal of a double (CPython repr / dtoa mode 0), via the
// Ryu algorithm: interval [vm, vp] of decimals that round back to the value,
// computed with 128-bit multipliers, then digit removal.
SKG_HD inline uint64_t umul128_hi(uint64_t a, uint64_t b, uint64_t* lo) {
#if defined(__CUDA_ARCH__)
  *lo = a * b;
  return __umul64hi(a, b);
#else
  unsigned __int128 r = (unsigned __int128)a * b;
  *lo = (uint64_t)r;
  return (uint64_t)(r >> 64);
#endif
}

SKG_HD inline uint64_t mul_shift64(uint64_t m, const uint64_t* mul, int32_t j) {
  // ((m * mul) >> j), mul = mul[1]:mul[0] (128 bit), 64 <= j < 128
  uint64_t lo0, lo2;
  uint64_t hi0 = umul128_hi(m, mul[0], &lo0);
  uint64_t hi2 = umul128_hi(m, mul[1], &lo2);
  uint64_t sum_lo = hi0 + lo2;
  uint64_t carry = sum_lo < hi0;
  uint64_t sum_hi = hi2 + carry;
  int32_t s = j - 64;
  if (s == 0) return sum_lo;
  return (sum_lo >> s) | (sum_hi << (64 - s));
}

SKG_HD inline uint32_t pow5bits(int32_t e) { return (uint32_t)(((e * 1217359) >> 19) + 1); }
SKG_HD inline uint32_t log10pow2(int32_t e) { return (uint32_t)((e * 78913) >> 18); }
SKG_HD inline uint32_t log10pow5(int32_t e) { return (uint32_t)((e * 732923) >> 20); }
SKG_HD inline uint32_t pow5_factor(uint64_t v) {
  uint32_t c = 0;
  while (v % 5 == 0) { v /= 5; ++c; }
  return c;
}
SKG_HD inline bool mult_pow5(uint64_t v, uint32_t p) { return pow5_factor(v) >= p; }
SKG_HD inline bool mult_pow2(uint64_t v, uint32_t p) { return p < 64 && (v & ((1ull << p) - 1)) == 0; }

// Decompose a finite nonzero double into (digits, exponent): value = digits * 10^exp,
// digits shortest with round-half-even acceptance of the interval ends.
SKG_HD SKG_NOINLINE void shortest_decimal(uint64_t bits, uint64_t& out_digits, int32_t& out_exp) {
  const uint64_t ieee_m = bits & ((1ull << 52) - 1);
  const uint32_t ieee_e = (uint32_t)((bits >> 52) & 0x7FF);
  int32_t e2;
  uint64_t m2;
  if (ieee_e == 0) { e2 = 1 - 1023 - 52 - 2; m2 = ieee_m; }
  else { e2 = (int32_t)ieee_e - 1023 - 52 - 2; m2 = (1ull << 52) | ieee_m; }
  const bool accept = (m2 & 1) == 0;
  const uint64_t mv = 4 * m2;
  const uint32_t mm_shift = (ieee_m != 0 || ieee_e <= 1) ? 1 : 0;
  uint64_t vr, vp, vm;
  int32_t e10;
  bool vm_tz = false, vr_tz = false;
  if (e2 >= 0) {
    const uint32_t q = log10pow2(e2) - (e2 > 3);
    e10 = (int32_t)q;
    const int32_t k = 125 + (int32_t)pow5bits((int32_t)q) - 1;
    const int32_t i = -e2 + (int32_t)q + k;
#if defined(__CUDA_ARCH__)
    uint64_t mul[2] = {__ldg(&POW5_INV_SPLIT[q][0]), __ldg(&POW5_INV_SPLIT[q][1])};
#elif defined(__CUDACC__)
    uint64_t mul[2] = {0, 0};   // host pass of the CUDA build: never called
#else
    uint64_t mul[2] = {POW5_INV_SPLIT[q][0], POW5_INV_SPLIT[q][1]};
#endif
    vr = mul_shift64(4 * m2, mul, i);
    vp = mul_shift64(4 * m2 + 2, mul, i);
    vm = mul_shift64(4 * m2 - 1 - mm_shift, mul, i);
    if (q <= 21) {
      if (mv % 5 == 0) vr_tz = mult_pow5(mv, q);
      else if (accept) vm_tz = mult_pow5(mv - 1 - mm_shift, q);
      else vp -= mult_pow5(mv + 2, q) ? 1 : 0;
    }
  } else {
    const uint32_t q = log10pow5(-e2) - (-e2 > 1);
    e10 = (int32_t)q + e2;
    const int32_t i = -e2 - (int32_t)q;
    const int32_t k = (int32_t)pow5bits(i) - 125;
    const int32_t j = (int32_t)q - k;
#if defined(__CUDA_ARCH__)
    uint64_t mul[2] = {__ldg(&POW5_SPLIT[i][0]), __ldg(&POW5_SPLIT[i][1])};
#elif defined(__CUDACC__)
    uint64_t mul[2] = {0, 0};   // host pass of the CUDA build: never called
#else
    uint64_t mul[2] = {POW5_SPLIT[i][0], POW5_SPLIT[i][1]};
#endif
    vr = mul_shift64(4 * m2, mul, j);
    vp = mul_shift64(4 * m2 + 2, mul, j);
    vm = mul_shift64(4 * m2 - 1 - mm_shift, mul, j);
    if (q <= 1) {
      vr_tz = true;
      if (accept) vm_tz = mm_shift == 1;
      else --vp;
    } else if (q < 63) {
      vr_tz = mult_pow2(mv, q);
    }
  }
  int32_t removed = 0;
  uint32_t last = 0;
  uint64_t output;
  if (vm_tz || vr_tz) {
    for (;;) {
      uint64_t vpd = vp / 10, vmd = vm / 10;
      if (vpd <= vmd) break;
      uint32_t vm_mod = (uint32_t)(vm - 10 * vmd);
      uint64_t vrd = vr / 10;
      uint32_t vr_mod = (uint32_t)(vr - 10 * vrd);
      vm_tz &= vm_mod == 0;
      vr_tz &= last == 0;
      last = vr_mod;
      vr = vrd; vp = vpd; vm = vmd;
      ++removed;
    }
    if (vm_tz) {
      for (;;) {
        uint64_t vmd = vm / 10;
        uint32_t vm_mod = (uint32_t)(vm - 10 * vmd);
        if (vm_mod != 0) break;
        uint64_t vpd = vp / 10, vrd = vr / 10;
        uint32_t vr_mod = (uint32_t)(vr - 10 * vrd);
        vr_tz &= last == 0;
        last = vr_mod;
        vr = vrd; vp = vpd; vm = vmd;
        ++removed;
      }
    }
    if (vr_tz && last == 5 && vr % 2 == 0) last = 4;
    output = vr + (((vr == vm && (!accept || !vm_tz)) || last >= 5) ? 1 : 0);
  } else {
    bool round_up = false;
    uint64_t vpd100 = vp / 100, vmd100 = vm / 100;
    if (vpd100 > vmd100) {
      uint64_t vrd100 = vr / 100;
      uint32_t vr_mod100 = (uint32_t)(vr - 100 * vrd100);
      round_up = vr_mod100 >= 50;
      vr = vrd100; vp = vpd100; vm = vmd100;
      removed += 2;
    }
    for (;;) {
      uint64_t vpd = vp / 10, vmd = vm / 10;
      if (vpd <= vmd) break;
      uint64_t vrd = vr / 10;
      uint32_t vr_mod = (uint32_t)(vr - 10 * vrd);
      round_up = vr_mod >= 5;
      vr = vrd; vp = vpd; vm = vmd;
      ++removed;
    }
    output = vr + ((vr == vm || round_up) ? 1 : 0);
  }
  int32_t exp = e10 + removed;
  while (output % 10 == 0 && output != 0) { output /= 10; ++exp; }
  out_digits = output;
  out_exp = exp;
}

// CPython repr(float) pieces of a double: kind 0 finite nonzero, 1 nan, 2 inf, 3 zero.
struct FloatParts {
  uint64_t digits;
  int32_t exp;
  uint8_t kind;
  bool neg;
};

SKG_HD SKG_NOINLINE FloatParts repr_parts(uint64_t bits) {
  FloatParts p;
  p.neg = bits >> 63;
  const uint32_t e = (uint32_t)((bits >> 52) & 0x7FF);
  const uint64_t m = bits & ((1ull << 52) - 1);
  p.digits = 0; p.exp = 0;
  if (e == 0x7FF) { p.kind = m ? 1 : 2; if (m) p.neg = false; return p; }
  if (e == 0 && m == 0) { p.kind = 3; return p; }
  p.kind = 0;
  shortest_decimal(bits, p.digits, p.exp);
  return p;
}

// length of repr() text (disasm.py:93-94 / float_repr_style 'short')
SKG_HD SKG_NOINLINE uint32_t repr_len(const FloatParts& p) {
  const uint32_t sgn = p.neg ? 1 : 0;
  if (p.kind != 0) return sgn + 3;                        // nan / inf / 0.0
  const int32_t n = (int32_t)dec_len_u64(p.digits);
  const int32_t decpt = n + p.exp;
  if (decpt <= -4 || decpt > 16) {
    int32_t x = decpt - 1;
    uint32_t xl = dec_len_u64((uint64_t)(x < 0 ? -x : x));
    return sgn + 1 + (n > 1 ? (uint32_t)n : 0) + 2 + (xl < 2 ? 2 : xl);
  }
  if (decpt <= 0) return sgn + 2 + (uint32_t)(-decpt) + (uint32_t)n;
  if (decpt < n) return sgn + (uint32_t)n + 1;
  return sgn + (uint32_t)decpt + 2;
}

template <class S>
SKG_HD SKG_NOINLINE void put_repr_parts(S& s, const FloatParts& p) {
  if (p.kind == 1) { put_cstr(s, "nan"); return; }
  if (p.neg) s.put('-');
  if (p.kind == 2) { put_cstr(s, "inf"); return; }
  if (p.kind == 3) { put_cstr(s, "0.0"); return; }
  char buf[20];
  int n = 0;
  { uint64_t v = p.digits; do { buf[n++] = (char)('0' + v % 10); v /= 10; } while (v); }
  // buf holds digits reversed; value = 0.d1..dn * 10^decpt
  const int32_t decpt = n + p.exp;
  if (decpt <= -4 || decpt > 16) {
    s.put((uint8_t)buf[n - 1]);
    if (n > 1) {
      s.put('.');
      #pragma unroll 1
      for (int i = n - 2; i >= 0; --i) s.put((uint8_t)buf[i]);
    }
    s.put('e');
    int32_t x = decpt - 1;
    if (x < 0) { s.put('-'); x = -x; } else s.put('+');
    if (x < 10) s.put('0');
    put_u64(s, (uint64_t)x);
    return;
  }
  if (decpt <= 0) {
    s.put('0'); s.put('.');
    #pragma unroll 1
    for (int32_t i = 0; i < -decpt; ++i) s.put('0');
    #pragma unroll 1
    for (int i = n - 1; i >= 0; --i) s.put((uint8_t)buf[i]);
    return;
  }
  if (decpt < n) {
    #pragma unroll 1
    for (int i = n - 1; i >= n - decpt; --i) s.put((uint8_t)buf[i]);
    s.put('.');
    #pragma unroll 1
    for (int i = n - decpt - 1; i >= 0; --i) s.put((uint8_t)buf[i]);
    return;
  }
  #pragma unroll 1
  for (int i = n - 1; i >= 0; --i) s.put((uint8_t)buf[i]);
  #pragma unroll 1
  for (int32_t i = n; i < decpt; ++i) s.put('0');
  s.put('.'); s.put('0');
}

// CPython repr(float) of a double given by its bits (disasm.py:93-94).
template <class S>
SKG_HD inline void put_repr_double(S& s, uint64_t bits) {
  put_repr_parts(s, repr_parts(bits));
}

// f16 / f32 bits widened to double bits (struct '<e' / '<f' unpack, codec.py:174-178)
SKG_HD inline uint64_t f32_to_f64_bits(uint32_t f) {
  const uint64_t sign = (uint64_t)(f >> 31) << 63;
  uint32_t e = (f >> 23) & 0xFF, m = f & 0x7FFFFF;
  if (e == 0xFF) return sign | (0x7FFull << 52) | ((uint64_t)m << 29);
  if (e == 0) {
    if (m == 0) return sign;
    int sh = 0;
    while (!(m & 0x800000)) { m <<= 1; ++sh; }
    m &= 0x7FFFFF;
    return sign | ((uint64_t)(1023 - 126 - sh) << 52) | ((uint64_t)m << 29);
  }
  return sign | ((uint64_t)(e - 127 + 1023) << 52) | ((uint64_t)m << 29);
}

SKG_HD inline uint64_t f16_to_f64_bits(uint32_t h) {
  const uint64_t sign = (uint64_t)((h >> 15) & 1) << 63;
  uint32_t e = (h >> 10) & 0x1F, m = h & 0x3FF;
  if (e == 0x1F) return sign | (0x7FFull << 52) | ((uint64_t)m << 42);
  if (e == 0) {
    if (m == 0) return sign;
    int sh = 0;
    while (!(m & 0x400)) { m <<= 1; ++sh; }
    m &= 0x3FF;
    return sign | ((uint64_t)(1023 - 14 - sh) << 52) | ((uint64_t)m << 42);
  }
  return sign | ((uint64_t)(e - 15 + 1023) << 52) | ((uint64_t)m << 42);
}

// ---------------------------------------------------------------------------
// Strict UTF-8 check with CPython's error report (Objects/stringlib/codecs.h
// utf8_decode + unicode_decode_utf8 error handling): returns 0 if valid, else
// a reason (1 invalid start byte, 2 invalid continuation byte, 3 unexpected end
// of data) and the [start, end) byte range.
enum : uint32_t { U8_OK = 0, U8_START = 1, U8_CONT = 2, U8_END = 3 };

template <class ByteAt>
SKG_HD SKG_NOINLINE uint32_t utf8_check(const ByteAt& at, uint32_t len, uint32_t& start, uint32_t& end) {
  uint32_t s = 0;
  while (s < len) {
    uint32_t ch = at(s);
    if (ch < 0x80) { ++s; continue; }
    uint32_t left = len - s;
    auto cont = [&](uint32_t k) { uint32_t c = at(s + k); return (c & 0xC0) == 0x80; };
    if (ch < 0xC2) { start = s; end = s + 1; return U8_START; }
    if (ch < 0xE0) {
      if (left < 2) { start = s; end = len; return U8_END; }
      if (!cont(1)) { start = s; end = s + 1; return U8_CONT; }
      s += 2;
      continue;
    }
    if (ch < 0xF0) {
      if (left < 3) {
        if (left >= 2) {
          uint32_t c2 = at(s + 1);
          if ((c2 & 0xC0) != 0x80 || (c2 < 0xA0 ? ch == 0xE0 : ch == 0xED)) {
            start = s; end = s + 1; return U8_CONT;
          }
        }
        start = s; end = len; return U8_END;
      }
      uint32_t c2 = at(s + 1);
      if ((c2 & 0xC0) != 0x80) { start = s; end = s + 1; return U8_CONT; }
      if (ch == 0xE0 ? c2 < 0xA0 : (ch == 0xED && c2 >= 0xA0)) { start = s; end = s + 1; return U8_CONT; }
      if (!cont(2)) { start = s; end = s + 2; return U8_CONT; }
      s += 3;
      continue;
    }
    if (ch < 0xF5) {
      if (left < 4) {
        if (left >= 2) {
          uint32_t c2 = at(s + 1);
          if ((c2 & 0xC0) != 0x80 || (c2 < 0x90 ? ch == 0xF0 : ch == 0xF4)) {
            start = s; end = s + 1; return U8_CONT;
          }
          if (left >= 3 && !cont(2)) { start = s; end = s + 2; return U8_CONT; }
        }
        start = s; end = len; return U8_END;
      }
      uint32_t c2 = at(s + 1);
      if ((c2 & 0xC0) != 0x80) { start = s; end = s + 1; return U8_CONT; }
      if (ch == 0xF0 ? c2 < 0x90 : (ch == 0xF4 && c2 >= 0x90)) { start = s; end = s + 1; return U8_CONT; }
      if (!cont(2)) { start = s; end = s + 2; return U8_CONT; }
      if (!cont(3)) { start = s; end = s + 3; return U8_CONT; }
      s += 4;
      continue;
    }
    start = s; end = s + 1;
    return U8_START;
  }
  return U8_OK;
}

}  // namespace skg
