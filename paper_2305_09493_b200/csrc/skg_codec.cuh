// Standalone codec / tokenizer kernels behind the reference's per-item API
// (SURVEY.md 8(b)): tokenize_line (asm.py:51-90), encode_header /
// encode_instruction / encode_module (codec.py:61-101, 192-196),
// encode_string_literal (codec.py:104-114) and
// encode_context_dependent_literal (codec.py:132-168), each as a batch kernel
// over many items.  The big kernels (skg_asm, skg_disasm) run the same rules
// inside their own phases; these entry points serve the reference's
// fine-grained functions and batch builder serialization (ModuleScope.serialize
// = encode_header + encode_instruction per instruction, builder.py:208-224).
#pragma once
#include <cstdint>
#include "skg_text.cuh"

namespace skg {

// ---- tokenize_line ------------------------------------------------------------------
// One thread per line.  Token k of line l goes to slot line_off[l] + k (a token
// takes at least one byte).  String tokens are stored unescaped in `esc` at the
// offset of their first content byte; bare tokens are read from `text` in place.
enum : uint8_t { TOKF_STR = 1 };
enum : int32_t { TOKL_BLANK = 0, TOKL_INST = 1, TOKL_RESULT = 2, TOKL_UNTERMINATED = 3 };

__device__ __forceinline__ bool tok_ws(uint32_t c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n'; }
__device__ __forceinline__ bool tok_delim(uint32_t c) { return tok_ws(c) || c == ';' || c == '"'; }
__device__ __forceinline__ uint32_t is_lead(uint32_t c) { return (c & 0xC0u) != 0x80u; }

__global__ void tokenize_kernel(const uint8_t* __restrict__ text, const int64_t* __restrict__ line_off,
                                const int64_t* __restrict__ line_len, uint32_t n_lines,
                                uint64_t* __restrict__ tok_off, uint32_t* __restrict__ tok_len,
                                uint32_t* __restrict__ tok_col, uint8_t* __restrict__ tok_fl,
                                uint8_t* __restrict__ esc, int32_t* __restrict__ kind,
                                int32_t* __restrict__ ntok, uint32_t* __restrict__ err_col) {
  for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n_lines; l += gridDim.x * blockDim.x) {
    const uint64_t s0 = (uint64_t)line_off[l];
    const uint32_t n = (uint32_t)line_len[l];
    const uint8_t* t = text + s0;
    uint32_t i = 0, cp = 0, nt = 0;   // cp: code points before byte i (1-based columns)
    int32_t k = TOKL_BLANK;
    while (i < n) {
      const uint32_t c = t[i];
      if (tok_ws(c)) { ++i; ++cp; continue; }
      if (c == ';') break;
      const uint32_t start = i, col = cp + 1;
      if (c == '"') {                 // asm.py:67-79: \x -> x; a trailing backslash is literal
        ++i; ++cp;
        uint32_t w = 0;
        while (i < n && t[i] != '"') {
          if (t[i] == '\\' && i + 1 < n) { ++i; ++cp; }
          esc[s0 + start + 1 + w] = t[i];
          cp += is_lead(t[i]);
          ++w; ++i;
        }
        if (i >= n) { k = TOKL_UNTERMINATED; err_col[l] = col; break; }
        ++i; ++cp;
        tok_off[s0 + nt] = s0 + start + 1; tok_len[s0 + nt] = w; tok_col[s0 + nt] = col;
        tok_fl[s0 + nt] = TOKF_STR;
        ++nt;
        continue;
      }
      while (i < n && !tok_delim(t[i])) { cp += is_lead(t[i]); ++i; }   // asm.py:80-82
      tok_off[s0 + nt] = s0 + start; tok_len[s0 + nt] = i - start; tok_col[s0 + nt] = col;
      tok_fl[s0 + nt] = 0;
      ++nt;
    }
    if (k != TOKL_UNTERMINATED && nt > 0) {
      k = TOKL_INST;
      if (nt >= 3) {   // asm.py:86-88: tokens[0].text starts with '%' and tokens[1].text == "="
        const uint8_t* p0 = ((tok_fl[s0] & TOKF_STR) ? esc : text) + tok_off[s0];
        const uint8_t* p1 = ((tok_fl[s0 + 1] & TOKF_STR) ? esc : text) + tok_off[s0 + 1];
        if (tok_len[s0] >= 1 && p0[0] == '%' && tok_len[s0 + 1] == 1 && p1[0] == '=') k = TOKL_RESULT;
      }
    }
    kind[l] = k;
    ntok[l] = k == TOKL_UNTERMINATED ? 0 : (int32_t)nt;
  }
}

// ---- encode_module: header + instructions -> words ------------------------------------
// codes (python: codec.py messages, formatted by the host from its own values)
enum : uint32_t {
  ENC_OK = 0, ENC_BOUND0 = 1, ENC_BOUND_RANGE = 2, ENC_VERSION = 3, ENC_COUNT = 4, ENC_OPCODE = 5
};

// module m: hdr[5m..5m+4] = major, minor, generator (masked), bound, schema (masked);
// instructions inst_base[m] .. inst_base[m+1]; output words of module m start at
// 5m + inst_base[m] + op_off[inst_base[m]] (op_off has n_inst + 1 entries)
__global__ void encode_headers_kernel(const int64_t* __restrict__ hdr, uint32_t n_mod,
                                      const int64_t* __restrict__ inst_base, const int64_t* __restrict__ op_off,
                                      uint32_t* __restrict__ out, unsigned long long* __restrict__ err) {
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < n_mod; m += gridDim.x * blockDim.x) {
    const int64_t* h = hdr + 5ull * m;
    const int64_t ib = inst_base[m];
    const uint64_t o = 5ull * m + (uint64_t)ib + (uint64_t)op_off[ib];
    uint32_t code = ENC_OK;
    if (h[3] == 0) code = ENC_BOUND0;                                        // codec.py:67-68
    else if (!(h[3] > 0 && h[3] <= 0xFFFFFFFFll)) code = ENC_BOUND_RANGE;     // :69-70
    else if (!(h[0] >= 0 && h[0] <= 0xFF && h[1] >= 0 && h[1] <= 0xFF)) code = ENC_VERSION;   // :71-72
    err[m] = code ? (unsigned long long)code : ~0ull;
    if (code) continue;
    out[o] = 0x07230203u;
    out[o + 1] = ((uint32_t)h[0] << 16) | ((uint32_t)h[1] << 8);
    out[o + 2] = (uint32_t)h[2];
    out[o + 3] = (uint32_t)h[3];
    out[o + 4] = (uint32_t)h[4];
  }
}

__device__ __forceinline__ uint32_t upper_index(const int64_t* a, uint32_t n, int64_t v) {
  // largest k in [0, n) with a[k] <= v (a ascending, a[0] <= v)
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid; else hi = mid;
  }
  return lo;
}

// one thread per instruction: the first word, or the module's first error (count
// before opcode, codec.py:95-98), by atomicMin on (instruction, code)
__global__ void encode_insts_kernel(const int64_t* __restrict__ opcode, const int64_t* __restrict__ op_off,
                                    uint64_t n_inst, const int64_t* __restrict__ inst_base, uint32_t n_mod,
                                    uint32_t* __restrict__ out, unsigned long long* __restrict__ err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_inst; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t m = upper_index(inst_base, n_mod, (int64_t)i);
    const int64_t ib = inst_base[m];
    const int64_t count = 1 + (op_off[i + 1] - op_off[i]);
    uint32_t code = ENC_OK;
    if (count > 0xFFFF) code = ENC_COUNT;
    else if (!(opcode[i] >= 0 && opcode[i] <= 0xFFFF)) code = ENC_OPCODE;
    if (code) {
      const unsigned long long key = ((unsigned long long)(i - (uint64_t)ib + 1) << 8) | code;
      atomicMin(err + m, key);
      continue;
    }
    const uint64_t o = 5ull * (m + 1) + (uint64_t)i + (uint64_t)op_off[i];
    out[o] = ((uint32_t)count << 16) | (uint32_t)opcode[i];
  }
}

// one thread per operand word (already masked to 32 bits by the caller)
__global__ void encode_operands_kernel(const uint32_t* __restrict__ ops, uint64_t n_ops,
                                       const int64_t* __restrict__ op_off, uint32_t n_inst,
                                       const int64_t* __restrict__ inst_base, uint32_t n_mod,
                                       uint32_t* __restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_ops; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = upper_index(op_off, n_inst + 1, (int64_t)j);   // op_off[i] <= j < op_off[i+1]
    const uint32_t m = upper_index(inst_base, n_mod, (int64_t)i);
    out[5ull * (m + 1) + i + 1 + j] = ops[j];
  }
}

// ---- encode_string_literal ------------------------------------------------------------
// string s (bytes [off, off+len)) -> len/4 + 1 words at word offset wo[s]; one thread
// per output word; bad[s] = 1 on an embedded NUL (codec.py:109-110)
__global__ void pack_strings_kernel(const uint8_t* __restrict__ bytes, const int64_t* __restrict__ off,
                                    const int64_t* __restrict__ len, const int64_t* __restrict__ wo,
                                    uint32_t n_str, uint64_t n_words, uint32_t* __restrict__ out,
                                    int32_t* __restrict__ bad) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_words; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = upper_index(wo, n_str, (int64_t)j);
    const uint64_t b = 4 * (j - (uint64_t)wo[s]);
    const uint64_t L = (uint64_t)len[s];
    const uint8_t* p = bytes + off[s];
    uint32_t w = 0;
    bool nul = false;
    #pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
      if (b + q < L) {
        const uint32_t c = p[b + q];
        nul |= c == 0;
        w |= c << (8 * q);
      }
    }
    out[j] = w;
    if (nul) bad[s] = 1;
  }
}

// ---- encode_context_dependent_literal ----------------------------------------------------
enum : int32_t {
  LIT_OK = 0, LIT_UNRESOLVED = 1, LIT_WIDTH = 2, LIT_FWIDTH = 3, LIT_OVF_E = 4, LIT_OVF_F = 5,
  LIT_FIT_SIGNED = 6, LIT_FIT_UNSIGNED = 7
};
enum : uint32_t { LITF_SIGNED = 1, LITF_FLOAT = 2, LITF_NEG = 4, LITF_BIG = 8, LITF_NONE = 16 };

// literal k: width[k] (LITF_NONE in flags[k] = None), flags[k], val[k] = |int value| (u64; LITF_NEG / LITF_BIG
// for the sign / a magnitude of 2^64 or more) or the IEEE double bits (LITF_FLOAT)
__global__ void ctx_literals_kernel(const int64_t* __restrict__ width, const uint32_t* __restrict__ flags,
                                    const uint64_t* __restrict__ val, uint32_t n, uint32_t* __restrict__ words,
                                    int32_t* __restrict__ nwords, int32_t* __restrict__ status) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int64_t w = width[k];
    const uint32_t f = flags[k];
    uint32_t lo = 0, hi = 0;
    int32_t nw = 0, st = LIT_OK;
    if (f & LITF_NONE) st = LIT_UNRESOLVED;                                  // codec.py:140-141
    else if (!(w == 8 || w == 16 || w == 32 || w == 64)) st = LIT_WIDTH;     // :142-143
    else if (f & LITF_FLOAT) {                                               // :144-151
      const uint64_t bits = val[k];
      if (w == 8) st = LIT_FWIDTH;
      else if (w == 64) { lo = (uint32_t)bits; hi = (uint32_t)(bits >> 32); nw = 2; }
      else if (w == 32) { if (pack_f32(bits, lo)) nw = 1; else st = LIT_OVF_F; }
      else { if (pack_f16(bits, lo)) nw = 1; else st = LIT_OVF_E; }
    } else {                                                                  // :152-168
      const uint64_t mag = val[k];
      const bool neg = (f & LITF_NEG) && (mag != 0 || (f & LITF_BIG));
      const bool big = (f & LITF_BIG) != 0;
      const uint32_t wd = (uint32_t)w;
      if (f & LITF_SIGNED) {
        const uint64_t lim = 1ull << (wd - 1);
        if (big || (neg ? mag > lim : mag >= lim)) st = LIT_FIT_SIGNED;
      } else {
        if (big || neg || (wd < 64 && mag >= (1ull << wd))) st = LIT_FIT_UNSIGNED;
      }
      if (st == LIT_OK) {
        const uint64_t bits = neg ? (uint64_t)0 - mag : mag;
        if (wd == 64) { lo = (uint32_t)bits; hi = (uint32_t)(bits >> 32); nw = 2; }
        else {
          lo = (uint32_t)bits & (wd == 32 ? 0xFFFFFFFFu : ((1u << wd) - 1));
          if ((f & LITF_SIGNED) && neg && wd < 32) lo |= 0xFFFFFFFFu << wd;   // sign-extend
          nw = 1;
        }
      }
    }
    words[2ull * k] = lo;
    words[2ull * k + 1] = hi;
    nwords[k] = nw;
    status[k] = st;
  }
}

// ---- self-test: repr(float) of every float32 value (SURVEY.md 7 hard part 2) ---------------
// disasm renders f32 literals as CPython repr() of the value widened to double
// (codec.py:174-178, disasm.py:93-94; skg_fmt.cuh).  For each f32 bit pattern the
// kernel checks the two properties that define the shortest round-trip repr, with
// the assembler's independent float() parser (skg_text.cuh parse_float): the text
// parses back to exactly the same double, and neither (n-1)-digit neighbour of its
// n significant digits does.  nan / inf / zero must read "nan" / "inf" / "0.0".
struct BufSink {
  uint8_t b[48];
  uint32_t n = 0;
  __device__ void put(uint8_t c) { if (n < sizeof(b)) b[n] = c; ++n; }
  __device__ void putn(const uint8_t* s, uint32_t k) { for (uint32_t i = 0; i < k; ++i) put(s[i]); }
  __device__ void fill(uint8_t c, uint32_t k) { for (uint32_t i = 0; i < k; ++i) put(c); }
};

__device__ __forceinline__ bool sci_parses_to(bool neg, uint64_t digits, int32_t exp, const Uni& U, uint64_t bits) {
  BufSink s;
  if (neg) s.put('-');
  put_u64(s, digits);
  s.put('e');
  if (exp < 0) { s.put('-'); put_u64(s, (uint64_t)(-exp)); } else put_u64(s, (uint64_t)exp);
  uint64_t got = 0;
  return parse_float(s.b, s.n, U, got) == FLT_OK && got == bits;
}

__global__ void selftest_repr_f32_kernel(Uni U, uint64_t start, uint64_t count, unsigned long long* ctr,
                                         unsigned int* first_fail) {
  unsigned long long fails = 0;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = (uint32_t)(start + k);
    const uint64_t bits = f32_to_f64_bits(f);
    const FloatParts p = repr_parts(bits);
    BufSink s;
    put_repr_parts(s, p);
    bool ok;
    if (p.kind == 1) ok = s.n == 3 && s.b[0] == 'n' && s.b[1] == 'a' && s.b[2] == 'n';
    else if (p.kind == 2) ok = s.n == 3u + p.neg && s.b[p.neg] == 'i';
    else if (p.kind == 3) ok = s.n == 3u + p.neg && s.b[p.neg] == '0' && s.b[p.neg + 2] == '0';
    else {
      uint64_t got = 0;
      ok = s.n <= sizeof(s.b) && parse_float(s.b, s.n, U, got) == FLT_OK && got == bits;
      if (ok && p.digits >= 10) {   // shortest: no (n-1)-digit string reads back as the value
        const uint64_t lo = p.digits / 10;
        ok = !sci_parses_to(p.neg, lo, p.exp + 1, U, bits) && !sci_parses_to(p.neg, lo + 1, p.exp + 1, U, bits);
      }
    }
    if (!ok) { ++fails; atomicMin(first_fail, f); }
  }
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) fails += __shfl_xor_sync(0xFFFFFFFFu, fails, o);
  if ((threadIdx.x & 31) == 0 && fails) atomicAdd(ctr, fails);
}

}  // namespace skg
