// Grammar-table slot walk: the device restatement of ops.decode_operands
// (reference ops.py:328-446).  One instruction per lane; the recursion of
// _DecodeState.one (enumerant parameters, composite bases) becomes an explicit
// stack of kind indices.  A visitor receives one event per decoded operand in
// exactly the order the reference appends DecodedOperand objects.
#pragma once
#include "skg_tables.cuh"
#include "skg_fmt.cuh"

namespace skg {

enum : uint32_t {
  W_OK = 0, W_EXHAUSTED = 1, W_LEFTOVER = 2, W_NONUL = 3, W_UNRESOLVED = 4,
  W_UNICODE = 5, W_KEY = 6, W_VALUE = 7
};

// CodecError family vs. exceptions that escape the reference's `except CodecError`
__host__ __device__ inline bool werr_is_codec(uint32_t e) { return e >= W_EXHAUSTED && e <= W_UNRESOLVED; }

struct WalkErr {
  uint32_t code = W_OK;
  uint32_t a = 0, b = 0, c = 0, d = 0;   // leftover n | width | utf8 start,end,reason,byte
};

// Width resolution result (disasm.py:69-79 RenderContext.literal_resolver)
struct Width {
  uint32_t width;
  bool sgn, flt, ok;
};

// Bytes of a NUL-terminated literal starting at ops[pos]; returns false if no
// NUL byte occurs before ops[n] (codec.py:117-129).
__device__ __noinline__ bool string_span(const uint32_t* ops, uint32_t pos, uint32_t n,
                                   uint32_t& nbytes, uint32_t& next) {
  for (uint32_t i = pos; i < n; ++i) {
    uint32_t w = ops[i];
    uint32_t z = ((w - 0x01010101u) & ~w & 0x80808080u);
    if (z) {
      uint32_t b = (__ffs(z) - 1) >> 3;
      nbytes = (i - pos) * 4 + b;
      next = i + 1;
      return true;
    }
  }
  return false;
}

struct WordBytes {
  const uint32_t* w;
  __device__ uint32_t operator()(uint32_t i) const { return (w[i >> 2] >> ((i & 3) * 8)) & 0xFF; }
};

__device__ __noinline__ uint32_t string_utf8(const uint32_t* ops, uint32_t pos, uint32_t nbytes, WalkErr& err) {
  {   // ASCII fast path, a word at a time
    uint32_t i = 0;
    const uint32_t nw = nbytes >> 2;
    while (i < nw && !(ops[pos + i] & 0x80808080u)) ++i;
    if (i == nw) {
      const uint32_t tail = nbytes & 3;
      if (!tail || !(ops[pos + nw] & 0x80808080u & ((1u << (8 * tail)) - 1))) return U8_OK;
    }
  }
  WordBytes at{ops + pos};
  uint32_t s = 0, e = 0;
  uint32_t r = utf8_check(at, nbytes, s, e);
  if (r != U8_OK) {
    err.code = W_UNICODE; err.a = s; err.b = e; err.c = r; err.d = at(s);
  }
  return r;
}

// Decode a width-typed literal (codec.py:171-185) into (bits, is_float, negative).
struct LitVal {
  uint64_t bits;      // int: two's complement 64-bit (sign-extended if negative); float: double bits
  bool flt;
  bool neg;           // int only
  bool wide_unsigned; // int: value >= 2^63 unsigned
  bool sgn;           // governing type (width, signedness)
  uint32_t width;
};

__device__ __noinline__ bool decode_typed(const uint32_t* raw, uint32_t width, bool sgn, bool flt,
                                    LitVal& out, WalkErr& err) {
  out.sgn = sgn;
  out.width = width;
  if (flt) {
    out.flt = true; out.neg = false; out.wide_unsigned = false;
    if (width == 64) { out.bits = (uint64_t)raw[0] | ((uint64_t)raw[1] << 32); return true; }
    if (width == 32) { out.bits = f32_to_f64_bits(raw[0]); return true; }
    if (width == 16) { out.bits = f16_to_f64_bits(raw[0] & 0xFFFF); return true; }
    err.code = W_KEY; err.a = width;
    return false;
  }
  out.flt = false; out.neg = false; out.wide_unsigned = false;
  if (width == 64) {
    uint64_t v = (uint64_t)raw[0] | ((uint64_t)raw[1] << 32);
    out.bits = v;
    if (sgn && (v >> 63)) out.neg = true;
    else if (v >> 63) out.wide_unsigned = true;
    return true;
  }
  if (sgn && width == 0) { err.code = W_VALUE; return false; }
  uint32_t bits = width >= 32 ? raw[0] : (raw[0] & ((1u << width) - 1));
  if (sgn && width <= 32 && width > 0 && (bits >> (width - 1)) & 1) {
    // bits - 2^width as a negative int64
    int64_t v = (int64_t)bits - (int64_t)((uint64_t)1 << width);
    out.bits = (uint64_t)v; out.neg = true;
    return true;
  }
  out.bits = bits;
  return true;
}

constexpr uint32_t STACK_MARK = 0xFFFFFFFFu;   // composite end marker
constexpr int WALK_STACK = 48;

// Visitor interface (all __device__; p = operand word index of the event):
//   id(role, value, depth, p)           role IDR_*
//   venum(kind, value, enum_index, p)   enum_index NONE32 if unknown
//   benum(kind, mask, full, comp, p)    full: covered by enumerants (comp = positions)
//   str(ops, word_pos, nbytes)
//   typed(LitVal, p, nwords)            ctx number / OpSwitch literal
//   lit(sub, value, p)                  LIT_PLAIN / LIT_EXTINST / LIT_SPECOP / LIT_INTEGER
//   comp_begin(), comp_end()
// Resolver: Width rt(uint32_t result_type_id), Width sel(uint32_t selector)
template <class V, class R>
__device__ __noinline__ WalkErr walk(const Tables& T, uint32_t idef, const uint32_t* ops, uint32_t n,
                        V& vis, const R& res) {
  WalkErr err;
  uint32_t pos = 0;
  bool have_rt = false, have_first = false, first_int = false;
  uint32_t rt = 0;
  uint64_t first_val = 0;
  const bool is_switch = T.special(idef) == SP_SWITCH;
  uint32_t st[WALK_STACK];
  int sp = 0;
  int depth = 0;

  auto note_first = [&](bool is_int, uint64_t v) {
    if (depth == 0 && !have_first) { have_first = true; first_int = is_int; first_val = v; }
  };
  auto resolve = [&]() -> Width {
    if (is_switch) {
      if (!have_first || !first_int || (first_val >> 32)) return Width{0, false, false, false};
      return res.sel((uint32_t)first_val);
    }
    if (!have_rt) return Width{0, false, false, false};
    return res.rt(rt);
  };

  // process one kind (and everything it expands to)
  auto one = [&](uint32_t kind0) -> bool {
    st[sp++] = kind0;
    while (sp > 0) {
      uint32_t k = st[--sp];
      if (k == STACK_MARK) {
        --depth;
        vis.comp_end();
        note_first(false, 0);
        continue;
      }
      uint32_t cat = T.kcat(k);
      if (cat == CAT_ID) {
        if (pos >= n) { err.code = W_EXHAUSTED; return false; }
        uint32_t v = ops[pos++];
        uint32_t role = T.ksub(k);
        if (depth == 0 && role == IDR_RESULT_TYPE && !have_rt) { have_rt = true; rt = v; }
        note_first(true, v);
        vis.id(role, v, depth, pos - 1);
      } else if (cat == CAT_VALUEENUM) {
        if (pos >= n) { err.code = W_EXHAUSTED; return false; }
        uint32_t v = ops[pos++];
        uint32_t e = T.venum_lookup(k, v);
        note_first(true, v);
        vis.venum(k, v, e, pos - 1);
        if (e != NONE32) {
          uint32_t np = T.enparams(e), po = T.eparam_off(e);
          if (sp + (int)np > WALK_STACK) { err.code = W_EXHAUSTED; return false; }
          for (int j = (int)np - 1; j >= 0; --j) st[sp++] = T.slot_kind(po + j);
        }
      } else if (cat == CAT_BITENUM) {
        if (pos >= n) { err.code = W_EXHAUSTED; return false; }
        uint32_t mask = ops[pos++];
        uint32_t eo = T.kenum_off(k), ne = T.knenum(k);
        uint64_t comp = 0;          // component positions within the kind (file order)
        uint32_t covered = 0;
        if (mask != 0) {
#pragma unroll 1
          for (uint32_t j = 0; j < ne && j < 64; ++j) {
            uint32_t ev = T.evalue(eo + j);
            if (ev && (mask & ev) == ev && (covered & ev) != ev) {
              comp |= 1ull << j; covered |= ev;
              if (covered == mask) break;   // later enumerants can only be skipped
            }
          }
        }
        bool full = mask != 0 && covered == mask;
        note_first(true, mask);
        vis.benum(k, mask, full, comp, pos - 1);
        if (full) {
          for (uint64_t rest = comp; rest; rest &= ~(1ull << (63 - __clzll((long long)rest)))) {
            const int j = 63 - __clzll((long long)rest);
            uint32_t e = eo + j;
            uint32_t np = T.enparams(e), po = T.eparam_off(e);
            if (sp + (int)np > WALK_STACK) { err.code = W_EXHAUSTED; return false; }
            for (int q = (int)np - 1; q >= 0; --q) st[sp++] = T.slot_kind(po + q);
          }
        }
      } else if (cat == CAT_COMPOSITE) {
        uint32_t nb = T.knbases(k), bo = T.kbase_off(k);
        if (sp + (int)nb + 1 > WALK_STACK) { err.code = W_EXHAUSTED; return false; }
        vis.comp_begin();
        st[sp++] = STACK_MARK;
        for (int j = (int)nb - 1; j >= 0; --j) st[sp++] = __ldg(T.slot + bo + j) & 0xFFFF;
        ++depth;
      } else {  // literal
        uint32_t sub = T.ksub(k);
        if (sub == LIT_STRING) {
          uint32_t nbytes, next;
          if (!string_span(ops, pos, n, nbytes, next)) { err.code = W_NONUL; return false; }
          if (string_utf8(ops, pos, nbytes, err) != U8_OK) return false;
          note_first(false, 0);
          vis.str(ops, pos, nbytes);
          pos = next;
        } else if (sub == LIT_CTXNUM) {
          Width wd = resolve();
          if (!wd.ok) { err.code = W_UNRESOLVED; return false; }
          uint32_t need = wd.width == 64 ? 2 : 1;
          uint32_t raw[2] = {0, 0};
          for (uint32_t j = 0; j < need; ++j) {
            if (pos >= n) { err.code = W_EXHAUSTED; return false; }
            raw[j] = ops[pos++];
          }
          LitVal lv;
          if (!decode_typed(raw, wd.width, wd.sgn, wd.flt, lv, err)) return false;
          note_first(!lv.flt && !lv.neg && !(lv.bits >> 32), lv.bits);
          vis.typed(lv, pos - need, need);
        } else {
          if (sub == LIT_INTEGER && is_switch) {
            Width wd = resolve();
            if (wd.ok) {
              uint32_t need = wd.width == 64 ? 2 : 1;
              uint32_t raw[2] = {0, 0};
              for (uint32_t j = 0; j < need; ++j) {
                if (pos >= n) { err.code = W_EXHAUSTED; return false; }
                raw[j] = ops[pos++];
              }
              LitVal lv;
              if (!decode_typed(raw, wd.width, wd.sgn, false, lv, err)) return false;
              note_first(!lv.neg && !(lv.bits >> 32), lv.bits);
              vis.typed(lv, pos - need, need);
              continue;
            }
          }
          if (pos >= n) { err.code = W_EXHAUSTED; return false; }
          uint32_t v = ops[pos++];
          note_first(true, v);
          vis.lit(sub, v, pos - 1);
        }
      }
    }
    return true;
  };

  // slot iteration as a state machine so `one` has a single call site
  // (decode_operands, ops.py:340-350): '*' repeats its kind to the end, '?' is
  // skipped when no words remain, LiteralSpecConstantOpInteger is followed by
  // IdRef operands until the words run out.
  const uint32_t ns = T.inslots(idef), so = T.islot_off(idef);
  uint32_t s = 0, rep_kind = 0;
  bool repeat = false, stop_after_repeat = false, pending_tail = false;
#pragma unroll 1
  for (;;) {
    uint32_t k;
    if (repeat) {
      if (pos >= n) {
        repeat = false;
        if (stop_after_repeat) break;
        continue;
      }
      k = rep_kind;
    } else {
      if (s >= ns) break;
      const uint32_t q = T.slot_quant(so + s);
      k = T.slot_kind(so + s);
      const bool tail = T.slot_spec_tail(so + s);
      ++s;
      if (q == Q_VAR) { repeat = true; stop_after_repeat = true; rep_kind = k; continue; }
      if (q == Q_OPT && pos >= n) continue;
      pending_tail = tail;
    }
    if (!one(k)) return err;
    if (pending_tail) { pending_tail = false; repeat = true; stop_after_repeat = false; rep_kind = T.idref; }
  }
  if (pos < n) { err.code = W_LEFTOVER; err.a = n - pos; }
  return err;
}

}  // namespace skg
