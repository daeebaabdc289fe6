// Batch disassembler: binary modules -> text, bit-exact with the reference
// Disassembler.to_text (disasm.py:117-127, 131-377).
//
// Persistent warps take module tickets in order (atomic counter).  Per module:
//   load/boundary -> prescan -> [names mode: decode pass collecting referenced
//   ids + friendly-name resolution] -> size pass (per-line lengths, width) ->
//   decoupled look-back across tickets for the module's text offset -> write
//   pass.  The text of module m is out[text_off[m] : text_off[m+1]].
#include "skg_module.cuh"

namespace skg {

enum : uint32_t { OPT_HIGHLIGHT = 1, OPT_INLINE = 2, OPT_NO_INDENT = 4, OPT_GROUP = 8,
                  OPT_NO_HEADER = 16, OPT_STRICT = 32 };

__device__ const char* const ANSI_OPCODE = "\x1b[36m";
__device__ const char* const ANSI_ID = "\x1b[33m";
__device__ const char* const ANSI_STRING = "\x1b[32m";
__device__ const char* const ANSI_COMMENT = "\x1b[90m";
__device__ const char* const ANSI_RESET = "\x1b[0m";

struct DisasmArgs {
  Tables T;
  const uint8_t* data;
  const int64_t* mod_off;
  const int64_t* mod_len;
  uint32_t n_mod;
  uint32_t opts;
  uint8_t* text;
  uint64_t text_cap;
  int64_t* text_off;          // n_mod + 1
  int32_t* status;            // n_mod
  unsigned long long* state;  // n_mod look-back words (zeroed)
  uint32_t* ticket;           // counters: [0] ticket, [1] err count, [2] overflow
  ErrRec* errs;
  uint32_t err_cap;
  uint8_t* gscratch;          // per-warp global slots
  uint64_t gslot_bytes;
  uint32_t smem_slab;         // bytes per warp in dynamic shared memory
};

// -- sanitized friendly names (disasm.py:82-86) --------------------------------
struct NameView {
  const uint32_t* w;   // string words
  uint32_t nbytes;
};

__device__ inline NameView name_of(const Mod& m, uint32_t name_inst) {
  const uint32_t* ops = inst_ops(m, name_inst);
  uint32_t n = inst_nops(m, name_inst), nb = 0, next = 0;
  string_span(ops, 1, n, nb, next);
  return NameView{ops + 1, nb};
}

__device__ __forceinline__ uint32_t byte_at(const uint32_t* w, uint32_t i) {
  return (w[i >> 2] >> ((i & 3) * 8)) & 0xFF;
}
__device__ __forceinline__ bool is_word_char(uint32_t c) {
  return (c >= '0' && c <= '9') || (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_';
}

// visit sanitized characters: optional '_' prefix, then one char per code point
template <class F>
__device__ inline void for_sanitized(const NameView& nv, F&& f) {
  uint32_t first = 0xFFFFFFFF;
  for (uint32_t i = 0; i < nv.nbytes; ++i) {
    uint32_t c = byte_at(nv.w, i);
    if ((c & 0xC0) != 0x80) { first = c; break; }
  }
  bool prefix = first == 0xFFFFFFFF || (first >= '0' && first <= '9');
  if (prefix) f('_');
  for (uint32_t i = 0; i < nv.nbytes; ++i) {
    uint32_t c = byte_at(nv.w, i);
    if ((c & 0xC0) == 0x80) continue;
    f(is_word_char(c) ? c : '_');
  }
}

// -- ref rendering -------------------------------------------------------------
template <class S>
__device__ inline void put_ref(S& s, const Mod& m, uint32_t id) {
  s.put('%');
  uint32_t slot = ht_find(m, id);
  if (slot != NONE32 && (m.hfl[slot] & HF_FRIENDLY)) {
    NameView nv = name_of(m, m.hname[slot]);
    for_sanitized(nv, [&](uint32_t c) { s.put((uint8_t)c); });
    if (m.hser[slot] != NONE32) { s.put('_'); put_u64(s, m.hser[slot]); }
    return;
  }
  put_u64(s, id);
}

__device__ inline uint32_t ref_len(const Mod& m, uint32_t id) {
  uint32_t slot = ht_find(m, id);
  if (slot != NONE32 && (m.hfl[slot] & HF_FRIENDLY)) return m.hrl[slot];
  return 1 + dec_len_u64(id);
}

// -- per-instruction renderer ------------------------------------------------------
struct BodyInfo {
  bool has_result = false;
  uint32_t result = 0;
  bool have_set = false;
  uint32_t set_id = 0;
};

template <class S>
struct RenderVis {
  S& s;
  const Mod& m;
  const Tables& T;
  bool hl;
  bool ext_known;
  BodyInfo& info;
  bool& has_result;
  uint32_t& result;
  bool& have_set;
  uint32_t& set_id;
  __device__ RenderVis(S& s_, const Mod& m_, const Tables& T_, bool hl_, bool ek, BodyInfo& bi)
      : s(s_), m(m_), T(T_), hl(hl_), ext_known(ek), info(bi), has_result(bi.has_result),
        result(bi.result), have_set(bi.have_set), set_id(bi.set_id) {}

  __device__ void open(const char* color) { if (hl) put_cstr(s, color); }
  __device__ void close() { if (hl) put_cstr(s, ANSI_RESET); }
  __device__ void sep() { s.put(' '); }

  __device__ void id(uint32_t role, uint32_t v, int depth) {
    if (depth == 0 && role == IDR_RESULT) { has_result = true; result = v; return; }
    if (depth == 0 && role == IDR_ID && !have_set) { have_set = true; set_id = v; }
    sep();
    if (role == IDR_RESULT) { put_u64(s, v); return; }   // result inside a composite: str(value)
    open(ANSI_ID); put_ref(s, m, v); close();
  }
  __device__ void venum(uint32_t k, uint32_t v, uint32_t e) {
    sep();
    if (e != NONE32) s.putn(T.str + T.ename_off(e), T.ename_len(e));
    else put_u64(s, v);
  }
  __device__ void benum(uint32_t k, uint32_t mask, bool full, uint64_t comp) {
    sep();
    if (mask == 0) {
      uint32_t z = T.kzero(k);
      if (z != NONE32) s.putn(T.str + T.ename_off(z), T.ename_len(z));
      else s.put('0');
      return;
    }
    if (!full) { put_hex_lower(s, mask); return; }
    uint32_t eo = T.kenum_off(k);
    bool firstc = true;
    for (int j = 0; j < 64; ++j) {
      if (!((comp >> j) & 1)) continue;
      if (!firstc) s.put('|');
      firstc = false;
      s.putn(T.str + T.ename_off(eo + j), T.ename_len(eo + j));
    }
  }
  __device__ void str(const uint32_t* ops, uint32_t pos, uint32_t nbytes) {
    sep();
    open(ANSI_STRING);
    s.put('"');
    const uint32_t* w = ops + pos;
    for (uint32_t i = 0; i < nbytes; ++i) {
      uint32_t c = byte_at(w, i);
      if (c == '\\' || c == '"') s.put('\\');
      s.put((uint8_t)c);
    }
    s.put('"');
    close();
  }
  __device__ void typed(const LitVal& lv) {
    sep();
    if (lv.flt) put_repr_double(s, lv.bits);
    else if (lv.neg) put_i64(s, (int64_t)lv.bits);
    else put_u64(s, lv.bits);
  }
  __device__ void lit(uint32_t sub, uint32_t v) {
    sep();
    if (sub == LIT_EXTINST && ext_known) {
      uint32_t off, len;
      if (T.ext_name(v, off, len)) { s.putn(T.str + off, len); return; }
    } else if (sub == LIT_SPECOP) {
      uint32_t d = T.inst_of(v);
      if (d != NONE32) { s.putn(T.str + T.iname_off(d) + 2, T.iname_len(d) - 2); return; }
    }
    put_u64(s, v);
  }
  __device__ void comp_begin() {}
  __device__ void comp_end() {}
};

// body (opcode + operands) of instruction i; returns walk status
template <class S>
__device__ inline WalkErr render_body(S& s, const Mod& m, const Tables& T, uint32_t i, bool hl,
                                      bool ext_known, BodyInfo* info = nullptr) {
  const uint32_t d = m.idef[i];
  const uint32_t* ops = inst_ops(m, i);
  const uint32_t n = inst_nops(m, i);
  if (d == NONE16) {
    if (hl) put_cstr(s, ANSI_OPCODE);
    put_cstr(s, "OpUnknown("); put_u64(s, inst_opcode(m, i)); s.put(')');
    if (hl) put_cstr(s, ANSI_RESET);
    for (uint32_t k = 0; k < n; ++k) { s.put(' '); s.put('!'); s.put('0'); s.put('x'); put_hex8_upper(s, ops[k]); }
    return WalkErr{};
  }
  if (hl) put_cstr(s, ANSI_OPCODE);
  s.putn(T.str + T.iname_off(d), T.iname_len(d));
  if (hl) put_cstr(s, ANSI_RESET);
  BodyInfo local;
  RenderVis<S> vis(s, m, T, hl, ext_known, info ? *info : local);
  Resolver res{&m, &T};
  return walk(T, d, ops, n, vis, res);
}

// id collection for the friendly-name simulation (disasm.py:221-240)
struct CollectVis {
  const Mod& m;
  __device__ void id(uint32_t, uint32_t v, int) {
    uint32_t s = ht_insert(m, v);
    if (s != NONE32) m.hA[s] = 1;
  }
  __device__ void venum(uint32_t, uint32_t, uint32_t) {}
  __device__ void benum(uint32_t, uint32_t, bool, uint64_t) {}
  __device__ void str(const uint32_t*, uint32_t, uint32_t) {}
  __device__ void typed(const LitVal&) {}
  __device__ void lit(uint32_t, uint32_t) {}
  __device__ void comp_begin() {}
  __device__ void comp_end() {}
};

__device__ inline bool is_opencl_std(const Mod& m, const Tables& T, uint32_t set_id) {
  uint32_t s = ht_find(m, set_id);
  if (s == NONE32 || m.himp[s] == NONE32) return false;
  NameView nv = name_of(m, m.himp[s]);
  if (nv.nbytes != T.ocl_len) return false;
  for (uint32_t i = 0; i < nv.nbytes; ++i)
    if (byte_at(nv.w, i) != T.str[T.ocl_off + i]) return false;
  return true;
}

// ----------------------------------------------------------------------------
// friendly names: uniquify (disasm.py:173-185) + closed-form demotion
__device__ inline uint32_t fnv_step(uint32_t h, uint32_t c) { return (h ^ c) * 16777619u; }

struct NameRec {   // nrec layout (6 words)
  static constexpr int SLOT = 0, H = 1, P = 2, LEN = 3, SUFFIX = 4, CP = 5;
};

// hash + length + "ends with _<canonical int>" info of a sanitized name
__device__ inline void name_info(const NameView& nv, uint32_t& h, uint32_t& len, uint32_t& ph,
                                 bool& suffix) {
  h = 2166136261u; len = 0;
  uint32_t h_at_us = 0, len_at_us = 0xFFFFFFFF, digits = 0, first_digit = 0;
  for_sanitized(nv, [&](uint32_t c) {
    if (c == '_') { h_at_us = h; len_at_us = len; digits = 0; }
    else if (c >= '0' && c <= '9') { if (digits == 0) first_digit = c; ++digits; }
    else { digits = 0; len_at_us = 0xFFFFFFFF; }
    h = fnv_step(h, c);
    ++len;
  });
  // canonical decimal suffix right after the last '_' that ends the string
  suffix = len_at_us != 0xFFFFFFFF && digits > 0 && len_at_us + 1 + digits == len &&
           (first_digit != '0' || digits == 1);
  ph = suffix ? h_at_us : 0;
}

__device__ inline bool name_eq(const Mod& m, uint32_t slot_a, uint32_t slot_b) {
  NameView a = name_of(m, m.hname[slot_a]), b = name_of(m, m.hname[slot_b]);
  // compare sanitized sequences; both are short, materialise lazily
  uint32_t la = 0, lb = 0;
  for_sanitized(a, [&](uint32_t) { ++la; });
  for_sanitized(b, [&](uint32_t) { ++lb; });
  if (la != lb) return false;
  // walk both in lockstep
  uint32_t ia = 0, ib = 0;
  bool pa = false, pb = false;
  {
    uint32_t fa = 0xFFFFFFFF, fb = 0xFFFFFFFF;
    for (uint32_t i = 0; i < a.nbytes; ++i) { uint32_t c = byte_at(a.w, i); if ((c & 0xC0) != 0x80) { fa = c; break; } }
    for (uint32_t i = 0; i < b.nbytes; ++i) { uint32_t c = byte_at(b.w, i); if ((c & 0xC0) != 0x80) { fb = c; break; } }
    pa = fa == 0xFFFFFFFF || (fa >= '0' && fa <= '9');
    pb = fb == 0xFFFFFFFF || (fb >= '0' && fb <= '9');
  }
  auto next = [](const NameView& nv, uint32_t& i, bool& p) -> uint32_t {
    if (p) { p = false; return '_'; }
    while (i < nv.nbytes) {
      uint32_t c = byte_at(nv.w, i++);
      if ((c & 0xC0) == 0x80) continue;
      return is_word_char(c) ? c : '_';
    }
    return 0;
  };
  for (uint32_t k = 0; k < la; ++k)
    if (next(a, ia, pa) != next(b, ib, pb)) return false;
  return true;
}

// candidate string = sanitized(base of nrec k) [+ "_" + serial]
__device__ inline uint32_t cand_hash(const Mod& m, uint32_t k, uint32_t serial) {
  uint32_t h = m.nrec[6 * k + NameRec::H];
  if (serial != NONE32) {
    h = fnv_step(h, '_');
    char buf[12]; int n = 0;
    uint32_t v = serial;
    do { buf[n++] = (char)('0' + v % 10); v /= 10; } while (v);
    while (n) h = fnv_step(h, (uint32_t)buf[--n]);
  }
  return h;
}

__device__ inline bool cand_eq(const Mod& m, uint32_t k1, uint32_t s1, uint32_t k2, uint32_t s2) {
  auto len = [&](uint32_t k, uint32_t s) {
    return m.nrec[6 * k + NameRec::LEN] + (s == NONE32 ? 0 : 1 + dec_len_u64(s));
  };
  if (len(k1, s1) != len(k2, s2)) return false;
  // materialise both into small buffers chunk by chunk via sink
  struct Gen {
    const Mod& m; uint32_t k, s;
    __device__ void emit(uint32_t* out, uint32_t& n, uint32_t cap, uint32_t from) const {
      uint32_t idx = 0;
      NameView nv = name_of(m, m.hname[m.nrec[6 * k + NameRec::SLOT]]);
      auto push = [&](uint32_t c) { if (idx >= from && n < cap) out[n++] = c; ++idx; };
      for_sanitized(nv, push);
      if (s != NONE32) {
        push('_');
        char buf[12]; int q = 0; uint32_t v = s;
        do { buf[q++] = (char)('0' + v % 10); v /= 10; } while (v);
        while (q) push((uint32_t)buf[--q]);
      }
    }
  };
  const uint32_t total = len(k1, s1);
  uint32_t ba[32], bb[32];
  for (uint32_t from = 0; from < total; from += 32) {
    uint32_t na = 0, nb = 0;
    Gen{m, k1, s1}.emit(ba, na, 32, from);
    Gen{m, k2, s2}.emit(bb, nb, 32, from);
    for (uint32_t q = 0; q < na; ++q) if (ba[q] != bb[q]) return false;
  }
  return true;
}

__device__ inline void resolve_names(Mod& m, const Tables& T) {
  const uint32_t lane = lane_id();
  // 1. flags per entry: named definition / pinned (P0 = A - named definitions)
  for (uint32_t s = lane; s <= m.C; s += 32) {
    bool present = s < m.C ? m.hkey[s] != EMPTY : *m.top_present != 0;
    uint8_t f = 0;
    if (present) {
      bool named_d = m.hname[s] != NONE32 && m.hdef[s] != NONE32;
      if (named_d) f |= HF_NAMED_D;
      if (m.hA[s] && !named_d) f |= HF_P0;
    }
    m.hfl[s] = f;
  }
  __syncwarp();
  // 2. walk instructions in order: definitions (first occurrence) give D;
  //    C = D without P0 (index j), named D entries listed in D order.
  uint32_t nP0 = 0;
  for (uint32_t s = lane; s <= m.C; s += 32) nP0 += (m.hfl[s] & HF_P0) ? 1 : 0;
  nP0 = warp_sum_u32(nP0);
  uint32_t cj = 0, nd = 0;
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane;
    bool isC = false, isN = false;
    uint32_t slot = NONE32;
    if (i < m.I) {
      uint32_t d = m.idef[i];
      if (d != NONE16 && T.has_result(d)) {
        uint32_t idx = T.has_rtype(d) ? 1 : 0;
        if (idx < inst_nops(m, i)) {
          slot = ht_find(m, inst_ops(m, i)[idx]);
          if (slot != NONE32 && m.hdef[slot] == i) {
            isC = !(m.hfl[slot] & HF_P0);
            isN = (m.hfl[slot] & HF_NAMED_D) != 0;
          }
        }
      }
    }
    unsigned bc = __ballot_sync(FULL, isC), bn = __ballot_sync(FULL, isN);
    uint32_t below = (1u << lane) - 1;
    if (isC) m.ib[i] = cj + __popc(bc & below);          // j of this definition
    if (isN) m.nrec[6 * (nd + __popc(bn & below)) + NameRec::SLOT] = slot;
    if (i < m.I) m.iflag[i] = (m.iflag[i] & ~IF_FIRSTDEF) | (isC ? IF_FIRSTDEF : 0);
    cj += __popc(bc);
    nd += __popc(bn);
  }
  __syncwarp();
  // 3. closed form: pos[v] = -1 (P0) / j (c_j) / INF, prefix max, keep test
  const uint32_t N = nP0 + cj;
  const int32_t INF = 0x7FFFFFFF;
  for (uint32_t v = lane; v <= N && v < m.npos; v += 32) m.pos[v] = INF;
  __syncwarp();
  for (uint32_t s = lane; s <= m.C; s += 32) {
    if (!(m.hfl[s] & HF_P0)) continue;
    uint32_t key = s < m.C ? m.hkey[s] : EMPTY;
    if (key >= 1 && key <= N) m.pos[key] = -1;
  }
  __syncwarp();
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane;
    if (i < m.I && (m.iflag[i] & IF_FIRSTDEF)) {
      uint32_t d = m.idef[i];
      uint32_t key = inst_ops(m, i)[T.has_rtype(d) ? 1 : 0];
      if (key >= 1 && key <= N) m.pos[key] = (int32_t)m.ib[i];
    }
  }
  __syncwarp();
  // inclusive prefix max over pos[1..N] (in place)
  int32_t carry = -2;   // below every j and -1
  for (uint32_t base = 1; base <= N; base += 32) {
    uint32_t v = base + lane;
    int32_t x = v <= N ? m.pos[v] : -2;
    x = warp_incl_max(x);
    x = max(x, carry);
    if (v <= N) m.pos[v] = x;
    carry = __shfl_sync(FULL, x, 31);
  }
  __syncwarp();
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane;
    if (i < m.I && (m.iflag[i] & IF_FIRSTDEF)) {
      uint32_t d = m.idef[i];
      uint32_t key = inst_ops(m, i)[T.has_rtype(d) ? 1 : 0];
      int32_t j = (int32_t)m.ib[i];
      bool kept = key >= 1 && key <= N && (key == 1 || m.pos[key - 1] < j);
      if (kept) {
        uint32_t slot = ht_find(m, key);
        m.hfl[slot] |= HF_KEPT;
      }
    }
  }
  __syncwarp();
  // 4. uniquify names in D order
  for (uint32_t k = lane; k < nd; k += 32) {
    uint32_t slot = m.nrec[6 * k + NameRec::SLOT];
    NameView nv = name_of(m, m.hname[slot]);
    uint32_t h, len, ph;
    bool suffix;
    name_info(nv, h, len, ph, suffix);
    m.nrec[6 * k + NameRec::H] = h;
    m.nrec[6 * k + NameRec::P] = ph;
    m.nrec[6 * k + NameRec::LEN] = len;
    m.nrec[6 * k + NameRec::SUFFIX] = suffix;
  }
  __syncwarp();
  bool slow = false;
  for (uint32_t k = lane; k < nd; k += 32) {
    if (!m.nrec[6 * k + NameRec::SUFFIX]) continue;
    uint32_t ph = m.nrec[6 * k + NameRec::P];
    for (uint32_t q = 0; q < nd && !slow; ++q)
      if (m.nrec[6 * q + NameRec::H] == ph) slow = true;
  }
  slow = __any_sync(FULL, slow);
  if (!slow) {
    for (uint32_t k = lane; k < nd; k += 32) {
      uint32_t h = m.nrec[6 * k + NameRec::H];
      uint32_t slot = m.nrec[6 * k + NameRec::SLOT];
      uint32_t rank = 0;
      for (uint32_t q = 0; q < k; ++q)
        if (m.nrec[6 * q + NameRec::H] == h && name_eq(m, slot, m.nrec[6 * q + NameRec::SLOT])) ++rank;
      m.hser[slot] = rank == 0 ? NONE32 : rank - 1;
    }
  } else if (lane == 0) {
    // sequential simulation with a taken set of (k, serial) candidates
    uint32_t TS = 16;
    while (TS < 2 * nd + 2) TS <<= 1;
    int32_t* tk = m.pos;              // TS pairs (k, serial); pos no longer needed
    for (uint32_t t = 0; t < 2 * TS; ++t) tk[t] = -1;
    for (uint32_t k = 0; k < nd; ++k) {
      uint32_t serial = NONE32;
      while (true) {
        uint32_t h = cand_hash(m, k, serial);
        uint32_t p = h & (TS - 1);
        bool taken = false;
        while (tk[2 * p] != -1) {
          if (cand_eq(m, (uint32_t)tk[2 * p], (uint32_t)tk[2 * p + 1], k, serial)) { taken = true; break; }
          p = (p + 1) & (TS - 1);
        }
        if (!taken) { tk[2 * p] = (int32_t)k; tk[2 * p + 1] = (int32_t)serial; break; }
        serial = serial == NONE32 ? 0 : serial + 1;
      }
      m.hser[m.nrec[6 * k + NameRec::SLOT]] = serial;
    }
  }
  __syncwarp();
  // 5. friendly = named definition that keeps its number; cache its ref length
  for (uint32_t k = lane; k < nd; k += 32) {
    uint32_t slot = m.nrec[6 * k + NameRec::SLOT];
    if (m.hfl[slot] & HF_KEPT) {
      m.hfl[slot] |= HF_FRIENDLY;
      uint32_t ser = m.hser[slot];
      m.hrl[slot] = 1 + m.nrec[6 * k + NameRec::LEN] + (ser == NONE32 ? 0 : 1 + dec_len_u64(ser));
    }
  }
  __syncwarp();
}

// ----------------------------------------------------------------------------
// section tracking for the `group` option (disasm.py:253-267)
__device__ inline void compute_sections(Mod& m, const Tables& T) {
  if (lane_id() == 0) {
    uint32_t sec = 0;
    bool in_fn = false;
    for (uint32_t i = 0; i < m.I; ++i) {
      uint32_t d = m.idef[i];
      if (d != NONE16) {
        uint32_t sp = T.special(d);
        if (sp == SP_FUNCTION) { sec = 9; in_fn = true; }
        else if (in_fn) { sec = 9; in_fn = sp != SP_FUNCTIONEND; }
        else {
          uint32_t c = T.section(d);
          if (c != SECTION_KEEP) { sec = c; in_fn = false; }
        }
      }
      m.isec[i] = (uint8_t)sec;
    }
  }
  __syncwarp();
}

template <class S>
__device__ inline void put_header(S& s, const Mod& m, bool hl) {
  auto line = [&](auto&& body) {
    if (hl) put_cstr(s, ANSI_COMMENT);
    body();
    if (hl) put_cstr(s, ANSI_RESET);
    s.put('\n');
  };
  line([&] { put_cstr(s, "; SPIR-V"); });
  line([&] { put_cstr(s, "; Version: "); put_u64(s, m.major); s.put('.'); put_u64(s, m.minor); });
  line([&] { put_cstr(s, "; Generator: "); put_u64(s, m.gen >> 16); put_cstr(s, "; "); put_u64(s, m.gen & 0xFFFF); });
  line([&] { put_cstr(s, "; Bound: "); put_u64(s, m.bound); });
  line([&] { put_cstr(s, "; Schema: "); put_u64(s, m.schema); });
}

// record the exception of instruction i (re-walk for the message)
__device__ inline void report_inst_error(const Mod& m, const Tables& T, uint32_t i, ErrRec* rec,
                                         int32_t module, int32_t& cls) {
  uint32_t d = m.idef[i];
  CountSink cs;
  WalkErr e = render_body(cs, m, T, i, false, true);
  cls = walk_status(e.code);
  if (rec) {
    ErrWriter ew{rec};
    put_walk_error(ew, T, d, e);
    rec->module = module; rec->cls = cls; rec->len = ew.n;
    rec->a = e.a; rec->b = e.b; rec->c = e.c; rec->d = e.d;
  }
}

__device__ inline void report_prescan_error(const Mod& m, const Tables& T, uint32_t i, ErrRec* rec,
                                            int32_t module) {
  const uint32_t* ops = inst_ops(m, i);
  uint32_t nb, next;
  string_span(ops, 1, inst_nops(m, i), nb, next);
  WalkErr e;
  string_utf8(ops, 1, nb, e);
  if (rec) {
    ErrWriter ew{rec};
    put_walk_error(ew, T, 0, e);
    rec->module = module; rec->cls = ST_UNICODE; rec->len = ew.n;
    rec->a = e.a; rec->b = e.b; rec->c = e.c; rec->d = e.d;
  }
}

// first instruction index (in order) for which pred holds, or NONE32
template <class P>
__device__ inline uint32_t first_where(const Mod& m, P&& pred) {
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane_id();
    unsigned b = __ballot_sync(FULL, i < m.I && pred(i));
    if (b) return base + __ffs(b) - 1;
  }
  return NONE32;
}

// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) disasm_kernel(DisasmArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = lane_id();
  const uint32_t warp_in_block = threadIdx.x >> 5;
  const uint32_t gwarp = blockIdx.x * (blockDim.x >> 5) + warp_in_block;
  uint8_t* slab = smem + (size_t)warp_in_block * a.smem_slab;
  uint8_t* gslot = a.gscratch + (size_t)gwarp * a.gslot_bytes;
  const Tables& T = a.T;
  const bool hl = a.opts & OPT_HIGHLIGHT;
  ErrSink es{a.errs, a.ticket + 1, a.err_cap};

  while (true) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1u);
    t = __shfl_sync(FULL, t, 0);
    if (t >= a.n_mod) break;
    const int64_t nbytes = a.mod_len[t];
    const uint8_t* src = a.data + a.mod_off[t];
    int32_t status = ST_OK;
    ErrRec* erec = nullptr;
    uint64_t total = 0;
    uint32_t width = 0;
    Mod m;
    const uint32_t W = (nbytes >= 0 && nbytes % 4 == 0) ? (uint32_t)(nbytes / 4) : 0;
    bool in_smem = head_bytes(W) <= a.smem_slab;
    if (!in_smem && worst_bytes(W) > a.gslot_bytes) {
      status = ST_INTERNAL;
      if (lane == 0) {
        erec = es.alloc();
        if (erec) {
          ErrWriter ew{erec};
          put_cstr(ew, "internal: module exceeds the per-warp scratch slot");
          erec->module = (int32_t)t; erec->cls = ST_INTERNAL; erec->len = ew.n;
        }
      }
    } else {
      layout_head(m, in_smem ? slab : gslot, W);
      status = load_and_split(m, src, (uint64_t)nbytes, &es, (int32_t)t);
    }
    if (status == ST_OK) {
      // choose table capacity; move to the global slot if the slab is too small
      uint32_t C = table_capacity(m.I);
      for (int attempt = 0; attempt < 3; ++attempt) {
        if (head_bytes(m.W) + tables_bytes(m.I, C) > (in_smem ? a.smem_slab : a.gslot_bytes)) {
          if (in_smem) {
            // copy words + offsets into the global slot
            Mod g;
            layout_head(g, gslot, m.W);
            for (uint32_t k = lane; k < m.W; k += 32) g.w[k] = m.w[k];
            for (uint32_t k = lane; k < m.I; k += 32) g.ioff[k] = m.ioff[k];
            g.I = m.I; g.major = m.major; g.minor = m.minor; g.gen = m.gen; g.bound = m.bound; g.schema = m.schema;
            __syncwarp();
            m = g;
            in_smem = false;
          }
          if (head_bytes(m.W) + tables_bytes(m.I, C) > a.gslot_bytes) { status = ST_INTERNAL; break; }
        }
        layout_tables(m, C);
        init_tables(m);
        bool any_name = prescan(m, T);
        bool names_mode = (a.opts & OPT_INLINE) && any_name;
        if (names_mode) {
          // decode pass collecting referenced ids (A) + per-instruction status
          for (uint32_t base = 0; base < m.I; base += 32) {
            uint32_t i = base + lane;
            if (i < m.I && m.idef[i] != NONE16) {
              CollectVis cv{m};
              Resolver res{&m, &T};
              WalkErr e = walk(T, m.idef[i], inst_ops(m, i), inst_nops(m, i), cv, res);
              m.ierr[i] = (uint8_t)e.code;
            }
          }
          __syncwarp();
        }
        if (*m.overflow) {
          C = C * 4;
          while (C < 2 * m.W + 8) C <<= 1;
          __syncwarp();
          continue;
        }
        // --- exceptions, in the reference's evaluation order ---
        uint32_t bad = first_where(m, [&](uint32_t i) { return (m.iflag[i] & IF_PRESCAN_UTF8) != 0; });
        if (bad != NONE32) {
          status = ST_UNICODE;
          if (lane == 0) { erec = es.alloc(); report_prescan_error(m, T, bad, erec, (int32_t)t); }
          break;
        }
        if (names_mode) {
          bad = first_where(m, [&](uint32_t i) { uint32_t e = m.ierr[i]; return e != W_OK && !werr_is_codec(e); });
          if (bad != NONE32) {
            if (lane == 0) { erec = es.alloc(); report_inst_error(m, T, bad, erec, (int32_t)t, status); }
            status = __shfl_sync(FULL, status, 0);
            break;
          }
          resolve_names(m, T);
        }
        // size pass: per-instruction body length, result ref, errors
        width = 0;
        for (uint32_t base = 0; base < m.I; base += 32) {
          uint32_t i = base + lane;
          if (i < m.I) {
            CountSink cs;
            bool ext_known = true;
            uint32_t d = m.idef[i];
            if (d != NONE16 && T.special(d) == SP_EXTINST) {
              // ext_set_known needs the set id: first pass over operands
              CountSink tmp;
              BodyInfo b0;
              render_body(tmp, m, T, i, false, true, &b0);
              ext_known = b0.have_set && is_opencl_std(m, T, b0.set_id);
            }
            BodyInfo vis;
            WalkErr e = render_body(cs, m, T, i, hl, ext_known, &vis);
            m.ierr[i] = (uint8_t)e.code;
            m.ia[i] = cs.n;
            uint8_t fl = m.iflag[i] & ~(IF_HAS_RESULT | IF_EXT_KNOWN);
            if (ext_known) fl |= IF_EXT_KNOWN;
            if (d != NONE16 && vis.has_result) {
              fl |= IF_HAS_RESULT;
              m.ib[i] = vis.result;
              uint32_t rl = ref_len(m, vis.result);
              m.irl[i] = rl;
              width = max(width, rl);
            }
            m.iflag[i] = fl;
          }
        }
        __syncwarp();
        bad = first_where(m, [&](uint32_t i) {
          return (m.idef[i] == NONE16 && (a.opts & OPT_STRICT)) || (m.idef[i] != NONE16 && m.ierr[i] != W_OK);
        });
        if (bad != NONE32) {
          if (lane == 0) {
            erec = es.alloc();
            if (m.idef[bad] == NONE16) {
              status = ST_CODEC;
              if (erec) {
                ErrWriter ew{erec};
                put_cstr(ew, "unknown opcode "); put_u64(ew, inst_opcode(m, bad));
                erec->module = (int32_t)t; erec->cls = ST_CODEC; erec->len = ew.n;
              }
            } else {
              report_inst_error(m, T, bad, erec, (int32_t)t, status);
            }
          }
          status = __shfl_sync(FULL, status, 0);
          break;
        }
        width = (a.opts & OPT_NO_INDENT) ? 0 : warp_max_u32(width);
        if (a.opts & OPT_GROUP) compute_sections(m, T);
        // line lengths -> offsets (ia := start offset of the line, relative)
        CountSink hs;
        if (!(a.opts & OPT_NO_HEADER)) put_header(hs, m, hl);
        uint64_t run = hs.n;
        const uint32_t paint_extra = hl ? 9 : 0;   // "\x1b[33m" + "\x1b[0m"
        for (uint32_t base = 0; base < m.I; base += 32) {
          uint32_t i = base + lane;
          uint32_t len = 0, blank = 0;
          if (i < m.I) {
            uint32_t body = m.ia[i];
            if (m.iflag[i] & IF_HAS_RESULT) {
              uint32_t rl = m.irl[i];
              len = (width ? width - rl : 0) + rl + paint_extra + 3 + body;
            } else {
              len = (width ? width + 3 : 0) + body;
            }
            if ((a.opts & OPT_GROUP) && i > 0 && m.isec[i] != m.isec[i - 1]) blank = 1;
            len += 1 + blank;
          }
          uint32_t incl = warp_incl_sum(len);
          if (i < m.I) m.ia[i] = (uint32_t)(run + incl - len + blank);
          run += __shfl_sync(FULL, incl, 31);
        }
        __syncwarp();
        total = run;
        break;
      }
    }
    // publish size, get offset
    if (status != ST_OK) total = 0;
    uint64_t off = lookback(a.state, t, total);
    if (lane == 0) {
      a.text_off[t] = (int64_t)off;
      a.status[t] = status;
      if (t == a.n_mod - 1) a.text_off[a.n_mod] = (int64_t)(off + total);
    }
    if (status == ST_OK && total > 0) {
      if (off + total > a.text_cap) {
        if (lane == 0) atomicExch(a.ticket + 2, 1u);
      } else {
        uint8_t* out = a.text + off;
        if (lane == 0 && !(a.opts & OPT_NO_HEADER)) { MemSink ms(out); put_header(ms, m, hl); }
        for (uint32_t base = 0; base < m.I; base += 32) {
          uint32_t i = base + lane;
          if (i >= m.I) continue;
          uint32_t lo = m.ia[i];
          if ((a.opts & OPT_GROUP) && i > 0 && m.isec[i] != m.isec[i - 1]) out[lo - 1] = '\n';
          MemSink ms(out + lo);
          if (m.iflag[i] & IF_HAS_RESULT) {
            uint32_t rl = m.irl[i];
            if (width) ms.fill(' ', width - rl);
            if (hl) put_cstr(ms, ANSI_ID);
            put_ref(ms, m, m.ib[i]);
            if (hl) put_cstr(ms, ANSI_RESET);
            put_cstr(ms, " = ");
          } else if (width) {
            ms.fill(' ', width + 3);
          }
          render_body(ms, m, T, i, hl, (m.iflag[i] & IF_EXT_KNOWN) != 0);
          ms.put('\n');
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace skg
