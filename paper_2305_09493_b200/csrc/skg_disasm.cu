// Batch disassembler: binary modules -> text, bit-exact with the reference
// Disassembler.to_text (disasm.py:117-127, 131-377).
//
// Persistent warps take module tickets in order (atomic counter).  Per module:
//   load/boundary -> prescan -> [names mode: decode pass collecting referenced
//   ids + friendly-name resolution] -> size pass (per-line lengths, width) ->
//   bump allocation of the module's text bytes -> write pass.  The text of
//   module m is text[span[2m] : span[2m] + span[2m+1]].
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
  int64_t* text_span;         // 2 * n_mod: offset, length
  int32_t* status;            // n_mod
  uint32_t* ticket;           // counters: [0] ticket, [1] err count, [2] overflow, [4..5] cursor
  ErrRec* errs;
  uint32_t err_cap;
  uint8_t* gscratch;          // per-warp global slots
  uint64_t gslot_bytes;
  uint8_t* gtext;             // per-warp text scratch (L2-resident working set)
  uint64_t gtext_bytes;
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

__device__ inline uint32_t cand_len(const Mod& m, uint32_t slot, uint32_t serial);

__device__ inline uint32_t ref_len(const Mod& m, uint32_t id) {
  uint32_t slot = ht_find(m, id);
  if (slot != NONE32 && (m.hfl[slot] & HF_FRIENDLY)) {
    if (m.hrl[slot] != 0xFFFF) return m.hrl[slot];
    uint32_t n = 1;
    for_sanitized(name_of(m, m.hname[slot]), [&](uint32_t) { ++n; });
    if (m.hser[slot] != NONE32) n += 1 + dec_len_u64(m.hser[slot]);
    return n;
  }
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

constexpr uint8_t HF_SUFFIX = 16;

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
  suffix = len_at_us != 0xFFFFFFFF && digits > 0 && len_at_us + 1 + digits == len &&
           (first_digit != '0' || digits == 1);
  ph = suffix ? h_at_us : 0;
}

// candidate string of named slot `slot` = sanitized base [+ "_" + serial]
template <class F>
__device__ inline void for_candidate(const Mod& m, uint32_t slot, uint32_t serial, F&& f) {
  for_sanitized(name_of(m, m.hname[slot]), f);
  if (serial != NONE32) {
    f('_');
    char buf[12]; int q = 0; uint32_t v = serial;
    do { buf[q++] = (char)('0' + v % 10); v /= 10; } while (v);
    while (q) f((uint32_t)buf[--q]);
  }
}

__device__ inline uint32_t cand_len(const Mod& m, uint32_t slot, uint32_t serial) {
  return m.nLen[slot] + (serial == NONE32 ? 0 : 1 + dec_len_u64(serial));
}

__device__ inline uint32_t cand_hash(const Mod& m, uint32_t slot, uint32_t serial) {
  uint32_t h = m.nH[slot];
  if (serial != NONE32) {
    h = fnv_step(h, '_');
    char buf[12]; int n = 0; uint32_t v = serial;
    do { buf[n++] = (char)('0' + v % 10); v /= 10; } while (v);
    while (n) h = fnv_step(h, (uint32_t)buf[--n]);
  }
  return h;
}

// compare two candidate strings 32 characters at a time
__device__ inline bool cand_eq(const Mod& m, uint32_t s1, uint32_t r1, uint32_t s2, uint32_t r2) {
  const uint32_t total = cand_len(m, s1, r1);
  if (total != cand_len(m, s2, r2)) return false;
  uint32_t ba[32], bb[32];
  for (uint32_t from = 0; from < total; from += 32) {
    uint32_t na = 0, nb = 0, ia = 0, ib = 0;
    for_candidate(m, s1, r1, [&](uint32_t c) { if (ia >= from && na < 32) ba[na++] = c; ++ia; });
    for_candidate(m, s2, r2, [&](uint32_t c) { if (ib >= from && nb < 32) bb[nb++] = c; ++ib; });
    for (uint32_t q = 0; q < na; ++q) if (ba[q] != bb[q]) return false;
  }
  return true;
}

__device__ inline void resolve_names(Mod& m, const Tables& T) {
  const uint32_t lane = lane_id();
  // 1. per slot: named definition / pinned (P0 = A - named definitions)
  uint32_t nP0 = 0;
  for (uint32_t s = lane; s < m.S; s += 32) {
    uint8_t f = 0;
    if (m.hpres[s]) {
      bool named_d = m.hname[s] != NONE32 && m.hdef[s] != NONE32;
      if (named_d) f |= HF_NAMED_D;
      if (m.hA[s] && !named_d) { f |= HF_P0; ++nP0; }
    }
    m.hfl[s] = f;
  }
  nP0 = warp_sum_u32(nP0);
  __syncwarp();
  // 2. definitions in document order: C = D without P0 (index j in ib), named list ndl
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
    if (isC) m.ib[i] = cj + __popc(bc & below);
    if (isN) m.ndl[nd + __popc(bn & below)] = slot;
    if (i < m.I) m.iflag[i] = (m.iflag[i] & ~IF_FIRSTDEF) | (isC ? IF_FIRSTDEF : 0);
    cj += __popc(bc);
    nd += __popc(bn);
  }
  __syncwarp();
  // 3. closed form: pos[v] = -1 (P0) / j (c_j) / INF for v in [1, N]; prefix max; keep test.
  //    Values above N can never keep a name, so the array is N+1 <= S+1 long.
  const uint32_t N = nP0 + cj;
  const int32_t INF = 0x7FFFFFFF;
  for (uint32_t v = lane; v <= N; v += 32) m.pos[v] = INF;
  __syncwarp();
  for (uint32_t s = lane; s < m.S; s += 32) {
    if (!(m.hfl[s] & HF_P0)) continue;
    uint32_t key = slot_key(m, s);
    if (key >= 1 && key <= N) m.pos[key] = -1;
  }
  __syncwarp();
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane;
    if (i < m.I && (m.iflag[i] & IF_FIRSTDEF)) {
      uint32_t key = inst_ops(m, i)[T.has_rtype(m.idef[i]) ? 1 : 0];
      if (key >= 1 && key <= N) m.pos[key] = (int32_t)m.ib[i];
    }
  }
  __syncwarp();
  int32_t carry = -2;
  for (uint32_t base = 1; base <= N; base += 32) {
    uint32_t v = base + lane;
    int32_t x = v <= N ? m.pos[v] : -2;
    x = max(warp_incl_max(x), carry);
    if (v <= N) m.pos[v] = x;
    carry = __shfl_sync(FULL, x, 31);
  }
  __syncwarp();
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane;
    if (i < m.I && (m.iflag[i] & IF_FIRSTDEF)) {
      uint32_t key = inst_ops(m, i)[T.has_rtype(m.idef[i]) ? 1 : 0];
      int32_t j = (int32_t)m.ib[i];
      if (key >= 1 && key <= N && (key == 1 || m.pos[key - 1] < j)) m.hfl[ht_find(m, key)] |= HF_KEPT;
    }
  }
  __syncwarp();
  // 4. uniquify in D order (disasm.py:173-185): the k-th ident gets the first of
  //    base, base_0, base_1, ... not taken yet.  Exact reformulation: group idents
  //    by sanitized base; a candidate base_s can only collide with the *base* of
  //    another group that reads "base_<s>" (a child group), so a per-group counter
  //    plus per-group "base taken" flags reproduce the sequential result in one
  //    O(nd) pass; only grouping/child detection needs string compares.
  constexpr uint8_t HF_TB = 32, HF_HASCHILD = 64;
  for (uint32_t k = lane; k < nd; k += 32) {
    uint32_t slot = m.ndl[k];
    uint32_t h, len, ph;
    bool suffix;
    NameView nv = name_of(m, m.hname[slot]);
    name_info(nv, h, len, ph, suffix);
    m.nH[slot] = h; m.nP[slot] = ph; m.nLen[slot] = len;
    uint32_t n = NONE32;
    if (suffix) {   // numeric value of the canonical suffix (ignored if >= 2^32)
      uint64_t v = 0;
      uint32_t idx = 0, start = 0;
      for_sanitized(nv, [&](uint32_t c) { if (c == '_') start = idx + 1; ++idx; });
      idx = 0;
      for_sanitized(nv, [&](uint32_t c) { if (idx >= start && v <= 0xFFFFFFFFull) v = v * 10 + (c - '0'); ++idx; });
      if (v < 0xFFFFFFFFull) { n = (uint32_t)v; m.hfl[slot] |= HF_SUFFIX; }
    }
    m.ia[k] = n;
  }
  __syncwarp();
  // leader = first ident (D order) with the same sanitized base
  for (uint32_t k = lane; k < nd; k += 32) {
    uint32_t slot = m.ndl[k], h = m.nH[slot], lead = k;
    for (uint32_t q = 0; q < k; ++q) {
      uint32_t o = m.ndl[q];
      if (m.nH[o] == h && cand_eq(m, slot, NONE32, o, NONE32)) { lead = q; break; }
    }
    m.pos[k] = (int32_t)lead;
  }
  __syncwarp();
  // child groups: leader c whose base is "<base of leader g>_<n>"
  for (uint32_t k = lane; k < nd; k += 32) {
    uint32_t parent = NONE32;
    uint32_t slot = m.ndl[k];
    if (m.pos[k] == (int32_t)k && (m.hfl[slot] & HF_SUFFIX)) {
      const uint32_t ph = m.nP[slot], n = m.ia[k];
      for (uint32_t q = 0; q < nd && parent == NONE32; ++q) {
        uint32_t o = m.ndl[q];
        if (m.pos[q] != (int32_t)q || m.nH[o] != ph) continue;
        if (m.nLen[o] + 1 + dec_len_u64(n) != m.nLen[slot]) continue;
        // compare the first nLen[o] characters
        bool eq = true;
        const uint32_t L = m.nLen[o];
        uint32_t ba[32], bb[32];
        for (uint32_t from = 0; from < L && eq; from += 32) {
          uint32_t na = 0, nb = 0, ia = 0, ib = 0;
          for_sanitized(name_of(m, m.hname[slot]), [&](uint32_t c) { if (ia >= from && ia < L && na < 32) ba[na++] = c; ++ia; });
          for_sanitized(name_of(m, m.hname[o]), [&](uint32_t c) { if (ib >= from && nb < 32) bb[nb++] = c; ++ib; });
          for (uint32_t z = 0; z < na; ++z) if (ba[z] != bb[z]) { eq = false; break; }
        }
        if (eq) parent = q;
      }
    }
    m.ib[k] = parent;
  }
  __syncwarp();
  for (uint32_t k = lane; k < nd; k += 32) {
    if (m.ib[k] != NONE32) {
      uint8_t* f = &m.hfl[m.ndl[m.ib[k]]];
      atomicOr(reinterpret_cast<unsigned int*>(reinterpret_cast<uintptr_t>(f) & ~(uintptr_t)3),
               (unsigned)HF_HASCHILD << (8 * (reinterpret_cast<uintptr_t>(f) & 3)));
    }
  }
  __syncwarp();
  if (lane == 0) {
    auto child_of = [&](uint32_t g, uint32_t s) -> uint32_t {
      for (uint32_t q = 0; q < nd; ++q)
        if (m.ib[q] == g && m.ia[q] == s) return q;
      return NONE32;
    };
    for (uint32_t k = 0; k < nd; ++k) {
      const uint32_t g = (uint32_t)m.pos[k];
      const uint32_t gs = m.ndl[g];
      if (g == k) m.nP[gs] = 0;                       // group counter (nP no longer needed)
      uint32_t serial = NONE32;
      if (!(m.hfl[gs] & HF_TB)) {
        m.hfl[gs] |= HF_TB;
      } else {
        uint32_t sv = m.nP[gs];
        if (m.hfl[gs] & HF_HASCHILD) {
          uint32_t c;
          while ((c = child_of(g, sv)) != NONE32 && (m.hfl[m.ndl[c]] & HF_TB)) ++sv;
          if (c != NONE32) m.hfl[m.ndl[c]] |= HF_TB;  // our candidate is that child's base
        }
        serial = sv;
        m.nP[gs] = sv + 1;
      }
      m.hser[m.ndl[k]] = serial;
    }
  }
  __syncwarp();
  // 5. friendly = named definition that keeps its number; cache its ref length
  for (uint32_t k = lane; k < nd; k += 32) {
    uint32_t slot = m.ndl[k];
    if (m.hfl[slot] & HF_KEPT) {
      m.hfl[slot] |= HF_FRIENDLY;
      uint32_t rl = 1 + cand_len(m, slot, m.hser[slot]);
      m.hrl[slot] = (uint16_t)(rl > 0xFFFF ? 0xFFFF : rl);
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
// Coalesced copy of staged text: shared `stage` holds bytes for global [g0, g1)
// starting at stage + (g0 & 15), so 16-byte blocks line up on both sides.
__device__ inline void flush_stage(uint8_t* g0, uint8_t* g1, const uint8_t* stage) {
  const uint32_t lane = lane_id();
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(g0), a1 = reinterpret_cast<uintptr_t>(g1);
  const uint8_t* src = stage + (a0 & 15);
  uintptr_t m0 = (a0 + 15) & ~(uintptr_t)15, m1 = a1 & ~(uintptr_t)15;
  if (m0 >= m1) {   // no full block
    for (uintptr_t x = a0 + lane; x < a1; x += 32) *reinterpret_cast<uint8_t*>(x) = src[x - a0];
    return;
  }
  if (a0 + lane < m0) *reinterpret_cast<uint8_t*>(a0 + lane) = src[lane];
  if (m1 + lane < a1) *reinterpret_cast<uint8_t*>(m1 + lane) = src[m1 - a0 + lane];
  const uint32_t nb = (uint32_t)((m1 - m0) >> 4);
  const uint4* s4 = reinterpret_cast<const uint4*>(src + (m0 - a0));
  uint4* d4 = reinterpret_cast<uint4*>(m0);
  for (uint32_t k = lane; k < nb; k += 32) d4[k] = s4[k];
}

// one text line (with its optional preceding blank line) into sink-space at `lo`
template <class S>
__device__ inline void write_line(S& ms, const Mod& m, const Tables& T, uint32_t i, uint32_t width,
                                  bool hl) {
  if (m.iflag[i] & IF_HAS_RESULT) {
    uint32_t rl = m.irl[i] == 0xFFFF ? ref_len(m, m.ib[i]) : m.irl[i];
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

// ============================================================================
// Token pipeline.  Per chunk of 32 instructions: every lane walks its
// instruction once and emits compact tokens (with exact byte lengths) into
// shared memory; a warp scan places the lines; then the tokens of the chunk are
// rendered cooperatively (token t -> lane t % 32; strings and padding are split
// into <= 16-byte pieces so lanes get similar work) into a shared staging buffer
// that is flushed with 16-byte stores.
enum : uint32_t {
  K_TAB = 0, K_OPNAME = 1, K_REF = 2, K_DEC = 3, K_SIDE = 4, K_STR = 5, K_HEX = 6, K_UNKW = 7,
  K_UNKOP = 8, K_PAD = 9, K_EQ = 10, K_NL = 11, K_ZERO = 12
};
enum : uint32_t { F_SP = 1, F_BAR = 2, F_QOPEN = 4, F_QCLOSE = 8 };
constexpr int TOKMAX = 12;
constexpr int SIDEMAX = 2;
constexpr uint32_t PIECE = 16;
constexpr uint32_t RENDER_MIN = 32 * TOKMAX * 8 + 32 * SIDEMAX * 16 + 3 * 33 * 4 + 16 + 3072;

struct RenderWS {
  uint2* tok;         // [32][TOKMAX]
  uint4* side;        // [32][SIDEMAX]: u64 value, u32 exp, u32 kind|neg<<8
  uint32_t* ntok;     // [32]
  uint32_t* lstart;   // [33] line start within the chunk
  uint32_t* tpre;     // [33] token prefix counts of a line window
  uint8_t* stage;
  uint32_t stage_bytes;
};

__device__ inline RenderWS carve_ws(const Mod& m) {
  RenderWS r;
  uint8_t* p = m.work;
  r.tok = reinterpret_cast<uint2*>(p); p += 32 * TOKMAX * 8;
  r.side = reinterpret_cast<uint4*>(p); p += 32 * SIDEMAX * 16;
  r.ntok = reinterpret_cast<uint32_t*>(p); p += 33 * 4;
  r.lstart = reinterpret_cast<uint32_t*>(p); p += 33 * 4;
  r.tpre = reinterpret_cast<uint32_t*>(p); p += 33 * 4;
  p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~(uintptr_t)15);
  r.stage = p;
  r.stage_bytes = (uint32_t)(m.work + m.work_bytes - p);
  return r;
}

// per-lane token emitter (also the walk visitor)
struct TokEmit {
  const Mod& m;
  const Tables& T;
  uint2* tok;        // this lane's TOKMAX slots
  uint4* side;       // this lane's SIDEMAX slots
  uint32_t side_base;
  bool hl;
  uint32_t n = 0, nside = 0, len = 0;
  bool overflow = false;   // too many tokens / needs look-ahead: lane renders directly
  bool have_set = false;
  uint32_t set_id = 0;
  int8_t ext_known = -1;   // -1 unknown yet

  __device__ TokEmit(const Mod& m_, const Tables& T_, uint2* t, uint4* sd, uint32_t sb, bool h)
      : m(m_), T(T_), tok(t), side(sd), side_base(sb), hl(h) {}

  __device__ void add(uint32_t kind, uint32_t flags, uint32_t tlen, uint32_t payload) {
    if (n >= (uint32_t)TOKMAX || len > 0xFFF || tlen > 0xFFF) { overflow = true; return; }
    tok[n++] = make_uint2(kind | (flags << 4) | (tlen << 8) | (len << 20), payload);
    len += tlen;
  }
  __device__ uint32_t add_side(uint64_t v, uint32_t x, uint32_t kind) {
    if (nside >= (uint32_t)SIDEMAX) { overflow = true; return 0; }
    side[nside] = make_uint4((uint32_t)v, (uint32_t)(v >> 32), x, kind);
    return side_base + nside++;
  }
  __device__ void pad(uint32_t k) {
    while (k > 0) { uint32_t c = k > PIECE ? PIECE : k; add(K_PAD, 0, c, c); k -= c; }
  }
  __device__ uint32_t color() const { return hl ? 9 : 0; }

  // walk visitor -------------------------------------------------------------
  __device__ void id(uint32_t role, uint32_t v, int depth) {
    if (depth == 0 && role == IDR_RESULT) return;                 // emitted in the prefix
    if (depth == 0 && role == IDR_ID && !have_set) { have_set = true; set_id = v; }
    if (role == IDR_RESULT) { add(K_DEC, F_SP, 1 + dec_len_u64(v), v); return; }
    add(K_REF, F_SP, 1 + ref_len(m, v) + color(), v);
  }
  __device__ void venum(uint32_t, uint32_t v, uint32_t e) {
    if (e != NONE32) add(K_TAB, F_SP, 1 + T.ename_len(e), T.ename_off(e) | (T.ename_len(e) << 24));
    else add(K_DEC, F_SP, 1 + dec_len_u64(v), v);
  }
  __device__ void benum(uint32_t k, uint32_t mask, bool full, uint64_t comp) {
    if (mask == 0) {
      uint32_t z = T.kzero(k);
      if (z != NONE32) add(K_TAB, F_SP, 1 + T.ename_len(z), T.ename_off(z) | (T.ename_len(z) << 24));
      else add(K_ZERO, F_SP, 2, 0);
      return;
    }
    if (!full) {
      uint32_t hd = 1;
      for (uint32_t x = mask >> 4; x; x >>= 4) ++hd;
      add(K_HEX, F_SP, 3 + hd, mask);
      return;
    }
    uint32_t eo = T.kenum_off(k);
    bool first = true;
    for (int j = 0; j < 64; ++j) {
      if (!((comp >> j) & 1)) continue;
      uint32_t e = eo + j;
      add(K_TAB, first ? F_SP : F_BAR, 1 + T.ename_len(e), T.ename_off(e) | (T.ename_len(e) << 24));
      first = false;
    }
  }
  __device__ void str(const uint32_t* ops, uint32_t pos, uint32_t nbytes) {
    const uint32_t base = (uint32_t)((ops + pos - m.w) * 4);   // byte offset in the module
    uint32_t done = 0;
    do {
      uint32_t c = nbytes - done > PIECE ? PIECE : nbytes - done;
      uint32_t fl = (done == 0 ? F_QOPEN | F_SP : 0) | (done + c == nbytes ? F_QCLOSE : 0);
      uint32_t tl = c;
      for (uint32_t q = 0; q < c; ++q) {
        uint32_t b = byte_at(m.w, base + done + q);
        if (b == '\\' || b == '"') ++tl;
      }
      if (fl & F_QOPEN) tl += 2 + (hl ? 5 : 0);
      if (fl & F_QCLOSE) tl += 1 + (hl ? 4 : 0);
      add(K_STR, fl, tl, (base + done) | (c << 24));
      done += c;
    } while (done < nbytes);
    if (base + nbytes >= (1u << 24)) overflow = true;
  }
  __device__ void typed(const LitVal& lv) {
    if (lv.flt) {
      FloatParts p = repr_parts(lv.bits);
      uint32_t sl = add_side(p.digits, (uint32_t)p.exp, 2 | ((uint32_t)p.kind << 8) | ((p.neg ? 1u : 0u) << 16));
      add(K_SIDE, F_SP, 1 + repr_len(p), sl);
    } else if (lv.neg) {
      uint32_t sl = add_side(lv.bits, 0, 0);
      add(K_SIDE, F_SP, 2 + dec_len_u64((uint64_t)0 - lv.bits), sl);
    } else if (lv.bits >> 32) {
      uint32_t sl = add_side(lv.bits, 0, 1);
      add(K_SIDE, F_SP, 1 + dec_len_u64(lv.bits), sl);
    } else {
      add(K_DEC, F_SP, 1 + dec_len_u64(lv.bits), (uint32_t)lv.bits);
    }
  }
  __device__ void lit(uint32_t sub, uint32_t v) {
    if (sub == LIT_EXTINST) {
      if (ext_known < 0) {
        if (!have_set) { overflow = true; return; }          // reference looks ahead
        ext_known = is_opencl_std(m, T, set_id) ? 1 : 0;
      }
      uint32_t off, ln;
      if (ext_known && T.ext_name(v, off, ln)) { add(K_TAB, F_SP, 1 + ln, off | (ln << 24)); return; }
    } else if (sub == LIT_SPECOP) {
      uint32_t d = T.inst_of(v);
      if (d != NONE32) {
        uint32_t ln = T.iname_len(d) - 2;
        add(K_TAB, F_SP, 1 + ln, (T.iname_off(d) + 2) | (ln << 24));
        return;
      }
    }
    add(K_DEC, F_SP, 1 + dec_len_u64(v), v);
  }
  __device__ void comp_begin() {}
  __device__ void comp_end() {}
};

// render one token at `dst` (shared staging or global)
__device__ inline void render_token(uint8_t* dst, uint2 tk, const Mod& m, const Tables& T,
                                    const uint4* side, bool hl) {
  const uint32_t kind = tk.x & 15, fl = (tk.x >> 4) & 15;
  MemSink s(dst);
  if (fl & F_SP) s.put(' ');
  if (fl & F_BAR) s.put('|');
  switch (kind) {
    case K_TAB: {
      const uint8_t* src = T.str + (tk.y & 0xFFFFFF);
      const uint32_t ln = tk.y >> 24;
      for (uint32_t q = 0; q < ln; ++q) s.put(__ldg(src + q));
      break;
    }
    case K_OPNAME: {
      if (hl) put_cstr(s, ANSI_OPCODE);
      const uint8_t* src = T.str + (tk.y & 0xFFFFFF);
      const uint32_t ln = tk.y >> 24;
      for (uint32_t q = 0; q < ln; ++q) s.put(__ldg(src + q));
      if (hl) put_cstr(s, ANSI_RESET);
      break;
    }
    case K_REF:
      if (hl) put_cstr(s, ANSI_ID);
      put_ref(s, m, tk.y);
      if (hl) put_cstr(s, ANSI_RESET);
      break;
    case K_DEC: put_u64(s, tk.y); break;
    case K_SIDE: {
      uint4 sd = side[tk.y];
      uint64_t v = (uint64_t)sd.x | ((uint64_t)sd.y << 32);
      uint32_t k = sd.w & 0xFF;
      if (k == 0) put_i64(s, (int64_t)v);
      else if (k == 1) put_u64(s, v);
      else {
        FloatParts p;
        p.digits = v; p.exp = (int32_t)sd.z; p.kind = (uint8_t)((sd.w >> 8) & 0xFF); p.neg = (sd.w >> 16) & 1;
        put_repr_parts(s, p);
      }
      break;
    }
    case K_STR: {
      if (fl & F_QOPEN) { if (hl) put_cstr(s, ANSI_STRING); s.put('"'); }
      const uint32_t b0 = tk.y & 0xFFFFFF, c = tk.y >> 24;
      for (uint32_t q = 0; q < c; ++q) {
        uint32_t b = byte_at(m.w, b0 + q);
        if (b == '\\' || b == '"') s.put('\\');
        s.put((uint8_t)b);
      }
      if (fl & F_QCLOSE) { s.put('"'); if (hl) put_cstr(s, ANSI_RESET); }
      break;
    }
    case K_HEX: put_hex_lower(s, tk.y); break;
    case K_UNKW: s.put('!'); s.put('0'); s.put('x'); put_hex8_upper(s, tk.y); break;
    case K_UNKOP:
      if (hl) put_cstr(s, ANSI_OPCODE);
      put_cstr(s, "OpUnknown("); put_u64(s, tk.y); s.put(')');
      if (hl) put_cstr(s, ANSI_RESET);
      break;
    case K_PAD: for (uint32_t q = 0; q < tk.y; ++q) s.put(' '); break;
    case K_EQ: s.put(' '); s.put('='); s.put(' '); break;
    case K_NL: s.put('\n'); break;
    case K_ZERO: s.put('0'); break;
    default: break;
  }
}

// Emit the tokens of instruction i's text line.  Returns the walk status;
// e.overflow asks the caller to render this line directly.
__device__ inline WalkErr emit_line(TokEmit& e, const Mod& m, const Tables& T, uint32_t i,
                                    uint32_t width, bool blank) {
  if (blank) e.add(K_NL, 0, 1, 0);
  const uint32_t d = m.idef[i];
  const uint32_t* ops = inst_ops(m, i);
  const uint32_t n = inst_nops(m, i);
  if (m.iflag[i] & IF_HAS_RESULT) {
    uint32_t rl = m.irl[i] == 0xFFFF ? ref_len(m, m.ib[i]) : m.irl[i];
    if (width) e.pad(width - rl);
    e.add(K_REF, 0, rl + e.color(), m.ib[i]);
    e.add(K_EQ, 0, 3, 0);
  } else if (width) {
    e.pad(width + 3);
  }
  WalkErr err;
  if (d == NONE16) {
    uint32_t op = inst_opcode(m, i);
    e.add(K_UNKOP, 0, 11 + dec_len_u64(op) + e.color(), op);
    for (uint32_t k = 0; k < n; ++k) e.add(K_UNKW, F_SP, 12, ops[k]);
  } else {
    uint32_t ln = T.iname_len(d);
    e.add(K_OPNAME, 0, ln + e.color(), T.iname_off(d) | (ln << 24));
    Resolver res{&m, &T};
    err = walk(T, d, ops, n, e, res);
  }
  e.add(K_NL, 0, 1, 0);
  return err;
}

// result ref of every instruction -> irl/ib/iflag, module width (disasm.py:286-288)
__device__ inline uint32_t result_refs(Mod& m, const Tables& T) {
  uint32_t width = 0;
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane_id();
    if (i >= m.I) continue;
    uint8_t fl = m.iflag[i] & ~IF_HAS_RESULT;
    uint32_t d = m.idef[i];
    if (d != NONE16 && T.has_result(d)) {
      uint32_t idx = T.has_rtype(d) ? 1 : 0;
      if (idx < inst_nops(m, i)) {
        uint32_t id = inst_ops(m, i)[idx];
        uint32_t rl = ref_len(m, id);
        m.ib[i] = id;
        m.irl[i] = (uint16_t)(rl > 0xFFFF ? 0xFFFF : rl);
        fl |= IF_HAS_RESULT;
        width = max(width, rl);
      }
    }
    m.iflag[i] = fl;
  }
  return warp_max_u32(width);
}

// Coalesced 16-byte-aligned copy (dst and src both 16-byte aligned, bytes any).
__device__ inline void warp_copy16(uint8_t* dst, const uint8_t* src, uint64_t bytes) {
  const uint32_t lane = lane_id();
  const uint64_t nb = bytes >> 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (uint64_t k = lane; k < nb; k += 32) __stcs(d4 + k, __ldcg(s4 + k));
  for (uint64_t k = nb * 16 + lane; k < bytes; k += 32) dst[k] = src[k];
}

// Render the module text into `gtext` (per-warp scratch, capacity gcap) with
// the token pipeline.  Returns the text length, or NONE64 when the scratch is
// too small (caller falls back); sets `bad` to the first failing instruction.
constexpr uint64_t NONE64 = ~0ull;

__device__ inline uint64_t token_text(const Mod& m, const Tables& T, uint32_t opts, uint32_t width,
                                      uint8_t* gtext, uint64_t gcap, uint32_t& bad) {
  const uint32_t lane = lane_id();
  const bool hl = opts & OPT_HIGHLIGHT, group = opts & OPT_GROUP;
  RenderWS ws = carve_ws(m);
  bad = NONE32;
  uint64_t pos = 0;
  // header lines
  if (!(opts & OPT_NO_HEADER)) {
    CountSink hs;
    put_header(hs, m, hl);
    if (hs.n > gcap) return NONE64;
    if (lane == 0) { MemSink ms(gtext); put_header(ms, m, hl); }
    pos = hs.n;
  }
  for (uint32_t base = 0; base < m.I; base += 32) {
    const uint32_t i = base + lane;
    const bool act = i < m.I;
    // 1. emit
    TokEmit e(m, T, ws.tok + lane * TOKMAX, ws.side + lane * SIDEMAX, lane * SIDEMAX, hl);
    WalkErr err;
    bool direct = false;
    uint32_t llen = 0;
    if (act) {
      const bool blank = group && i > 0 && m.isec[i] != m.isec[i - 1];
      err = emit_line(e, m, T, i, width, blank);
      if (m.idef[i] == NONE16 && (opts & OPT_STRICT)) err.code = 0xFF;
      if (e.overflow && err.code == W_OK) {
        direct = true;
        CountSink cs;
        if (blank) cs.put('\n');
        write_line(cs, m, T, i, width, hl);
        llen = cs.n;
      } else {
        llen = e.len;
      }
    }
    unsigned eb = __ballot_sync(FULL, act && err.code != W_OK);
    if (eb) { bad = base + __ffs(eb) - 1; return 0; }
    ws.ntok[lane] = (act && !direct) ? e.n : 0;
    // 2. place lines
    uint32_t incl = warp_incl_sum(llen);
    ws.lstart[lane] = incl - llen;
    const uint32_t chunk = __shfl_sync(FULL, incl, 31);
    if (lane == 31) ws.lstart[32] = incl;
    if (pos + chunk > gcap) return NONE64;
    __syncwarp();
    // 3. render line windows that fit the staging buffer
    uint32_t l0 = 0;
    while (l0 < 32) {
      const uint32_t w0 = ws.lstart[l0];
      const uint64_t g0 = pos + w0;
      const uint32_t shift = (uint32_t)(g0 & 15);
      uint32_t l1 = l0;
      while (l1 < 32 && ws.lstart[l1 + 1] - w0 + shift <= ws.stage_bytes) ++l1;
      if (l1 == l0) {
        // a single line larger than the staging buffer: write it straight to gtext
        if (lane == l0 && base + l0 < m.I) {
          MemSink ms(gtext + g0);
          const uint32_t ii = base + l0;
          if (group && ii > 0 && m.isec[ii] != m.isec[ii - 1]) ms.put('\n');
          write_line(ms, m, T, ii, width, hl);
        }
        __syncwarp();
        ++l0;
        continue;
      }
      uint8_t* st = ws.stage + shift - w0;   // staging pointer for chunk offset 0
      // token prefix over the window
      uint32_t cnt = (lane >= l0 && lane < l1) ? ws.ntok[lane] : 0;
      uint32_t tin = warp_incl_sum(cnt);
      ws.tpre[lane] = tin - cnt;
      const uint32_t ntot = __shfl_sync(FULL, tin, 31);
      __syncwarp();
      for (uint32_t t = lane; t < ntot; t += 32) {
        // owning line: largest l in [l0, l1) with tpre[l] <= t
        uint32_t lo = l0, hi = l1 - 1;
        while (lo < hi) {
          uint32_t mid = (lo + hi + 1) >> 1;
          if (ws.tpre[mid] <= t) lo = mid; else hi = mid - 1;
        }
        const uint2 tk = ws.tok[lo * TOKMAX + (t - ws.tpre[lo])];
        render_token(st + ws.lstart[lo] + (tk.x >> 20), tk, m, T, ws.side, hl);
      }
      // directly rendered lines of the window
      if (lane >= l0 && lane < l1 && act && ws.ntok[lane] == 0) {
        MemSink ms(st + ws.lstart[lane]);
        if (group && i > 0 && m.isec[i] != m.isec[i - 1]) ms.put('\n');
        write_line(ms, m, T, i, width, hl);
      }
      __syncwarp();
      flush_stage(gtext + g0, gtext + pos + ws.lstart[l1], ws.stage);
      __syncwarp();
      l0 = l1;
    }
    pos += chunk;
  }
  return pos;
}

// Fallback renderer (module text larger than the per-warp scratch): size pass
// with per-line lengths, then direct writes at the final position.
__device__ inline uint64_t legacy_size(Mod& m, const Tables& T, uint32_t opts, uint32_t width) {
  const bool hl = opts & OPT_HIGHLIGHT, group = opts & OPT_GROUP;
  CountSink hs;
  if (!(opts & OPT_NO_HEADER)) put_header(hs, m, hl);
  uint64_t run = hs.n;
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane_id();
    uint32_t len = 0;
    if (i < m.I) {
      CountSink cs;
      if (group && i > 0 && m.isec[i] != m.isec[i - 1]) cs.put('\n');
      write_line(cs, m, T, i, width, hl);
      len = cs.n;
    }
    uint32_t incl = warp_incl_sum(len);
    if (i < m.I) m.ia[i] = (uint32_t)(run + incl - len);
    run += __shfl_sync(FULL, incl, 31);
  }
  __syncwarp();
  return run;
}

__device__ inline void legacy_write(const Mod& m, const Tables& T, uint32_t opts, uint32_t width,
                                    uint8_t* out) {
  const bool hl = opts & OPT_HIGHLIGHT, group = opts & OPT_GROUP;
  if (lane_id() == 0 && !(opts & OPT_NO_HEADER)) { MemSink ms(out); put_header(ms, m, hl); }
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane_id();
    if (i >= m.I) continue;
    MemSink ms(out + m.ia[i]);
    if (group && i > 0 && m.isec[i] != m.isec[i - 1]) ms.put('\n');
    write_line(ms, m, T, i, width, hl);
  }
}

__device__ inline void report_internal(ErrSink& es, int32_t t, const char* what) {
  if (lane_id() == 0) {
    ErrRec* erec = es.alloc();
    if (erec) {
      ErrWriter ew{erec};
      put_cstr(ew, what);
      erec->module = t; erec->cls = ST_INTERNAL; erec->len = ew.n;
    }
  }
}

__global__ void __launch_bounds__(128) disasm_kernel(DisasmArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = lane_id();
  const uint32_t warp_in_block = threadIdx.x >> 5;
  const uint32_t gwarp = blockIdx.x * (blockDim.x >> 5) + warp_in_block;
  uint8_t* slab = smem + (size_t)warp_in_block * a.smem_slab;
  uint8_t* gslot = a.gscratch + (size_t)gwarp * a.gslot_bytes;
  uint8_t* gtext = a.gtext + (size_t)gwarp * a.gtext_bytes;
  const Tables& T = a.T;
  ErrSink es{a.errs, a.ticket + 1, a.err_cap};

  while (true) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1u);
    t = __shfl_sync(FULL, t, 0);
    if (t >= a.n_mod) break;
    const int64_t nbytes = a.mod_len[t];
    const uint8_t* src = a.data + a.mod_off[t];
    int32_t status = ST_OK;
    uint64_t total = 0;
    uint32_t width = 0;
    bool legacy = false;
    Mod m;
    const uint32_t W = (nbytes >= 0 && nbytes % 4 == 0) ? (uint32_t)(nbytes / 4) : 0;
    bool in_smem = head_bytes(W) <= a.smem_slab;
    if (!in_smem && worst_bytes(W, RENDER_MIN) > a.gslot_bytes) {
      status = ST_INTERNAL;
      report_internal(es, (int32_t)t, "internal: module exceeds the per-warp scratch slot");
    } else {
      layout_head(m, in_smem ? slab : gslot, W);
      status = load_and_split(m, src, (uint64_t)nbytes, &es, (int32_t)t);
    }
    if (status == ST_OK) {
      bool direct = m.bound <= 2 * m.W + 64;
      for (int attempt = 0; attempt < 2; ++attempt) {
        if (!place_tables(m, direct, in_smem, gslot, a.gslot_bytes, a.smem_slab, RENDER_MIN)) {
          status = ST_INTERNAL;
          report_internal(es, (int32_t)t, "internal: module exceeds the per-warp scratch slot");
          break;
        }
        init_tables(m);
        bool any_name = prescan(m, T);
        bool names_mode = (a.opts & OPT_INLINE) && any_name;
        if (names_mode && !*m.overflow) {
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
        if (*m.overflow) {   // an id at/above the bound: redo with the hash table
          __syncwarp();
          direct = false;
          continue;
        }
        // --- exceptions, in the reference's evaluation order ---
        uint32_t bad = first_where(m, [&](uint32_t i) { return (m.iflag[i] & IF_PRESCAN_UTF8) != 0; });
        if (bad != NONE32) {
          status = ST_UNICODE;
          if (lane == 0) report_prescan_error(m, T, bad, es.alloc(), (int32_t)t);
          break;
        }
        if (names_mode) {
          bad = first_where(m, [&](uint32_t i) { uint32_t e = m.ierr[i]; return e != W_OK && !werr_is_codec(e); });
          if (bad != NONE32) {
            if (lane == 0) report_inst_error(m, T, bad, es.alloc(), (int32_t)t, status);
            status = __shfl_sync(FULL, status, 0);
            break;
          }
          resolve_names(m, T);
        }
        width = result_refs(m, T);
        if (a.opts & OPT_NO_INDENT) width = 0;
        if (a.opts & OPT_GROUP) compute_sections(m, T);
        // render: token pipeline into the per-warp text scratch
        uint32_t badi = NONE32;
        total = token_text(m, T, a.opts, width, gtext, a.gtext_bytes, badi);
        if (badi != NONE32) {
          if (lane == 0) {
            ErrRec* erec = es.alloc();
            if (m.idef[badi] == NONE16) {
              status = ST_CODEC;
              if (erec) {
                ErrWriter ew{erec};
                put_cstr(ew, "unknown opcode "); put_u64(ew, inst_opcode(m, badi));
                erec->module = (int32_t)t; erec->cls = ST_CODEC; erec->len = ew.n;
              }
            } else {
              report_inst_error(m, T, badi, erec, (int32_t)t, status);
            }
          }
          status = __shfl_sync(FULL, status, 0);
          break;
        }
        if (total == NONE64) {            // scratch too small: two-pass fallback
          legacy = true;
          total = legacy_size(m, T, a.opts, width);
        }
        break;
      }
    }
    // reserve the module's bytes (16-byte aligned starts) and copy the text out
    if (status != ST_OK) total = 0;
    bool fits;
    uint64_t off = alloc_text(a.ticket, (total + 15) & ~15ull, a.text_cap, fits);
    if (lane == 0) {
      a.text_span[2 * t] = (int64_t)off;
      a.text_span[2 * t + 1] = (int64_t)total;
      a.status[t] = status;
    }
    if (status == ST_OK && total > 0 && fits) {
      if (legacy) legacy_write(m, T, a.opts, width, a.text + off);
      else warp_copy16(a.text + off, gtext, total);
    }
    __syncwarp();
  }
}

}  // namespace skg
