// Batch disassembler: binary modules -> text, bit-exact with the reference
// Disassembler.to_text (disasm.py:117-127, 131-377).
//
// Persistent warps take module tickets (atomic counter).  Per module:
//   load/boundary -> prescan -> classify (ONE grammar walk per instruction,
//   tagging every operand word with a render code) -> [names mode: referenced
//   ids collected word-parallel + friendly-name resolution] -> result refs and
//   width -> word-parallel length pass -> bump allocation of the module's bytes
//   -> word-parallel write pass through a shared-memory stage flushed with
//   16-byte stores.  Lanes work on consecutive operand words, so the common
//   one-word operands (ids, enums, literals, 4 string bytes) render with
//   nearly uniform work per lane.  The text of module m is
//   text[span[2m] : span[2m] + span[2m+1]].
#include "skg_module.cuh"

namespace skg {

enum : uint32_t { OPT_HIGHLIGHT = 1, OPT_INLINE = 2, OPT_NO_INDENT = 4, OPT_GROUP = 8,
                  OPT_NO_HEADER = 16, OPT_STRICT = 32 };

__device__ const char* const ANSI_OPCODE = "\x1b[36m";
__device__ const char* const ANSI_ID = "\x1b[33m";
__device__ const char* const ANSI_STRING = "\x1b[32m";
__device__ const char* const ANSI_COMMENT = "\x1b[90m";
__device__ const char* const ANSI_RESET = "\x1b[0m";

constexpr uint32_t RENDER_MIN = 0;      // the text stage is separate shared memory

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
  uint32_t smem_slab;         // bytes per warp in dynamic shared memory (module scratch)
  uint32_t stage_bytes;       // bytes per warp of text stage (dynamic shared memory, first)
  const uint32_t* order;      // ticket -> module index (skg_sched.cuh)
  uint32_t group_warps;       // warps per phase-barrier group (divides the CTA's warps)
  const uint32_t* ovr;        // explicit refs (Mod::ovr), n_ovr entries; nullptr = none
  const uint8_t* ovr_text;
  uint32_t n_ovr;
  // fused validation (pipeline_kernel): the validate_kernel outputs
  uint8_t* vtext;
  uint64_t vtext_cap;
  int64_t* vspan;
  int32_t* vstatus;
  uint32_t* vctr;             // [1] error records, [2] overflow, [4..5] cursor
  ErrRec* verrs;
  uint32_t verr_cap;
};

// -- sanitized friendly names (disasm.py:82-86) --------------------------------
struct NameView {
  const uint32_t* w;   // string words
  uint32_t nbytes;
};

__device__ __noinline__ NameView name_of(const Mod& m, uint32_t name_inst) {
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
  #pragma unroll 1
  for (uint32_t i = 0; i < nv.nbytes; ++i) {
    uint32_t c = byte_at(nv.w, i);
    if ((c & 0xC0) != 0x80) { first = c; break; }
  }
  bool prefix = first == 0xFFFFFFFF || (first >= '0' && first <= '9');
  if (prefix) f('_');
  // one word load per 4 bytes
  #pragma unroll 1
  for (uint32_t i = 0; i < nv.nbytes; i += 4) {
    const uint32_t x = nv.w[i >> 2];
    const uint32_t nb = min(4u, nv.nbytes - i);
    #pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
      if (q < nb) {
        const uint32_t c = (x >> (8 * q)) & 0xFF;
        if ((c & 0xC0) != 0x80) f(is_word_char(c) ? c : '_');
      }
    }
  }
}

// -- ref lengths ----------------------------------------------------------------
// friendly ids render as '%' + sanitized base (narena) + ['_' + serial]
__device__ __forceinline__ uint32_t dlen32(uint32_t v) {
  return v < 10 ? 1 : v < 100 ? 2 : v < 1000 ? 3 : v < 10000 ? 4 : v < 100000 ? 5 :
         v < 1000000 ? 6 : v < 10000000 ? 7 : v < 100000000 ? 8 : v < 1000000000 ? 9 : 10;
}

// per-slot ref text lengths for direct-mode modules (P5, before any length is needed)
__device__ __noinline__ void fill_ref_lengths(Mod& m);

// explicit ref of `id` (Mod::ovr): entry index or NONE32
__device__ __noinline__ uint32_t ovr_find(const Mod& m, uint32_t id) {
  uint32_t lo = 0, hi = m.n_ovr;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint32_t v = m.ovr[3 * mid];
    if (v == id) return mid;
    if (v < id) lo = mid + 1; else hi = mid;
  }
  return NONE32;
}

__device__ __forceinline__ uint32_t ref_len_slow(const Mod& m, uint32_t id) {
  if (m.n_ovr) {
    const uint32_t k = ovr_find(m, id);
    if (k != NONE32) return m.ovr[3 * k + 2];
  }
  const uint32_t slot = ht_find(m, id);
  if (slot != NONE32 && (m.hfl[slot] & HF_FRIENDLY)) {
    const uint32_t ser = m.hser[slot];
    return 1 + m.nLen[slot] + (ser != NONE32 ? 1 + dlen32(ser) : 0);
  }
  return 1 + dlen32(id);
}

__device__ __forceinline__ uint32_t ref_len(const Mod& m, uint32_t id) {
  if (m.direct && id < m.S) { const uint32_t r = m.hrl[id]; if (r != 0xFFFF) return r; }
  return ref_len_slow(m, id);
}

__device__ __noinline__ void fill_ref_lengths(Mod& m) {
  if (!m.direct) return;
  for (uint32_t s = lane_id(); s < m.S; s += 32) {
    const uint32_t r = ref_len_slow(m, s);
    m.hrl[s] = (uint16_t)(r > 0xFFFE ? 0xFFFF : r);
  }
  __syncwarp();
}

__device__ __noinline__ bool is_opencl_std(const Mod& m, const Tables& T, uint32_t set_id) {
  uint32_t s = ht_find(m, set_id);
  if (s == NONE32 || m.himp[s] == NONE32) return false;
  NameView nv = name_of(m, m.himp[s]);
  if (nv.nbytes != T.ocl_len) return false;
  #pragma unroll 1
  for (uint32_t i = 0; i < nv.nbytes; ++i)
    if (byte_at(nv.w, i) != T.str[T.ocl_off + i]) return false;
  return true;
}

// ----------------------------------------------------------------------------
// friendly names: uniquify (disasm.py:173-185) + closed-form demotion
__device__ inline uint32_t fnv_step(uint32_t h, uint32_t c) { return (h ^ c) * 16777619u; }

constexpr uint8_t HF_SUFFIX = 16;

// hash + length + "ends with _<canonical int>" info of a sanitized name
__device__ __noinline__ void name_info(const NameView& nv, uint32_t& h, uint32_t& len, uint32_t& ph,
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
    #pragma unroll 1
    do { buf[q++] = (char)('0' + v % 10); v /= 10; } while (v);
    #pragma unroll 1
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
    #pragma unroll 1
    do { buf[n++] = (char)('0' + v % 10); v /= 10; } while (v);
    #pragma unroll 1
    while (n) h = fnv_step(h, (uint32_t)buf[--n]);
  }
  return h;
}

// compare two candidate strings 32 characters at a time
__device__ __noinline__ bool cand_eq(const Mod& m, uint32_t s1, uint32_t r1, uint32_t s2, uint32_t r2) {
  const uint32_t total = cand_len(m, s1, r1);
  if (total != cand_len(m, s2, r2)) return false;
  uint32_t ba[32], bb[32];
  #pragma unroll 1
  for (uint32_t from = 0; from < total; from += 32) {
    uint32_t na = 0, nb = 0, ia = 0, ib = 0;
    for_candidate(m, s1, r1, [&](uint32_t c) { if (ia >= from && na < 32) ba[na++] = c; ++ia; });
    for_candidate(m, s2, r2, [&](uint32_t c) { if (ib >= from && nb < 32) bb[nb++] = c; ++ib; });
    #pragma unroll 1
    for (uint32_t q = 0; q < na; ++q) if (ba[q] != bb[q]) return false;
  }
  return true;
}

// ---- friendly names, per-item steps (shared by the warp driver resolve_names
// and the grid-wide driver of one large module) -------------------------------
constexpr uint8_t HF_TB = 32, HF_HASCHILD = 64;

// step 1 (slot s): named definition / pinned (P0 = referenced ids that are not
// named definitions); returns whether s is P0
__device__ __forceinline__ bool nm_slot_flags(Mod& m, uint32_t s) {
  uint8_t f = 0;
  if (m.hpres[s]) {
    const bool named_d = m.hname[s] != NONE32 && m.hdef[s] != NONE32;
    if (named_d) f |= HF_NAMED_D;
    if (m.hA[s] && !named_d) f |= HF_P0;
  }
  m.hfl[s] = f;
  return f & HF_P0;
}

// step 2 (instruction i): first definition of its result id: in C (= D without
// P0) and / or a named definition
__device__ __forceinline__ void nm_def_pred(const Mod& m, const Tables& T, uint32_t i, bool& isC, bool& isN,
                                            uint32_t& slot) {
  isC = isN = false;
  slot = NONE32;
  const uint32_t d = m.idef[i];
  if (d == NONE16 || !T.has_result(d)) return;
  const uint32_t idx = T.has_rtype(d) ? 1 : 0;
  if (idx >= inst_nops(m, i)) return;
  slot = ht_find(m, inst_ops(m, i)[idx]);
  if (slot != NONE32 && m.hdef[slot] == i) {
    isC = !(m.hfl[slot] & HF_P0);
    isN = (m.hfl[slot] & HF_NAMED_D) != 0;
  }
}

__device__ __forceinline__ uint32_t nm_def_key(const Mod& m, const Tables& T, uint32_t i) {
  return inst_ops(m, i)[T.has_rtype(m.idef[i]) ? 1 : 0];
}

// step 4 (named definition k): sanitized-name hash / prefix hash / length and
// the numeric value of a canonical "_<n>" suffix
__device__ __forceinline__ void nm_info(Mod& m, uint32_t k) {
  const uint32_t slot = m.ndl[k];
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

// base-hash table (key, smallest ident index), open addressing, in the spill area
__device__ __forceinline__ uint32_t nm_hkey(uint32_t h) { return h == EMPTY ? EMPTY - 1 : h; }

__device__ __forceinline__ void nm_hinsert(uint32_t* htab, uint32_t C, uint32_t h, uint32_t k) {
  const uint32_t key = nm_hkey(h);
  uint32_t e = (key * 0x9E3779B1u) & (C - 1);
  #pragma unroll 1
  while (true) {
    const uint32_t old = atomicCAS(&htab[2 * e], EMPTY, key);
    if (old == EMPTY || old == key) { atomicMin(&htab[2 * e + 1], k); return; }
    e = (e + 1) & (C - 1);
  }
}

__device__ __forceinline__ uint32_t nm_hmin(const uint32_t* htab, uint32_t C, uint32_t h) {
  const uint32_t key = nm_hkey(h);
  uint32_t e = (key * 0x9E3779B1u) & (C - 1);
  #pragma unroll 1
  while (true) {   // L2 reads: the table was filled with atomics (not in L1)
    const uint32_t kk = __ldcg(htab + 2 * e);
    if (kk == key) return __ldcg(htab + 2 * e + 1);
    if (kk == EMPTY) return NONE32;
    e = (e + 1) & (C - 1);
  }
}

// leader of ident k = first ident (D order) with the same sanitized base
__device__ __noinline__ uint32_t nm_leader(const Mod& m, const uint32_t* htab, uint32_t C, uint32_t k) {
  const uint32_t slot = m.ndl[k], h = m.nH[slot];
  uint32_t lead = nm_hmin(htab, C, h);
  if (lead != k && !(lead < k && cand_eq(m, slot, NONE32, m.ndl[lead], NONE32))) {
    lead = k;   // hash collision with another base: exact ordered scan
    #pragma unroll 1
    for (uint32_t q = 0; q < k; ++q) {
      const uint32_t o = m.ndl[q];
      if (m.nH[o] == h && cand_eq(m, slot, NONE32, o, NONE32)) { lead = q; break; }
    }
  }
  return lead;
}

// parent group of leader k whose base reads "<base of the parent>_<n>", or NONE32
__device__ __noinline__ uint32_t nm_parent(const Mod& m, const uint32_t* htab, uint32_t C, uint32_t nd,
                                           uint32_t k) {
  uint32_t parent = NONE32;
  const uint32_t slot = m.ndl[k];
  if (m.pos[k] != (int32_t)k || !(m.hfl[slot] & HF_SUFFIX)) return NONE32;
  const uint32_t ph = m.nP[slot], n = m.ia[k];
  // the parent (if any) is the leader of base hash ph: try the hash table's
  // smallest index first, then the exact scan
  const uint32_t hq = nm_hmin(htab, C, ph);
  #pragma unroll 1
  for (uint32_t it = 0; it <= nd && parent == NONE32; ++it) {
    const uint32_t q = it == 0 ? hq : it - 1;
    if (q == NONE32 || (it > 0 && q == hq)) continue;
    if (it == 1 && hq == NONE32) break;   // no base with that hash: no parent
    const uint32_t o = m.ndl[q];
    if (m.pos[q] != (int32_t)q || m.nH[o] != ph) continue;
    if (m.nLen[o] + 1 + dec_len_u64(n) != m.nLen[slot]) continue;
    // compare the first nLen[o] characters
    bool eq = true;
    const uint32_t L = m.nLen[o];
    uint32_t ba[32], bb[32];
    #pragma unroll 1
    for (uint32_t from = 0; from < L && eq; from += 32) {
      uint32_t na = 0, nb = 0, ia = 0, ib = 0;
      for_sanitized(name_of(m, m.hname[slot]), [&](uint32_t c) { if (ia >= from && ia < L && na < 32) ba[na++] = c; ++ia; });
      for_sanitized(name_of(m, m.hname[o]), [&](uint32_t c) { if (ib >= from && nb < 32) bb[nb++] = c; ++ib; });
      #pragma unroll 1
      for (uint32_t z = 0; z < na; ++z) if (ba[z] != bb[z]) { eq = false; break; }
    }
    if (eq) parent = q;
  }
  return parent;
}

__device__ __forceinline__ void nm_mark_parent(Mod& m, uint32_t k) {
  if (m.ib[k] == NONE32) return;
  uint8_t* f = &m.hfl[m.ndl[m.ib[k]]];
  atomicOr(reinterpret_cast<unsigned int*>(reinterpret_cast<uintptr_t>(f) & ~(uintptr_t)3),
           (unsigned)HF_HASCHILD << (8 * (reinterpret_cast<uintptr_t>(f) & 3)));
}

// uniquify in D order (disasm.py:173-185), one thread: the k-th ident gets the
// first of base, base_0, base_1, ... not taken yet.  Exact reformulation: group
// idents by sanitized base; a candidate base_s can only collide with the *base*
// of another group that reads "base_<s>" (a child group, clist: (parent group,
// suffix value, child leader)), so per-group counters plus per-group "base
// taken" flags reproduce the sequential result in one O(nd) pass.
__device__ __noinline__ void nm_dedup(Mod& m, uint32_t nd, const uint32_t* clist, uint32_t nc) {
  auto child_of = [&](uint32_t g, uint32_t sv) -> uint32_t {
    #pragma unroll 1
    for (uint32_t q = 0; q < nc; ++q)
      if (clist[3 * q] == g && clist[3 * q + 1] == sv) return clist[3 * q + 2];
    return NONE32;
  };
  // the (leader, leader slot, slot) of the next 8 idents are loaded ahead: they
  // do not depend on the pass's state, only the group flags / counters do
  constexpr uint32_t AHEAD = 8;
  #pragma unroll 1
  for (uint32_t k0 = 0; k0 < nd; k0 += AHEAD) {
  uint32_t gv[AHEAD], gsv[AHEAD], ksv[AHEAD];
  #pragma unroll
  for (uint32_t j = 0; j < AHEAD; ++j) {
    const uint32_t kk = min(k0 + j, nd - 1);
    gv[j] = (uint32_t)m.pos[kk];
    ksv[j] = m.ndl[kk];
  }
  #pragma unroll
  for (uint32_t j = 0; j < AHEAD; ++j) gsv[j] = m.ndl[gv[j]];
  #pragma unroll
  for (uint32_t j = 0; j < AHEAD; ++j) {
    const uint32_t k = k0 + j;
    if (k >= nd) break;
    const uint32_t g = gv[j];
    const uint32_t gs = gsv[j];
    if (!(m.hfl[gs] & HF_HASCHILD) && m.ib[g] == NONE32) continue;   // independent group: nm_dedup_simple
    if (g == k) m.nP[gs] = 0;                       // group counter (nP no longer needed)
    uint32_t serial = NONE32;
    const uint8_t fl = m.hfl[gs];
    if (!(fl & HF_TB)) {
      m.hfl[gs] = fl | HF_TB;
    } else {
      uint32_t sv = m.nP[gs];
      if (fl & HF_HASCHILD) {
        uint32_t c;
        #pragma unroll 1
        while ((c = child_of(g, sv)) != NONE32 && (m.hfl[m.ndl[c]] & HF_TB)) ++sv;
        if (c != NONE32) m.hfl[m.ndl[c]] |= HF_TB;  // our candidate is that child's base
      }
      serial = sv;
      m.nP[gs] = sv + 1;
    }
    m.hser[ksv[j]] = serial;
  }
  }
}

// The groups that neither have child groups nor are one never meet another group's
// candidates, so nm_dedup's rule reduces to: the group's r-th ident (D order) gets
// the bare base for r = 0 and serial r - 1 after.  Warp-parallel, 32 idents at a
// time (ranks by __match_any_sync plus a running count per group in nP); nm_dedup
// then walks only the idents of the other groups, in order.
__device__ __noinline__ void nm_dedup_simple(Mod& m, uint32_t nd) {
  const uint32_t lane = lane_id();
  #pragma unroll 1
  for (uint32_t base = 0; base < nd; base += 32) {
    const uint32_t k = base + lane;
    uint32_t g = 0, gs = 0;
    bool simple = false;
    if (k < nd) {
      g = (uint32_t)m.pos[k];
      gs = m.ndl[g];
      simple = !(m.hfl[gs] & HF_HASCHILD) && m.ib[g] == NONE32;
    }
    const unsigned peers = __match_any_sync(FULL, simple ? g : (0x80000000u | lane));
    if (simple) {
      const uint32_t r = (g >= base ? 0u : m.nP[gs]) + __popc(peers & ((1u << lane) - 1));
      m.hser[m.ndl[k]] = r == 0 ? NONE32 : r - 1;
      if (r == 0) m.hfl[gs] |= HF_TB;
      if (lane == 31 - __clz(peers)) m.nP[gs] = r + 1;   // the group's count so far
    }
    __syncwarp();
  }
}

// step 5 (named definition k, kept, arena offset off): the sanitized base into the arena
__device__ __forceinline__ void nm_arena_write(Mod& m, uint32_t k, uint32_t off) {
  const uint32_t slot = m.ndl[k];
  m.hfl[slot] |= HF_FRIENDLY;
  m.hnoff[slot] = off;
  uint8_t* dst = m.narena + off;
  uint32_t q = 0;
  for_sanitized(name_of(m, m.hname[slot]), [&](uint32_t c) { dst[q++] = (uint8_t)c; });
}

// friendly names of one module by one warp (disasm.py:159-206 via SURVEY A.3)
__device__ __noinline__ void resolve_names(Mod& m, const Tables& T) {
  const uint32_t lane = lane_id();
  // 1. per slot flags; |P0|
  uint32_t nP0 = 0;
  #pragma unroll 1
  for (uint32_t s = lane; s < m.S; s += 32) nP0 += nm_slot_flags(m, s) ? 1 : 0;
  nP0 = warp_sum_u32(nP0);
  __syncwarp();
  // 2. definitions in document order: C = D without P0 (index j in ib), named list ndl
  uint32_t cj = 0, nd = 0;
  #pragma unroll 1
  for (uint32_t base = 0; base < m.I; base += 32) {
    const uint32_t i = base + lane;
    bool isC = false, isN = false;
    uint32_t slot = NONE32;
    if (i < m.I) nm_def_pred(m, T, i, isC, isN, slot);
    const unsigned bc = __ballot_sync(FULL, isC), bn = __ballot_sync(FULL, isN);
    const uint32_t below = (1u << lane) - 1;
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
  #pragma unroll 1
  for (uint32_t v = lane; v <= N; v += 32) m.pos[v] = INF;
  __syncwarp();
  #pragma unroll 1
  for (uint32_t s = lane; s < m.S; s += 32) {
    if (!(m.hfl[s] & HF_P0)) continue;
    const uint32_t key = slot_key(m, s);
    if (key >= 1 && key <= N) m.pos[key] = -1;
  }
  __syncwarp();
  #pragma unroll 1
  for (uint32_t i = lane; i < m.I; i += 32) {
    if (!(m.iflag[i] & IF_FIRSTDEF)) continue;
    const uint32_t key = nm_def_key(m, T, i);
    if (key >= 1 && key <= N) m.pos[key] = (int32_t)m.ib[i];
  }
  __syncwarp();
  int32_t carry = -2;
  #pragma unroll 1
  for (uint32_t base = 1; base <= N; base += 32) {
    const uint32_t v = base + lane;
    int32_t x = v <= N ? m.pos[v] : -2;
    x = max(warp_incl_max(x), carry);
    if (v <= N) m.pos[v] = x;
    carry = __shfl_sync(FULL, x, 31);
  }
  __syncwarp();
  #pragma unroll 1
  for (uint32_t i = lane; i < m.I; i += 32) {
    if (!(m.iflag[i] & IF_FIRSTDEF)) continue;
    const uint32_t key = nm_def_key(m, T, i);
    const int32_t j = (int32_t)m.ib[i];
    if (key >= 1 && key <= N && (key == 1 || m.pos[key - 1] < j)) m.hfl[ht_find(m, key)] |= HF_KEPT;
  }
  __syncwarp();
  // 4. uniquify: base info, leaders (hash table of base -> first ident in the
  //    spill area: capacity C = pow2 >= 2 nd, 8 C < 32 nd <= spill bytes), parents
  #pragma unroll 1
  for (uint32_t k = lane; k < nd; k += 32) nm_info(m, k);
  __syncwarp();
  uint32_t C = 4;
  while (C < 2 * nd) C <<= 1;
  uint32_t* htab = reinterpret_cast<uint32_t*>(m.spill);
  #pragma unroll 1
  for (uint32_t e = lane; e < C; e += 32) { __stcg(htab + 2 * e, EMPTY); __stcg(htab + 2 * e + 1, EMPTY); }
  __threadfence_block();
  __syncwarp();
  #pragma unroll 1
  for (uint32_t k = lane; k < nd; k += 32) nm_hinsert(htab, C, m.nH[m.ndl[k]], k);
  __threadfence_block();
  __syncwarp();
  #pragma unroll 1
  for (uint32_t k = lane; k < nd; k += 32) m.pos[k] = (int32_t)nm_leader(m, htab, C, k);
  __syncwarp();
  #pragma unroll 1
  for (uint32_t k = lane; k < nd; k += 32) m.ib[k] = nm_parent(m, htab, C, nd, k);
  __syncwarp();
  #pragma unroll 1
  for (uint32_t k = lane; k < nd; k += 32) nm_mark_parent(m, k);
  __syncwarp();
  // child entries compacted into the spill area (the table is no longer needed)
  uint32_t nc = 0;
  uint32_t* clist = reinterpret_cast<uint32_t*>(m.spill);
  #pragma unroll 1
  for (uint32_t base = 0; base < nd; base += 32) {
    const uint32_t k = base + lane;
    const bool isc = k < nd && m.ib[k] != NONE32;
    const unsigned b = __ballot_sync(FULL, isc);
    if (isc) {
      const uint32_t at = nc + __popc(b & ((1u << lane) - 1));
      clist[3 * at] = m.ib[k]; clist[3 * at + 1] = m.ia[k]; clist[3 * at + 2] = k;
    }
    nc += __popc(b);
  }
  __syncwarp();
  nm_dedup_simple(m, nd);
  if (lane == 0) nm_dedup(m, nd, clist, nc);
  __syncwarp();
  // 5. friendly = named definition that keeps its number; its sanitized base
  //    name goes into the module's name arena once (refs copy it from there)
  uint32_t acarry = 0;
  #pragma unroll 1
  for (uint32_t base = 0; base < nd; base += 32) {
    const uint32_t k = base + lane;
    const uint32_t slot = k < nd ? m.ndl[k] : 0;
    const bool kept = k < nd && (m.hfl[slot] & HF_KEPT);
    const uint32_t len = kept ? m.nLen[slot] : 0;
    const uint32_t incl = warp_incl_sum(len);
    if (kept) nm_arena_write(m, k, acarry + incl - len);
    acarry += __shfl_sync(FULL, incl, 31);
  }
  __syncwarp();
}

// ----------------------------------------------------------------------------
// section tracking for the `group` option (disasm.py:253-267)
__device__ __noinline__ void compute_sections(Mod& m, const Tables& T) {
  if (lane_id() == 0) {
    uint32_t sec = 0;
    bool in_fn = false;
    #pragma unroll 1
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

// length of put_header's text, arithmetically
__device__ __forceinline__ uint32_t header_len(const Mod& m, bool hl) {
  return 9 + (11 + dlen32(m.major) + 1 + dlen32(m.minor) + 1) +
         (13 + dlen32(m.gen >> 16) + 2 + dlen32(m.gen & 0xFFFF) + 1) + (9 + dlen32(m.bound) + 1) +
         (10 + dlen32(m.schema) + 1) + (hl ? 5 * 9 : 0);
}

template <class S>
__device__ __noinline__ void put_header(S& s, const Mod& m, bool hl) {
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

// first instruction index (in order) for which pred holds, or NONE32
template <class P>
__device__ inline uint32_t first_where(const Mod& m, P&& pred) {
  #pragma unroll 1
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane_id();
    unsigned b = __ballot_sync(FULL, i < m.I && pred(i));
    if (b) return base + __ffs(b) - 1;
  }
  return NONE32;
}

// ----------------------------------------------------------------------------
// Bulk-copy engine (sm_100a cp.async.bulk, non-tensor): shared -> global.
// SKG_BULK_FLUSH=1 flushes the write pass's text stage with one bulk copy per
// window from lane 0 (UBLKCP) instead of 16-byte stores by every lane.  Measured
// on the 200k-module batch: disasm 24.6 -> 25.4 ms, fused pipeline 27.4 -> 27.9 ms
// (the next window must wait for the copy to read the stage; two half stages,
// so the wait overlaps, cut the windows and measured 26.9 ms).  Off by default.
#ifndef SKG_BULK_FLUSH
#define SKG_BULK_FLUSH 0
#endif
__device__ __forceinline__ void bulk_fence_smem() {   // generic-proxy smem writes -> async proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
               "cp.async.bulk.commit_group;" :: "l"(gdst), "r"(s), "r"(bytes) : "memory");
}
// the issuing lane: every bulk copy it started has finished reading shared memory
__device__ __forceinline__ void bulk_read_wait() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// the issuing lane: every bulk copy it started has completed its global writes
__device__ __forceinline__ void bulk_write_wait() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Coalesced copy of staged text: shared `stage` holds bytes for global [g0, g1)
// starting at stage + (g0 & 15), so 16-byte blocks line up on both sides.
__device__ inline void flush_stage(uint8_t* g0, uint8_t* g1, const uint8_t* stage) {
  const uint32_t lane = lane_id();
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(g0), a1 = reinterpret_cast<uintptr_t>(g1);
  const uint8_t* src = stage + (a0 & 15);
  uintptr_t m0 = (a0 + 15) & ~(uintptr_t)15, m1 = a1 & ~(uintptr_t)15;
  if (m0 >= m1) {   // no full block
    #pragma unroll 1
    for (uintptr_t x = a0 + lane; x < a1; x += 32) *reinterpret_cast<uint8_t*>(x) = src[x - a0];
    return;
  }
  if (a0 + lane < m0) *reinterpret_cast<uint8_t*>(a0 + lane) = src[lane];
  if (m1 + lane < a1) *reinterpret_cast<uint8_t*>(m1 + lane) = src[m1 - a0 + lane];
#if SKG_BULK_FLUSH
  // the aligned middle leaves through the bulk-copy engine (cp.async.bulk S2G):
  // one instruction on lane 0 instead of a 16-byte store per lane and block;
  // the caller waits for its read of the stage before refilling it (bulk_read_wait)
  bulk_fence_smem();
  __syncwarp();
  if (lane == 0) bulk_s2g(reinterpret_cast<void*>(m0), src + (m0 - a0), (uint32_t)(m1 - m0));
#else
  const uint32_t nb = (uint32_t)((m1 - m0) >> 4);
  const uint4* s4 = reinterpret_cast<const uint4*>(src + (m0 - a0));
  uint4* d4 = reinterpret_cast<uint4*>(m0);
  #pragma unroll 1
  for (uint32_t k = lane; k < nb; k += 32) __stcs(d4 + k, s4[k]);   // streaming: keep L2 for scratch
#endif
}


// ============================================================================
// Word render codes (wk[w]): bits 0-3 code, bit 4 last word of its instruction,
// bit 5 blank line before (group), bits 6-31 payload.
enum : uint32_t {
  C_OPC = 0,    // opcode word: line prefix + opcode name (payload = instruction index)
  C_NONE = 1,   // no output (continuation word of a 64-bit literal)
  C_REF = 2,    // id reference (A member)
  C_DEC = 3,    // decimal of the word
  C_VEN = 4,    // value enum: payload = enumerant index
  C_BEN = 5,    // bit enum: payload = kind index
  C_STR = 6,    // 4 string bytes: payload first | last << 1 | nbytes << 2
  C_TYP = 7,    // width-typed literal: payload flt | sgn << 1 | width << 2
  C_EXT = 8,    // OpenCL.std instruction number: payload = ext_known
  C_SPO = 9,    // OpSpecConstantOp opcode
  C_UNK = 10,   // operand of an unknown opcode: !0x%08X
  C_RES = 11,   // the result id (rendered in the prefix; A member)
  C_DECID = 12  // IdResult inside a composite: decimal (A member)
};
constexpr uint32_t WK_LAST = 1u << 4, WK_BLANK = 1u << 5;
__device__ __forceinline__ uint32_t wk_code(uint32_t x) { return x & 15; }
__device__ __forceinline__ uint32_t wk_pay(uint32_t x) { return x >> 6; }

// classification visitor: one walk per instruction
struct ClassVis {
  const Mod& m;
  const Tables& T;
  uint32_t* wk;          // m.wk + first operand word
  bool have_set = false;
  uint32_t set_id = 0;
  uint32_t pending_ext = NONE32;

  __device__ void id(uint32_t role, uint32_t v, int depth, uint32_t p) {
    if (depth == 0 && role == IDR_RESULT) { wk[p] = C_RES; return; }
    if (depth == 0 && role == IDR_ID && !have_set) { have_set = true; set_id = v; }
    wk[p] = role == IDR_RESULT ? C_DECID : C_REF;
  }
  __device__ void venum(uint32_t, uint32_t, uint32_t e, uint32_t p) {
    wk[p] = e != NONE32 ? (C_VEN | (e << 6)) : C_DEC;
  }
  __device__ void benum(uint32_t k, uint32_t, bool, uint64_t, uint32_t p) { wk[p] = C_BEN | (k << 6); }
  __device__ __noinline__ void str(const uint32_t*, uint32_t pos, uint32_t nbytes) {
    const uint32_t nw = nbytes / 4 + 1;
#pragma unroll 1
    for (uint32_t j = 0; j < nw; ++j) {
      uint32_t nb = nbytes - 4 * j;
      if (nb > 4) nb = 4;
      wk[pos + j] = C_STR | (((j == 0 ? 1u : 0u) | (j == nw - 1 ? 2u : 0u) | (nb << 2)) << 6);
    }
  }
  __device__ void typed(const LitVal& lv, uint32_t p, uint32_t nw) {
    // width code: exact up to 32, 62 = any other single-word width, 63 = 64
    const uint32_t width = lv.width == 64 ? 63 : (lv.width > 32 ? 62 : lv.width);
    wk[p] = C_TYP | (((lv.flt ? 1u : 0u) | (lv.sgn ? 2u : 0u) | (width << 2)) << 6);
    if (nw == 2) wk[p + 1] = C_NONE;
  }
  __device__ void lit(uint32_t sub, uint32_t, uint32_t p) {
    if (sub == LIT_EXTINST) {
      if (!have_set) { pending_ext = p; wk[p] = C_EXT; return; }
      wk[p] = C_EXT | ((is_opencl_std(m, T, set_id) ? 1u : 0u) << 6);
      return;
    }
    wk[p] = sub == LIT_SPECOP ? C_SPO : C_DEC;
  }
  __device__ void comp_begin() {}
  __device__ void comp_end() {}
};

// walk every instruction once: word codes + per-instruction status
__device__ __forceinline__ void classify_one(Mod& m, const Tables& T, uint32_t i) {
    const uint32_t s0 = m.ioff[i];
    const uint32_t n = inst_nops(m, i);
    const uint32_t d = m.idef[i];
    uint8_t err = W_OK;
    if (d == NONE16) {
#pragma unroll 1
      for (uint32_t k = 0; k < n; ++k) m.wk[s0 + 1 + k] = C_UNK;
    } else {
      ClassVis cv{m, T, m.wk + s0 + 1};
      Resolver res{&m, &T};
      WalkErr e = walk(T, d, m.w + s0 + 1, n, cv, res);
      err = (uint8_t)e.code;
      if (cv.pending_ext != NONE32)   // the set id came after the number (custom grammars)
        m.wk[s0 + 1 + cv.pending_ext] = C_EXT | (((cv.have_set && is_opencl_std(m, T, cv.set_id)) ? 1u : 0u) << 6);
    }
    m.ierr[i] = err;
    m.wk[s0] = C_OPC | (i << 6);
    m.wk[s0 + n] |= WK_LAST;          // n == 0: the opcode word itself
}

__device__ __noinline__ void classify(Mod& m, const Tables& T) {
  for (uint32_t base = 0; base < m.I; base += 32) {
    const uint32_t i = base + lane_id();
    if (i < m.I) classify_one(m, T, i);
  }
  __syncwarp();
}

// referenced ids (A, disasm.py:221-240), word-parallel
__device__ __forceinline__ void collect_one(Mod& m, uint32_t w) {
  const uint32_t c = wk_code(m.wk[w]);
  if (c == C_REF || c == C_RES || c == C_DECID) {
    uint32_t s = ht_insert(m, m.w[w]);
    if (s != NONE32) m.hA[s] = 1;
  }
}

__device__ __noinline__ void collect_ids(Mod& m) {
  for (uint32_t w = 5 + lane_id(); w < m.W; w += 32) collect_one(m, w);
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Per-word length (arithmetic only) and emission (register-resident pointer).
__device__ __forceinline__ uint8_t* emit_u32(uint8_t* __restrict__ p, uint32_t v) {
  uint8_t* e = p + dlen32(v);
  uint8_t* q = e;
#pragma unroll 1
  do { *--q = (uint8_t)('0' + v % 10); v /= 10; } while (v);
  return e;
}
__device__ __forceinline__ uint8_t* emit_cstr(uint8_t* __restrict__ p, const char* z) {
#pragma unroll 1
  while (*z) *p++ = (uint8_t)*z++;
  return p;
}
__device__ __forceinline__ uint8_t* emit_tab(uint8_t* __restrict__ p, const Tables& T, uint32_t off, uint32_t len) {
  const uint8_t* src = T.str + off;
  uint32_t q = 0;
#pragma unroll 1
  for (; q + 4 <= len; q += 4) {
    const uint8_t c0 = __ldg(src + q), c1 = __ldg(src + q + 1), c2 = __ldg(src + q + 2), c3 = __ldg(src + q + 3);
    p[q] = c0; p[q + 1] = c1; p[q + 2] = c2; p[q + 3] = c3;
  }
#pragma unroll 1
  for (; q < len; ++q) p[q] = __ldg(src + q);
  return p + len;
}

__device__ __noinline__ uint8_t* emit_ref(uint8_t* __restrict__ p, const Mod& m, uint32_t id) {
  if (m.n_ovr) {
    const uint32_t k = ovr_find(m, id);
    if (k != NONE32) {
      const uint8_t* src = m.ovr_text + m.ovr[3 * k + 1];
      const uint32_t n = m.ovr[3 * k + 2];
      for (uint32_t q = 0; q < n; ++q) p[q] = src[q];
      return p + n;
    }
  }
  *p++ = '%';
  // direct mode: a slot that is not present has hfl == 0 (init_tables)
  const uint32_t slot = m.direct ? (id < m.S ? id : NONE32) : ht_find(m, id);
  if (slot != NONE32 && (m.hfl[slot] & HF_FRIENDLY)) {
    const uint8_t* src = m.narena + m.hnoff[slot];
    const uint32_t n = m.nLen[slot];
    uint32_t q = 0;
#pragma unroll 1
    for (; q + 4 <= n; q += 4) {
      const uint8_t c0 = src[q], c1 = src[q + 1], c2 = src[q + 2], c3 = src[q + 3];
      p[q] = c0; p[q + 1] = c1; p[q + 2] = c2; p[q + 3] = c3;
    }
#pragma unroll 1
    for (; q < n; ++q) p[q] = src[q];
    p += n;
    const uint32_t ser = m.hser[slot];
    if (ser != NONE32) { *p++ = '_'; p = emit_u32(p, ser); }
    return p;
  }
  return emit_u32(p, id);
}

// components of a BitEnum mask in file order (ops.py:77-89): total name bytes,
// count, and whether they cover the mask
__device__ __forceinline__ bool bit_cover(const Tables& T, uint32_t k, uint32_t v, uint32_t& bytes,
                                          uint32_t& count) {
  const uint32_t eo = T.kenum_off(k), ne = T.knenum(k);
  uint32_t covered = 0;
  bytes = 0; count = 0;
#pragma unroll 1
  for (uint32_t j = 0; j < ne; ++j) {
    const uint32_t ev = T.evalue(eo + j);
    if (ev && (v & ev) == ev && (covered & ev) != ev) {
      covered |= ev; bytes += T.ename_len(eo + j); ++count;
      if (covered == v) break;   // later enumerants can only be skipped
    }
  }
  return covered == v;
}

__device__ __forceinline__ uint32_t hex_digits(uint32_t v) {
  uint32_t hd = 1;
#pragma unroll 1
  for (uint32_t x = v >> 4; x; x >>= 4) ++hd;
  return hd;
}

__device__ __forceinline__ uint64_t typed_float_bits(const Mod& m, uint32_t w, uint32_t v, uint32_t width_t) {
  if (width_t == 63) return (uint64_t)v | ((uint64_t)m.w[w + 1] << 32);
  if (width_t == 32) return f32_to_f64_bits(v);
  return f16_to_f64_bits(v & 0xFFFF);
}

__device__ __forceinline__ LitVal typed_int(const Mod& m, uint32_t w, uint32_t v, uint32_t width_t, bool sgn) {
  LitVal lv;
  WalkErr e;
  uint32_t raw[2] = {v, width_t == 63 ? m.w[w + 1] : 0};
  decode_typed(raw, width_t == 63 ? 64 : (width_t == 62 ? 33 : width_t), sgn, false, lv, e);
  return lv;
}

// byte length of word w's text (disasm.py:284-377)
__device__ __noinline__ uint32_t word_len(const Mod& m, const Tables& T, uint32_t w, uint32_t x,
                                          uint32_t width, bool hl) {
  const uint32_t v = m.w[w];
  const uint32_t color = hl ? 9 : 0;
  uint32_t n = (x & WK_LAST) ? 1 : 0;
  switch (wk_code(x)) {
    case C_OPC: {
      const uint32_t i = wk_pay(x);
      if (x & WK_BLANK) n += 1;
      if (m.iflag[i] & IF_HAS_RESULT) {
        const uint32_t rl = m.irl[i] == 0xFFFF ? ref_len(m, m.ib[i]) : m.irl[i];
        n += (width ? width : rl) + color + 3;
      } else if (width) {
        n += width + 3;
      }
      const uint32_t d = m.idef[i];
      n += color + (d == NONE16 ? 11 + dlen32(v & 0xFFFF) : T.iname_len(d));
      return n;
    }
    case C_NONE: case C_RES: return n;
    case C_REF: return n + 1 + ref_len(m, v) + color;
    case C_DEC: case C_DECID: return n + 1 + dlen32(v);
    case C_VEN: return n + 1 + T.ename_len(wk_pay(x));
    case C_BEN: {
      const uint32_t k = wk_pay(x);
      if (v == 0) { const uint32_t z = T.kzero(k); return n + 1 + (z != NONE32 ? T.ename_len(z) : 1); }
      uint32_t bytes, cnt;
      if (!bit_cover(T, k, v, bytes, cnt)) return n + 3 + hex_digits(v);
      return n + 1 + bytes + cnt - 1;
    }
    case C_STR: {
      const uint32_t pl = wk_pay(x), nb = pl >> 2;
      n += nb;
#pragma unroll 1
      for (uint32_t q = 0; q < nb; ++q) { const uint32_t b = (v >> (8 * q)) & 0xFF; n += (b == '\\' || b == '"'); }
      if (pl & 1) n += 2 + (hl ? 5 : 0);
      if (pl & 2) n += 1 + (hl ? 4 : 0);
      return n;
    }
    case C_TYP: {
      const uint32_t pl = wk_pay(x), width_t = pl >> 2;
      if (pl & 1) {   // the repr's digits (Ryu) once: kept for the write pass
        const FloatParts fp = repr_parts(typed_float_bits(m, w, v, width_t));
        if (m.fpc) m.fpc[w] = make_uint4((uint32_t)fp.digits, (uint32_t)(fp.digits >> 32), (uint32_t)fp.exp,
                                         fp.kind | (fp.neg ? 0x100u : 0u));
        return n + 1 + repr_len(fp);
      }
      const LitVal lv = typed_int(m, w, v, width_t, pl & 2);
      return n + 1 + (lv.neg ? 1 + dec_len_u64((uint64_t)0 - lv.bits) : dec_len_u64(lv.bits));
    }
    case C_EXT: {
      uint32_t off, ln;
      if (wk_pay(x) && T.ext_name(v, off, ln)) return n + 1 + ln;
      return n + 1 + dlen32(v);
    }
    case C_SPO: {
      const uint32_t d = T.inst_of(v);
      return n + 1 + (d != NONE32 ? T.iname_len(d) - 2 : dlen32(v));
    }
    case C_UNK: return n + 12;
    default: return n;
  }
}

// emit word w's text at p; `spaces` = destination already holds spaces (skip padding).
// Every code's text is prefix + [ref] + [" = "] + [table name] + [digits] +
// [special] + ['\n'], so the stages run in that order with the expensive ones
// (reference, table-name copy, decimal digits) reached by all lanes that need
// them at the same program point: the warp runs each once, not once per code.
__device__ __noinline__ void word_emit(uint8_t* __restrict__ p, const Mod& m, const Tables& T, uint32_t w, uint32_t x,
                                       uint32_t width, bool hl, bool spaces) {
  const uint32_t v = m.w[w];
  const uint32_t code = wk_code(x);
  uint32_t ref = NONE32, tab_off = 0, tab_len = 0, num = 0;
  bool has_ref = false, has_num = false, opc_res = false, special = false;
  const char* ansi_tab = nullptr;
  // stage 1: prefix and what the later stages emit
  if (code == C_OPC) {
    const uint32_t i = wk_pay(x);
    if (x & WK_BLANK) *p++ = '\n';
    opc_res = m.iflag[i] & IF_HAS_RESULT;
    uint32_t pad;
    if (opc_res) {
      const uint32_t rl = m.irl[i] == 0xFFFF ? ref_len(m, m.ib[i]) : m.irl[i];
      pad = width ? width - rl : 0;
      has_ref = true;
      ref = m.ib[i];
    } else {
      pad = width ? width + 3 : 0;
    }
    if (!spaces) {
#pragma unroll 1
      for (uint32_t q = 0; q < pad; ++q) p[q] = ' ';
    }
    p += pad;
    const uint32_t d = m.idef[i];
    if (d == NONE16) { special = true; num = v & 0xFFFF; }
    else { tab_off = T.iname_off(d); tab_len = T.iname_len(d); ansi_tab = hl ? ANSI_OPCODE : nullptr; }
  } else if (code == C_REF) {
    *p++ = ' ';
    has_ref = true;
    ref = v;
  } else if (code == C_DEC || code == C_DECID) {
    *p++ = ' ';
    has_num = true;
    num = v;
  } else if (code == C_VEN) {
    *p++ = ' ';
    const uint32_t e = wk_pay(x);
    tab_off = T.ename_off(e); tab_len = T.ename_len(e);
  } else if (code == C_EXT) {
    *p++ = ' ';
    if (!(wk_pay(x) && T.ext_name(v, tab_off, tab_len))) { has_num = true; num = v; tab_len = 0; }
  } else if (code == C_SPO) {
    *p++ = ' ';
    const uint32_t d = T.inst_of(v);
    if (d != NONE32) { tab_off = T.iname_off(d) + 2; tab_len = T.iname_len(d) - 2; }
    else { has_num = true; num = v; }
  } else if (code != C_NONE && code != C_RES) {
    special = true;
  }
  // stage 2: the reference (result of an instruction line, or an id operand)
  if (has_ref) {
    if (hl) p = emit_cstr(p, ANSI_ID);
    p = emit_ref(p, m, ref);
    if (hl) p = emit_cstr(p, ANSI_RESET);
    if (opc_res) { p[0] = ' '; p[1] = '='; p[2] = ' '; p += 3; }
  }
  // stage 3: a name from the grammar tables (opcode, enumerant, ext instruction)
  if (tab_len) {
    if (ansi_tab) p = emit_cstr(p, ansi_tab);
    p = emit_tab(p, T, tab_off, tab_len);
    if (ansi_tab) p = emit_cstr(p, ANSI_RESET);
  }
  // stage 4: decimal digits
  if (has_num) p = emit_u32(p, num);
  // stage 5: the rest (bit masks, strings, typed literals, unknown opcodes / words)
  if (special) {
    switch (code) {
      case C_OPC: {   // opcode outside the grammar
        if (hl) p = emit_cstr(p, ANSI_OPCODE);
        p = emit_cstr(p, "OpUnknown("); p = emit_u32(p, num); *p++ = ')';
        if (hl) p = emit_cstr(p, ANSI_RESET);
        break;
      }
      case C_BEN: {
        const uint32_t k = wk_pay(x);
        *p++ = ' ';
        if (v == 0) {
          const uint32_t z = T.kzero(k);
          if (z != NONE32) p = emit_tab(p, T, T.ename_off(z), T.ename_len(z)); else *p++ = '0';
          break;
        }
        uint32_t bytes, cnt;
        if (!bit_cover(T, k, v, bytes, cnt)) {
          const uint32_t hd = hex_digits(v);
          *p++ = '0'; *p++ = 'x';
#pragma unroll 1
          for (uint32_t q = 0; q < hd; ++q) p[q] = (uint8_t)"0123456789abcdef"[(v >> (4 * (hd - 1 - q))) & 0xF];
          p += hd;
          break;
        }
        const uint32_t eo = T.kenum_off(k), ne = T.knenum(k);
        uint32_t covered = 0;
        bool first = true;
#pragma unroll 1
        for (uint32_t j = 0; j < ne; ++j) {
          const uint32_t ev = T.evalue(eo + j);
          if (covered == v) break;
          if (ev && (v & ev) == ev && (covered & ev) != ev) {
            covered |= ev;
            if (!first) *p++ = '|';
            first = false;
            p = emit_tab(p, T, T.ename_off(eo + j), T.ename_len(eo + j));
          }
        }
        break;
      }
      case C_STR: {
        const uint32_t pl = wk_pay(x), nb = pl >> 2;
        if (pl & 1) { *p++ = ' '; if (hl) p = emit_cstr(p, ANSI_STRING); *p++ = '"'; }
#pragma unroll 1
        for (uint32_t q = 0; q < nb; ++q) {
          const uint32_t b = (v >> (8 * q)) & 0xFF;
          if (b == '\\' || b == '"') *p++ = '\\';
          *p++ = (uint8_t)b;
        }
        if (pl & 2) { *p++ = '"'; if (hl) p = emit_cstr(p, ANSI_RESET); }
        break;
      }
      case C_TYP: {
        const uint32_t pl = wk_pay(x), width_t = pl >> 2;
        Sink sk(p);
        sk.put(' ');
        if (pl & 1) {
          FloatParts fp;
          if (m.fpc) {   // parts computed by the size pass (word_len)
            const uint4 c = m.fpc[w];
            fp.digits = c.x | ((uint64_t)c.y << 32); fp.exp = (int32_t)c.z;
            fp.kind = (uint8_t)(c.w & 0xFF); fp.neg = (c.w >> 8) & 1;
          } else {
            fp = repr_parts(typed_float_bits(m, w, v, width_t));
          }
          put_repr_parts(sk, fp);
        }
        else {
          const LitVal lv = typed_int(m, w, v, width_t, pl & 2);
          if (lv.neg) put_i64(sk, (int64_t)lv.bits); else put_u64(sk, lv.bits);
        }
        p += sk.n;
        break;
      }
      case C_UNK: {
        *p++ = ' '; *p++ = '!'; *p++ = '0'; *p++ = 'x';
#pragma unroll 1
        for (uint32_t q = 0; q < 8; ++q) p[q] = (uint8_t)"0123456789ABCDEF"[(v >> (28 - 4 * q)) & 0xF];
        p += 8;
        break;
      }
      default: break;
    }
  }
  if (x & WK_LAST) *p = '\n';
}

// result ref of every instruction -> irl/ib/iflag, module width (disasm.py:286-288)
__device__ __forceinline__ uint32_t result_ref_one(Mod& m, const Tables& T, uint32_t i) {
    uint32_t width = 0;
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
    return width;
}

__device__ __noinline__ uint32_t result_refs(Mod& m, const Tables& T) {
  fill_ref_lengths(m);
  uint32_t width = 0;
  for (uint32_t base = 0; base < m.I; base += 32) {
    const uint32_t i = base + lane_id();
    if (i < m.I) width = max(width, result_ref_one(m, T, i));
  }
  return warp_max_u32(width);
}

// blank-line marks for the group option (disasm.py:303-305)
__device__ __noinline__ void mark_blanks(Mod& m) {
  for (uint32_t base = 1; base < m.I; base += 32) {
    uint32_t i = base + lane_id();
    if (i < m.I && m.isec[i] != m.isec[i - 1]) m.wk[m.ioff[i]] |= WK_BLANK;
  }
  __syncwarp();
}

__device__ __noinline__ uint64_t text_size(const Mod& m, const Tables& T, uint32_t opts, uint32_t width) {
  const bool hl = opts & OPT_HIGHLIGHT;
  uint32_t sum = 0;
  for (uint32_t w = 5 + lane_id(); w < m.W; w += 32) {
    const uint32_t l = word_len(m, T, w, m.wk[w], width, hl);
    m.wl[w] = (uint16_t)(l > 0xFFFF ? 0xFFFF : l);   // 0xFFFF: recompute (huge names only)
    sum += l;
  }
  uint64_t total = warp_sum_u32(sum);
  if (!(opts & OPT_NO_HEADER)) total += header_len(m, hl);
  return total;
}

// Write the module text at `out` (16-byte aligned) through the warp's shared
// stage.  Each window takes the longest run of the next 32 words whose text
// fits the stage: the stage is pre-filled with spaces (indentation costs
// nothing), every lane emits its word at its scanned offset (lengths from the
// size pass), and the window is flushed with 16-byte stores.  A word too long
// for the stage on its own is written straight to global memory.
__device__ __noinline__ void text_write_range(const Mod& m, const Tables& T, uint32_t opts, uint32_t width,
                                              uint8_t* out, uint8_t* stage, uint32_t cap, uint32_t w_begin,
                                              uint32_t w_end, uint64_t pos0, bool header);

__device__ __noinline__ void text_write(const Mod& m, const Tables& T, uint32_t opts, uint32_t width,
                                        uint8_t* out, uint8_t* stage, uint32_t cap) {
  text_write_range(m, T, opts, width, out, stage, cap, 5, m.W, 0, !(opts & OPT_NO_HEADER));
}

// words [w_begin, w_end) whose text starts at out + pos0 (after the header when
// `header`: then pos0 must be 0)
__device__ __noinline__ void text_write_range(const Mod& m, const Tables& T, uint32_t opts, uint32_t width,
                                              uint8_t* out, uint8_t* stage, uint32_t cap, uint32_t w_begin,
                                              uint32_t w_end, uint64_t pos0, bool header) {
  const uint32_t lane = lane_id();
  const bool hl = opts & OPT_HIGHLIGHT;
  uint64_t pos = pos0;
  const uint4 sp4 = make_uint4(0x20202020u, 0x20202020u, 0x20202020u, 0x20202020u);
  if (header) {
    if (lane == 0) { Sink ms(stage); put_header(ms, m, hl); pos = ms.n; }
    pos = __shfl_sync(FULL, pos, 0);
    __syncwarp();
    flush_stage(out, out + pos, stage);
    __syncwarp();
  }
  uint32_t w0 = w_begin;
  const uint32_t* __restrict__ wk = m.wk;   // held in registers across the stage stores
  const uint16_t* __restrict__ wl = m.wl;
  // each window's codes and lengths are loaded while the previous window is rendered
  uint32_t x_next = 0, l_next = 0;
  if (w0 + lane < w_end) { x_next = wk[w0 + lane]; l_next = wl[w0 + lane]; }
  while (w0 < w_end) {
    const uint32_t w = w0 + lane;
    const uint32_t x = x_next;
    uint32_t len = l_next;
    if (w < w_end && len == 0xFFFF) len = word_len(m, T, w, x, width, hl);
    const uint32_t incl = warp_incl_sum(len);
    const uint32_t shift = (uint32_t)(reinterpret_cast<uintptr_t>(out + pos) & 15);
    const uint32_t take = __popc(__ballot_sync(FULL, w < w_end && shift + incl <= cap));
    {
      const uint32_t wn = w0 + (take ? take : 1) + lane;
      x_next = 0; l_next = 0;
      if (wn < w_end) { x_next = wk[wn]; l_next = wl[wn]; }
    }
    if (take == 0) {   // one word longer than the stage
      if (lane == 0) word_emit(out + pos, m, T, w, x, width, hl, false);
      __syncwarp();
      pos += __shfl_sync(FULL, len, 0);
      w0 += 1;
      continue;
    }
    const uint32_t chunk = __shfl_sync(FULL, incl, take - 1);
    const uint32_t n16 = (shift + chunk + 15) >> 4;
#if SKG_BULK_FLUSH
    if (lane == 0) bulk_read_wait();   // the previous window's bulk copy has left the stage
    __syncwarp();
#endif
    for (uint32_t k = lane; k < n16; k += 32) reinterpret_cast<uint4*>(stage)[k] = sp4;
    __syncwarp();
    if (lane < take && len) word_emit(stage + shift + incl - len, m, T, w, x, width, hl, true);
    __syncwarp();
    flush_stage(out + pos, out + pos + chunk, stage);
    __syncwarp();
    pos += chunk;
    w0 += take;
  }
#if SKG_BULK_FLUSH
  if (lane == 0) bulk_write_wait();   // text complete in global memory, stage free for the caller
  __syncwarp();
#endif
}

__device__ __noinline__ void report_inst_error(const Mod& m, const Tables& T, uint32_t i, ErrRec* rec,
                                               int32_t module, int32_t& cls) {
  const uint32_t d = m.idef[i];
  NullVis nv;
  Resolver res{&m, &T};
  WalkErr e = walk(T, d, inst_ops(m, i), inst_nops(m, i), nv, res);
  cls = walk_status(e.code);
  if (rec) {
    ErrWriter ew{rec};
    put_walk_error(ew, T, d, e);
    rec->module = module; rec->cls = cls; rec->len = ew.n;
    rec->a = e.a; rec->b = e.b; rec->c = e.c; rec->d = e.d;
  }
}

__device__ __noinline__ void report_prescan_error(const Mod& m, const Tables& T, uint32_t i, ErrRec* rec,
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

__device__ __noinline__ void report_internal(ErrSink& es, int32_t t, const char* what) {
  if (lane_id() == 0) {
    ErrRec* erec = es.alloc();
    if (erec) {
      ErrWriter ew{erec};
      put_cstr(ew, what);
      erec->module = t; erec->cls = ST_INTERNAL; erec->len = ew.n;
    }
  }
}

// ============================================================================
// Optional per-phase cycle counters (build with -DSKG_PHASE_TIMING; profiling only)
#ifdef SKG_PHASE_TIMING
__device__ unsigned long long g_dis_phase[16];
#define DPHASE_MARK(k)                                                  \
  do {                                                                  \
    __syncwarp();                                                       \
    const long long now_ = clock64();                                   \
    if (lane_id() == 0) atomicAdd(&g_dis_phase[k], (unsigned long long)(now_ - ph_t0_)); \
    ph_t0_ = now_;                                                      \
  } while (0)
#define DPHASE_START() long long ph_t0_ = clock64()
#else
#define DPHASE_MARK(k) do {} while (0)
#define DPHASE_START() do {} while (0)
#endif

// One module per warp; all warps of the CTA run the same phase at the same
// time (CTA barrier between phases), so the instruction working set of the SM
// is one phase rather than the whole program.
// VAL (pipeline_kernel): the same pass also validates the module (validate_one's V2/V3
// on the tables, prescan and decode this pass already built), writing the validator's
// outputs next to the text: one read and one decode of every module for both results.
template <bool VAL>
__device__ __noinline__ void disasm_one(const DisasmArgs& a, uint32_t ticket, uint8_t* slab, uint8_t* gslot,
                                        uint8_t* stage, ErrSink& es, uint32_t gid, uint32_t gw, Mod& m,
                                        uint64_t* veff, Mod* all, CtaSort* cs, const uint64_t (*effs)[MAX_CAPW]) {
  const uint32_t lane = lane_id();
  const Tables& T = a.T;
  DPHASE_START();
  const bool live = ticket < a.n_mod;
  const uint32_t t = live ? a.order[ticket] : 0;
  int32_t status = live ? ST_OK : ST_INTERNAL;
  uint64_t total = 0;
  uint32_t width = 0;
  bool in_smem = false, direct = false, names_mode = false;
  int32_t vstatus = status, decode_status = ST_OK;   // VAL: the validator's status / decode error
  uint64_t vtotal = 0;
  uint32_t vfast = 0;
  Shape sh{};
  int64_t nbytes = 0;
  // -- P0: load + boundary (A1, A2)
  if (live) {
    nbytes = a.mod_len[t];
    const uint8_t* src = a.data + a.mod_off[t];
    const uint32_t W = (nbytes >= 0 && nbytes % 4 == 0) ? (uint32_t)(nbytes / 4) : 0;
    in_smem = head_bytes(W) <= a.smem_slab;
    if (!in_smem && worst_bytes(W, RENDER_MIN) > a.gslot_bytes) {
      status = ST_INTERNAL;
      report_internal(es, (int32_t)t, "internal: module exceeds the per-warp scratch slot");
    } else {
      layout_head(m, in_smem ? slab : gslot, W);
      m.ovr = a.ovr; m.ovr_text = a.ovr_text; m.n_ovr = a.n_ovr;
      status = load_and_split(m, src, (uint64_t)nbytes, &es, (int32_t)t);
      if (VAL) {
        if (status == ST_TRUNCATED || status == ST_NOTSPIRV || status == ST_CORRUPT) decode_status = status;
        else vstatus = status;
      }
    }
  } else if (VAL) {
    vstatus = ST_INTERNAL;
  }
  DPHASE_MARK(0);
  group_sync(gid, gw);
  // -- P1: id tables + prescan (A15)
  bool any_name = false;
  if (status == ST_OK) {
    direct = m.bound <= 2 * m.W + 64;
    if (!place_tables(m, direct, in_smem, gslot, a.gslot_bytes, a.smem_slab, RENDER_MIN)) {
      status = ST_INTERNAL;
      if (VAL) vstatus = ST_INTERNAL;
      report_internal(es, (int32_t)t, "internal: module exceeds the per-warp scratch slot");
    } else {
      init_tables(m);
      any_name = prescan(m, T);
    }
  }
  DPHASE_MARK(1);
  group_sync(gid, gw);
  // -- P2: classify (A8-A12) + referenced ids; an id at/above the bound redoes
  //    P1+P2 with the hash table (rare: non-canonical modules)
  // (classification across the CTA's modules, classify_cta, measured -4% on a 200k-module
  //  batch of 2000 variants but +2% on the bench's 1M modules of 10000 variants: per module)
  if (status == ST_OK) classify(m, T);
  if (status == ST_OK) {
    names_mode = (a.opts & OPT_INLINE) && any_name;
    if (names_mode) collect_ids(m);
    if (*m.overflow && direct) {
      __syncwarp();
      direct = false;
      if (!place_tables(m, direct, in_smem, gslot, a.gslot_bytes, a.smem_slab, RENDER_MIN)) {
        status = ST_INTERNAL;
        if (VAL) vstatus = ST_INTERNAL;
        report_internal(es, (int32_t)t, "internal: module exceeds the per-warp scratch slot");
      } else {
        init_tables(m);
        any_name = prescan(m, T);
        names_mode = (a.opts & OPT_INLINE) && any_name;
        classify(m, T);
        if (names_mode) collect_ids(m);
      }
    }
  }
  DPHASE_MARK(2);
  group_sync(gid, gw);
  // -- P3: exceptions, in the reference's evaluation order
  if (status == ST_OK) {
    uint32_t bad = first_where(m, [&](uint32_t i) { return (m.iflag[i] & IF_PRESCAN_UTF8) != 0; });
    if (bad != NONE32) {
      status = ST_UNICODE;
      if (lane == 0) report_prescan_error(m, T, bad, es.alloc(), (int32_t)t);
    }
    if (status == ST_OK && names_mode) {
      bad = first_where(m, [&](uint32_t i) {
        uint32_t e = m.ierr[i]; return m.idef[i] != NONE16 && e != W_OK && !werr_is_codec(e); });
      if (bad != NONE32) {
        if (lane == 0) report_inst_error(m, T, bad, es.alloc(), (int32_t)t, status);
        status = __shfl_sync(FULL, status, 0);
      }
    }
    if (status == ST_OK) {
      bad = first_where(m, [&](uint32_t i) {
        return (m.idef[i] == NONE16 && (a.opts & OPT_STRICT)) || (m.idef[i] != NONE16 && m.ierr[i] != W_OK);
      });
      if (bad != NONE32) {
        if (lane == 0) {
          ErrRec* erec = es.alloc();
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
      }
    }
  }
  DPHASE_MARK(3);
  group_sync(gid, gw);
  // -- P4: friendly names (A16)
  if (status == ST_OK && names_mode) resolve_names(m, T);
  DPHASE_MARK(4);
  group_sync(gid, gw);
  // -- P5 (VAL): the validator's shape, capabilities, diagnostic sizes and offsets
  //    (validate_one V2); m.ia is free once the friendly names are resolved
  // The per-instruction walks of validate V2 / V3 run across the CTA's modules when the
  // barrier group is the whole CTA (val_walk_cta, as in validate_kernel): fused pass
  // on the bench's 1M-module batch 166 -> 149 ms (on a 200k batch of 2000 variants it
  // measured 2.5% slower: fewer distinct instructions per CTA).
  __shared__ uint32_t s_vfast[32];
  __shared__ uint8_t* s_vout[32];
  const bool vcross = gw == (blockDim.x >> 5);
  if (VAL) {
    const bool vmine = live && vstatus == ST_OK && decode_status == ST_OK;
    uint64_t eff[MAX_CAPW];
    for (int k = 0; k < MAX_CAPW; ++k) eff[k] = 0;
    ErrSink ves{a.verrs, a.vctr + 1, a.verr_cap};
    if (vmine) {
      // the classification walk's status is the validator's first walk; BoundTooSmall
      // needs an id operand at/above the bound (word-parallel check of the id words)
      bool big = false;
      if (status != ST_INTERNAL) {
        for (uint32_t w = 5 + lane; w < m.W; w += 32) {
          const uint32_t c = wk_code(m.wk[w]);
          big |= (c == C_REF || c == C_RES || c == C_DECID) && m.w[w] >= m.bound;
        }
      }
      big = __any_sync(FULL, big);
      vfast = VF_IERR_KNOWN | (big ? 0u : VF_NO_BIG_IDS);
    }
    if (vcross) {
      if (vmine) val_shape(m, T, eff, sh);
      if (lane == 0) {
        for (int k = 0; k < MAX_CAPW; ++k) veff[k] = eff[k];
        s_vfast[threadIdx.x >> 5] = vfast;
      }
      val_walk_cta(all, T, *cs, effs, s_vfast, nullptr, vmine, false);
      if (vmine) vtotal = val_finish(m, T, eff, sh, vstatus, ves, (int32_t)t);
    } else if (vmine) {
      vtotal = val_sizes(m, T, eff, sh, vstatus, ves, (int32_t)t, vfast);
      if (lane == 0) for (int k = 0; k < MAX_CAPW; ++k) veff[k] = eff[k];
    }
    __syncwarp();
  }
  if (VAL) group_sync(gid, gw);   // a phase of its own: the SM runs one phase's code at a time
  // -- P5: result refs, width, sections, text size (A17-A19)
  if (status == ST_OK) {
    width = result_refs(m, T);
    if (a.opts & OPT_NO_INDENT) width = 0;
    if (a.opts & OPT_GROUP) { compute_sections(m, T); mark_blanks(m); }
    total = text_size(m, T, a.opts, width);
  }
  DPHASE_MARK(5);
  group_sync(gid, gw);
  // -- P6: reserve the module's bytes (16-byte aligned starts) and write the text
  if (live) {
    if (status != ST_OK) total = 0;
    bool fits;
    uint64_t off = alloc_text(a.ticket, (total + 15) & ~15ull, a.text_cap, fits);
    if (lane == 0) {
      a.text_span[2 * t] = (int64_t)off;
      a.text_span[2 * t + 1] = (int64_t)total;
      a.status[t] = status;
    }
    if (status == ST_OK && total > 0 && fits) text_write(m, T, a.opts, width, a.text + off, stage, a.stage_bytes);
  }
  if (VAL) group_sync(gid, gw);
  bool vwrite = false;
  uint8_t* vout = nullptr;
  if (VAL && live) {
    {   // validate_one V3: the diagnostics, or the decode error as the only one
      uint64_t vt = vstatus == ST_OK ? vtotal : 0;
      ErrRec tmp;
      const char* code = nullptr;
      if (vstatus == ST_OK && decode_status != ST_OK) {
        code = decode_code(decode_status);
        CountSink cs;
        diag_head(cs, true, code, NONE32);
        ErrWriter ew{&tmp};
        put_decode_msg(ew, m, nbytes, decode_status);
        tmp.len = ew.n;
        vt = cs.n + (uint32_t)tmp.len + 1;
      }
      bool vfits;
      const uint64_t voff = alloc_text(a.vctr, vt, a.vtext_cap, vfits);
      if (lane == 0) {
        a.vspan[2 * t] = (int64_t)voff;
        a.vspan[2 * t + 1] = (int64_t)vt;
        a.vstatus[t] = vstatus;
      }
      if (vstatus == ST_OK && vfits && vt > 0) {
        if (code) {
          if (lane == 0) {
            MemSink ms(a.vtext + voff);
            diag_head(ms, true, code, NONE32);
            ms.putn((const uint8_t*)tmp.msg, (uint32_t)tmp.len);
            ms.put('\n');
          }
        } else {
          vwrite = true;
          vout = a.vtext + voff;
        }
      }
    }
  }
  if (VAL && vcross) {
    if (vwrite && lane == 0) { MemSink ms(vout); shape_diags(ms, sh); }
    if (lane == 0) s_vout[threadIdx.x >> 5] = vout;
    val_walk_cta(all, T, *cs, effs, s_vfast, s_vout, vwrite, true);
  } else if (VAL && vwrite) {
    val_write(vout, m, T, veff, sh, vfast);
  }
  DPHASE_MARK(6);
  group_sync(gid, gw);
}

#ifndef SKG_DIS_MAXT
#define SKG_DIS_MAXT 1024
#define SKG_DIS_MINB 1
#endif
template <bool VAL>
__device__ __forceinline__ void disasm_persistent(const DisasmArgs& a);

__global__ void __launch_bounds__(SKG_DIS_MAXT, SKG_DIS_MINB) disasm_kernel(const __grid_constant__ DisasmArgs a) {
  disasm_persistent<false>(a);
}

// decode -> validate -> disassemble in one pass (skg_disasm_validate)
__global__ void __launch_bounds__(SKG_DIS_MAXT, SKG_DIS_MINB) pipeline_kernel(const __grid_constant__ DisasmArgs a) {
  disasm_persistent<true>(a);
}

template <bool VAL>
__device__ __forceinline__ void disasm_persistent(const DisasmArgs& a) {
  __shared__ DisasmArgs s_args;   // one copy per CTA: field reads are shared loads
  if (threadIdx.x == 0) s_args = a;
  __syncthreads();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_base[16];
  // the module descriptor, one per warp in shared memory (a per-thread copy would
  // take 32 x sizeof(Mod) of L1 per warp as local memory); all lanes write the
  // same values into it
  __shared__ Mod s_mod[32];
  __shared__ CtaSort s_cs;   // cross-module work assignment (classification)
  __shared__ uint64_t s_eff[VAL ? 32 : 1][MAX_CAPW];   // VAL: effective capabilities per warp
  const uint32_t warps = blockDim.x >> 5;
  const uint32_t warp_in_block = threadIdx.x >> 5;
  const uint32_t gw = a.group_warps;                 // warps per barrier group
  const uint32_t gid = warp_in_block / gw, gwarp_in = warp_in_block % gw;
  const uint32_t gwarp = blockIdx.x * warps + warp_in_block;
  uint8_t* stage = smem + (size_t)warp_in_block * a.stage_bytes;
  uint8_t* slab = smem + (size_t)warps * a.stage_bytes + (size_t)warp_in_block * a.smem_slab;
  uint8_t* gslot = a.gscratch + (size_t)gwarp * a.gslot_bytes;
  ErrSink es{a.errs, a.ticket + 1, a.err_cap};
  while (true) {
    if (gwarp_in == 0 && lane_id() == 0) s_base[gid] = atomicAdd(a.ticket, gw);
    group_sync(gid, gw);
    const uint32_t base = s_base[gid];
    group_sync(gid, gw);
    if (base >= a.n_mod) break;
    disasm_one<VAL>(s_args, base + gwarp_in, slab, gslot, stage, es, gid, gw, s_mod[warp_in_block],
                    VAL ? s_eff[warp_in_block] : nullptr, s_mod, &s_cs, s_eff);
  }
}



// ---------------------------------------------------------------------------
// One large module over the whole GPU (skg_big.cuh): the phases of disasm_one as
// grid-stride kernels over instructions / words / ids / named definitions,
// device-wide scans where the warp version carries a running offset, and the
// text written per 1024-word range by one warp each at scanned offsets.
#define SKG_GRID_FOR(i, n) \
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += gridDim.x * blockDim.x)

__device__ __forceinline__ void warp_add(uint32_t* dst, uint32_t v) {   // warp-aggregated atomicAdd
  const unsigned act = __activemask();
  const uint32_t sum = __reduce_add_sync(act, v);
  if (lane_id() == (uint32_t)(__ffs(act) - 1) && sum) atomicAdd(dst, sum);
}

__global__ void bd_classify(const Mod* mp, Tables T) {
  Mod m = *mp;
  SKG_GRID_FOR(i, m.I) classify_one(m, T, i);
}

__global__ void bd_collect(const Mod* mp) {
  Mod m = *mp;
  SKG_GRID_FOR(k, m.W - 5) collect_one(m, 5 + k);
}

// first instruction of each error kind, in disasm_one's evaluation order
__global__ void bd_errors(const Mod* mp, uint32_t* ctl, uint32_t opts, bool names_mode) {
  const Mod m = *mp;
  uint32_t e1 = NONE32, e2 = NONE32, e3 = NONE32;
  SKG_GRID_FOR(i, m.I) {
    const uint32_t d = m.idef[i], e = m.ierr[i];
    if (m.iflag[i] & IF_PRESCAN_UTF8) e1 = min(e1, i);
    if (names_mode && d != NONE16 && e != W_OK && !werr_is_codec(e)) e2 = min(e2, i);
    if ((d == NONE16 && (opts & OPT_STRICT)) || (d != NONE16 && e != W_OK)) e3 = min(e3, i);
  }
  if (e1 != NONE32) atomicMin(&ctl[BC_E1], e1);
  if (e2 != NONE32) atomicMin(&ctl[BC_E2], e2);
  if (e3 != NONE32) atomicMin(&ctl[BC_E3], e3);
}

__global__ void bd_error_rec(const Mod* mp, Tables T, uint32_t which, uint32_t i, ErrRec* rec, int32_t* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const Mod m = *mp;
  int32_t st;
  if (which == 1) {
    st = ST_UNICODE;
    report_prescan_error(m, T, i, rec, 0);
  } else if (m.idef[i] == NONE16) {
    st = ST_CODEC;
    if (rec) {
      ErrWriter ew{rec};
      put_cstr(ew, "unknown opcode "); put_u64(ew, inst_opcode(m, i));
      rec->module = 0; rec->cls = ST_CODEC; rec->len = ew.n;
    }
  } else {
    report_inst_error(m, T, i, rec, 0, st);
  }
  *status = st;
}

// -- names (resolve_names, step by step) -------------------------------------------
__global__ void bn_flags(const Mod* mp, uint32_t* ctl) {
  Mod m = *mp;
  SKG_GRID_FOR(s, m.S) warp_add(&ctl[BC_NP0], nm_slot_flags(m, s) ? 1u : 0u);
}

// per instruction: ib = in C, ia = named definition (scanned into ranks next)
__global__ void bn_mark(const Mod* mp, Tables T) {
  Mod m = *mp;
  SKG_GRID_FOR(i, m.I) {
    bool isC, isN;
    uint32_t slot;
    nm_def_pred(m, T, i, isC, isN, slot);
    m.ib[i] = isC ? 1 : 0;
    m.ia[i] = isN ? 1 : 0;
    m.iflag[i] = (m.iflag[i] & ~IF_FIRSTDEF) | (isC ? IF_FIRSTDEF : 0);
  }
}

__global__ void bn_ndl(const Mod* mp, Tables T) {
  Mod m = *mp;
  SKG_GRID_FOR(i, m.I) {
    bool isC, isN;
    uint32_t slot;
    nm_def_pred(m, T, i, isC, isN, slot);
    if (isN) m.ndl[m.ia[i]] = slot;
  }
}

__global__ void bn_pos(const Mod* mp, Tables T, uint32_t N, uint32_t step) {
  Mod m = *mp;
  if (step == 0) { SKG_GRID_FOR(v, N + 1) m.pos[v] = 0x7FFFFFFF; }
  else if (step == 1) { SKG_GRID_FOR(s, m.S) if ((m.hfl[s] & HF_P0) && s >= 1 && s <= N) m.pos[s] = -1; }
  else {
    SKG_GRID_FOR(i, m.I) {
      if (!(m.iflag[i] & IF_FIRSTDEF)) continue;
      const uint32_t key = nm_def_key(m, T, i);
      if (key >= 1 && key <= N) m.pos[key] = (int32_t)m.ib[i];
    }
  }
}

__global__ void bn_kept(const Mod* mp, Tables T, uint32_t N) {
  Mod m = *mp;
  SKG_GRID_FOR(i, m.I) {
    if (!(m.iflag[i] & IF_FIRSTDEF)) continue;
    const uint32_t key = nm_def_key(m, T, i);
    const int32_t j = (int32_t)m.ib[i];
    if (key >= 1 && key <= N && (key == 1 || m.pos[key - 1] < j)) m.hfl[key] |= HF_KEPT;
  }
}

__global__ void bn_step(const Mod* mp, uint32_t* htab, uint32_t C, uint32_t nd, uint32_t step) {
  Mod m = *mp;
  if (step == 0) { SKG_GRID_FOR(k, nd) nm_info(m, k); }
  else if (step == 1) { SKG_GRID_FOR(e, C) { htab[2 * e] = EMPTY; htab[2 * e + 1] = EMPTY; } }
  else if (step == 2) { SKG_GRID_FOR(k, nd) nm_hinsert(htab, C, m.nH[m.ndl[k]], k); }
  else if (step == 3) { SKG_GRID_FOR(k, nd) m.pos[k] = (int32_t)nm_leader(m, htab, C, k); }
  else if (step == 4) { SKG_GRID_FOR(k, nd) m.ib[k] = nm_parent(m, htab, C, nd, k); }
  else if (step == 5) { SKG_GRID_FOR(k, nd) nm_mark_parent(m, k); }
}

// child list: flags -> (scan) -> entries; then the sequential dedup (one thread)
__global__ void bn_children(const Mod* mp, uint32_t* flags, uint32_t* clist, uint32_t nd, uint32_t step) {
  Mod m = *mp;
  if (step == 0) { SKG_GRID_FOR(k, nd) flags[k] = m.ib[k] != NONE32 ? 1 : 0; }
  else {
    SKG_GRID_FOR(k, nd) {
      if (m.ib[k] == NONE32) continue;
      const uint32_t at = flags[k];
      clist[3 * at] = m.ib[k]; clist[3 * at + 1] = m.ia[k]; clist[3 * at + 2] = k;
    }
  }
}

// ---- name de-duplication of one large module in closed form (replaced round 1's
// ordered pass on one CTA).  disasm.py:173-185 gives the k-th named ident
// (D order) the first free of base, base_0, base_1, ...  A candidate "B_s" of
// group B (idents with sanitized base B) can only be taken by an earlier member of
// B or by the bare name of the child group C whose literal base reads "B_s" (no
// other group generates that string); C's bare name can only be taken by B's
// serial s.  So with B's members sorted in D order, B's requests (all members but
// the first when B's bare name is free) take serials 0, 1, 2 ... skipping serial s
// exactly when child "B_s"'s first member comes before the request that would take
// s; otherwise B takes s and the child's bare name is taken.  Groups are decided
// top-down over the parent / child tree (one thread per group per tree level),
// then every member's serial is q + (skips at requests <= q).
__global__ void bnc_keys(const Mod* mp, uint32_t nd, uint32_t* keys, uint32_t* vals, const uint32_t* clist,
                         uint32_t nc, unsigned long long* ckeys, uint32_t* cvals) {
  const Mod m = *mp;
  SKG_GRID_FOR(k, nd) { keys[k] = (uint32_t)m.pos[k]; vals[k] = k; }
  SKG_GRID_FOR(j, nc) {
    ckeys[j] = ((unsigned long long)clist[3 * j] << 32) | clist[3 * j + 1];   // (parent leader, serial)
    cvals[j] = clist[3 * j + 2];                                               // child leader
  }
}

// group ranges in the sorted member list and in the sorted child list (indexed by
// leader); depth of every group with children (parent chain length)
__global__ void bnc_ranges(const Mod* mp, uint32_t nd, const uint32_t* skeys, uint32_t* gstart, uint32_t* gend,
                           uint32_t nc, const unsigned long long* sckeys, uint32_t* cstart, uint32_t* cend,
                           uint32_t* depth, uint32_t* ctl) {
  const Mod m = *mp;
  SKG_GRID_FOR(i, nd) {
    const uint32_t g = skeys[i];
    if (i == 0 || skeys[i - 1] != g) gstart[g] = i;
    if (i + 1 == nd || skeys[i + 1] != g) gend[g] = i + 1;
  }
  SKG_GRID_FOR(j, nc) {
    const uint32_t p = (uint32_t)(sckeys[j] >> 32);
    if (j == 0 || (uint32_t)(sckeys[j - 1] >> 32) != p) {
      cstart[p] = j;
      uint32_t d = 0;
      for (uint32_t q = m.ib[p]; q != NONE32 && d < nd; q = m.ib[q]) ++d;
      depth[p] = d;
      atomicMax(&ctl[BC_DEPTH], d);
    }
    if (j + 1 == nc || (uint32_t)(sckeys[j + 1] >> 32) != p) cend[p] = j + 1;
  }
}

// one thread per group with children at tree level `level`: its skips and its
// children's bare-name status
__global__ void bnc_level(uint32_t nc, const unsigned long long* sckeys, const uint32_t* scvals,
                          const uint32_t* svals, const uint32_t* gstart, const uint32_t* gend,
                          const uint32_t* cstart, const uint32_t* cend, const uint32_t* depth, uint32_t level,
                          uint8_t* btaken, uint32_t* skipq, uint32_t* nskip) {
  SKG_GRID_FOR(j0, nc) {
    const uint32_t g = (uint32_t)(sckeys[j0] >> 32);
    if (cstart[g] != j0 || depth[g] != level) continue;
    const bool bfree = !btaken[g];
    const uint32_t n = gend[g] - gstart[g];
    const uint32_t nreq = bfree ? n - 1 : n, off = gstart[g] + (bfree ? 1u : 0u);
    uint32_t delta = 0, ns = 0;
    #pragma unroll 1
    for (uint32_t j = j0; j < cend[g]; ++j) {
      const uint32_t sigma = (uint32_t)sckeys[j], c = scvals[j];
      const uint32_t q = sigma - delta;
      if (q >= nreq) break;                        // g never reaches this serial (nor the later ones)
      if (c < svals[off + q]) { skipq[j0 + ns++] = q; ++delta; }   // the child's bare name came first
      else btaken[c] = 1;                          // g took serial sigma before the child appeared
    }
    nskip[g] = ns;
  }
}

__global__ void bnc_assign(const Mod* mp, uint32_t nd, const uint32_t* skeys, const uint32_t* svals,
                           const uint32_t* gstart, const uint8_t* btaken, const uint32_t* cstart,
                           const uint32_t* skipq, const uint32_t* nskip) {
  const Mod m = *mp;
  SKG_GRID_FOR(i, nd) {
    const uint32_t g = skeys[i], k = svals[i];
    const bool bfree = !btaken[g];
    const uint32_t j = i - gstart[g];
    uint32_t serial = NONE32;
    if (!(bfree && j == 0)) {
      const uint32_t q = j - (bfree ? 1u : 0u);
      uint32_t lo = 0, hi = nskip[g];               // skips at requests <= q (ascending)
      const uint32_t* sk = skipq + cstart[g];
      while (lo < hi) { const uint32_t mid = (lo + hi) >> 1; if (sk[mid] <= q) lo = mid + 1; else hi = mid; }
      serial = q + lo;
    }
    m.hser[m.ndl[k]] = serial;
  }
}

__global__ void bn_arena(const Mod* mp, uint32_t* lens, uint32_t nd, uint32_t step) {
  Mod m = *mp;
  if (step == 0) {
    SKG_GRID_FOR(k, nd) { const uint32_t s = m.ndl[k]; lens[k] = (m.hfl[s] & HF_KEPT) ? m.nLen[s] : 0; }
  } else {
    SKG_GRID_FOR(k, nd) if (m.hfl[m.ndl[k]] & HF_KEPT) nm_arena_write(m, k, lens[k]);
  }
}

// -- refs, sizes, text -------------------------------------------------------------
__global__ void bd_refs(const Mod* mp, Tables T, uint32_t* ctl, uint32_t step) {
  Mod m = *mp;
  if (step == 0) {
    SKG_GRID_FOR(s, m.S) { const uint32_t r = ref_len_slow(m, s); m.hrl[s] = (uint16_t)(r > 0xFFFE ? 0xFFFF : r); }
  } else {
    uint32_t width = 0;
    SKG_GRID_FOR(i, m.I) width = max(width, result_ref_one(m, T, i));
    if (width) atomicMax(&ctl[BC_WIDTH], width);
  }
}

__global__ void bd_blanks(const Mod* mp) {
  Mod m = *mp;
  SKG_GRID_FOR(i, m.I) if (i >= 1 && m.isec[i] != m.isec[i - 1]) m.wk[m.ioff[i]] |= WK_BLANK;
}

__global__ void bd_sections(const Mod* mp, Tables T) {   // one warp (sequential section state)
  Mod m = *mp;
  compute_sections(m, T);
}

__global__ void bd_header_len(const Mod* mp, uint32_t opts, uint32_t* ctl) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    ctl[BC_TOTAL] = (opts & OPT_NO_HEADER) ? 0 : header_len(*mp, opts & OPT_HIGHLIGHT);
}

constexpr uint32_t BD_RANGE = 1024;   // words per render range (one warp each)

// word lengths (stored) and per-range sums
__global__ void bd_lengths(const Mod* mp, Tables T, uint32_t opts, uint32_t width, uint32_t* rsum) {
  const Mod m = *mp;
  const bool hl = opts & OPT_HIGHLIGHT;
  const uint32_t nr = (m.W - 5 + BD_RANGE - 1) / BD_RANGE;
  const uint32_t wpb = blockDim.x >> 5, warp = threadIdx.x >> 5;
  for (uint32_t r = blockIdx.x * wpb + warp; r < nr; r += gridDim.x * wpb) {
    const uint32_t w0 = 5 + r * BD_RANGE, w1 = min(w0 + BD_RANGE, m.W);
    uint32_t sum = 0;
    for (uint32_t w = w0 + lane_id(); w < w1; w += 32) {
      const uint32_t l = word_len(m, T, w, m.wk[w], width, hl);
      m.wl[w] = (uint16_t)(l > 0xFFFF ? 0xFFFF : l);
      sum += l;
    }
    sum = warp_sum_u32(sum);
    if (lane_id() == 0) rsum[r] = sum;
  }
}

__global__ void bd_render(const Mod* mp, Tables T, uint32_t opts, uint32_t width, uint8_t* out,
                          const uint32_t* roff, uint32_t head) {
  extern __shared__ __align__(16) uint8_t smem[];
  const Mod m = *mp;
  const uint32_t nr = (m.W - 5 + BD_RANGE - 1) / BD_RANGE;
  const uint32_t wpb = blockDim.x >> 5, warp = threadIdx.x >> 5;
  uint8_t* stage = smem + 1024 * warp;
  if (nr == 0 && blockIdx.x == 0 && warp == 0 && head)
    text_write_range(m, T, opts, width, out, stage, 1024, 5, 5, 0, true);
  for (uint32_t r = blockIdx.x * wpb + warp; r < nr; r += gridDim.x * wpb) {
    const uint32_t w0 = 5 + r * BD_RANGE, w1 = min(w0 + BD_RANGE, m.W);
    text_write_range(m, T, opts, width, out, stage, 1024, w0, w1, (uint64_t)head + roff[r], r == 0 && head);
  }
}

}  // namespace skg
