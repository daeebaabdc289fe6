// Per-module device state shared by the disassembler and validator kernels.
//
// One warp owns one module at a time.  Its scratch (words, instruction table,
// id hash table, ...) lives in a shared-memory slab when it fits and in a
// per-warp global-memory slot otherwise.  Phases (all warp-synchronous):
//   load      : 16-byte loads of the module bytes, byte-swap if big-endian
//               (codec.py:199-216)
//   boundary  : instruction-boundary walk with the exact wc==0 / overrun
//               errors (codec.py:217-230)
//   prescan   : per-instruction grammar lookup + the per-id maps the reference
//               keeps in dicts -- type_info / value_type (last wins), first
//               OpName, last OpExtInstImport, first definition (disasm.py:131-157,
//               208-219; validate.py:179-192).  "First/last wins" is resolved by
//               processing instructions in lane-strided chunks in document order
//               and letting the lowest/highest lane of each equal-key group write.
#pragma once
#include "skg_walk.cuh"

namespace skg {

constexpr uint32_t MAGIC = 0x07230203u;
constexpr uint32_t EMPTY = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xFFFFFFFFu;

// exception classes reported per module (python: _native.STATUS)
enum : int32_t {
  ST_OK = 0, ST_TRUNCATED = 1, ST_NOTSPIRV = 2, ST_CORRUPT = 3, ST_CODEC = 4, ST_UNICODE = 5,
  ST_KEY = 6, ST_VALUE = 7, ST_OVERFLOW = 8, ST_ASSEMBLY = 9, ST_STRUCTURE = 10,
  ST_SERIALIZATION = 11, ST_SCOPE = 12, ST_NOTFOUND = 13, ST_INTERNAL = 99
};

struct ErrRec {            // 256 bytes
  int32_t module;
  int32_t cls;
  uint32_t a, b, c, d;     // UnicodeDecodeError: start, end, reason, byte; KeyError: key
  int32_t len;
  char msg[228];
};

// iflag bits
enum : uint8_t { IF_PRESCAN_UTF8 = 1, IF_HAS_RESULT = 2, IF_EXT_KNOWN = 4, IF_FIRSTDEF = 8 };
// hfl bits
enum : uint8_t { HF_NAMED_D = 1, HF_P0 = 2, HF_KEPT = 4, HF_FRIENDLY = 8 };

struct Mod {
  uint8_t* base;          // scratch base (64-byte header of counters)
  uint32_t* w;            // words (normalised to little-endian values)
  uint32_t W;
  uint32_t* ioff;         // instruction start word offsets, I entries
  uint32_t I;
  // per instruction
  uint16_t* idef;
  uint8_t* iflag;
  uint8_t* ierr;
  uint8_t* isec;
  uint32_t* ia;
  uint32_t* ib;
  uint16_t* irl;
  uint32_t* wk;           // per word render code (disassembler)
  uint16_t* wl;           // per word text length (disassembler size pass)
  // per id "slot": direct mode slot = id (ids < bound, the canonical case);
  // hash mode (any id >= bound seen): open addressing over hkey, slot C holds 0xFFFFFFFF
  bool direct;
  uint32_t S;             // number of slots
  uint32_t C, shift;      // hash mode
  uint32_t* hkey;
  uint32_t* hdef;         // first definition (instruction index)
  uint32_t* hti;          // type_info: last OpTypeInt/OpTypeFloat
  uint32_t* hvt;          // value_type: last instruction with this result
  uint32_t* hname;        // first decodable OpName
  uint32_t* himp;         // last decodable OpExtInstImport
  uint32_t* hser;         // friendly-name serial (NONE32: bare base)
  uint32_t* nH;           // sanitized-name hash / prefix hash / length
  uint32_t* nP;
  uint32_t* nLen;
  uint32_t* ndl;          // named definitions in D order (slots)
  uint32_t* hnoff;        // friendly: offset of the sanitized base name in narena
  uint8_t* narena;        // sanitized base names of friendly ids (disassembler)
  uint4* fpc;             // per word: the float repr parts of a typed float literal, computed by
                          // the size pass for the write pass (nullptr: no room, recompute)
  uint32_t arena_need;    // bound on narena bytes: sum over OpName of 4 * string words + 1
  int32_t* pos;           // closed-form demotion scan, S + 2 entries
  uint16_t* hrl;          // friendly ref length
  uint8_t* hA;            // referenced by a decodable instruction
  uint8_t* hfl;
  uint8_t* hpres;         // slot in use
  uint8_t* spill;         // global scratch for the rare sequential name-dedup path
  uint8_t* work;          // name-resolution arrays, then the render workspace
  uint32_t work_bytes;
  bool work_shared;       // work region is in shared memory
  uint32_t* fill;         // header counters
  uint32_t* overflow;
  uint32_t* top_present;
  uint32_t major, minor, gen, bound, schema;
  // explicit refs (format_instruction with a RenderContext, disasm.py:57-67): ids in
  // ascending order with (text offset, length) of their full ref text; 0 = none
  const uint32_t* ovr;        // 3 words per entry
  const uint8_t* ovr_text;
  uint32_t n_ovr;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// Scratch layout of one module (shared slab or global slot):
//   [64 B counters][words: W][instruction offsets: I+1][per-instruction arrays]
//   [per-id slot arrays][work: friendly-name arrays, later the render workspace]
__host__ __device__ inline size_t head_bytes(uint32_t W) {      // before the boundary walk
  return 64 + align16(4ull * W) + align16(4ull * (W > 5 ? W - 5 : 1) + 4);
}
__host__ __device__ inline size_t head_used(uint32_t W, uint32_t I) {
  return 64 + align16(4ull * W) + align16(4ull * (I + 1));
}
__host__ __device__ inline size_t inst_bytes(uint32_t I) {
  return align16(2ull * I) + 3 * align16(1ull * I) + 2 * align16(4ull * I) + align16(2ull * I);
}
__host__ __device__ inline size_t word_bytes(uint32_t W) { return align16(4ull * W) + align16(2ull * W); }
__host__ __device__ inline size_t slot_bytes(uint32_t S, bool hash) {
  return (hash ? align16(4ull * S) : 0) + 6 * align16(4ull * S) + align16(2ull * S) +
         3 * align16(1ull * S);
}
__host__ __device__ inline size_t names_bytes(uint32_t S) {
  return 5 * align16(4ull * S) + align16(4ull * (S + 2));
}
__host__ __device__ inline size_t spill_bytes(uint32_t I) { return 32ull * I + 64; }
__host__ __device__ inline uint32_t hash_capacity(uint32_t W) {
  uint32_t C = 64;
  while (C < 2 * W + 8) C <<= 1;
  return C;
}
__host__ __device__ inline size_t work_need(uint32_t S, size_t work_min, size_t arena) {
  size_t nb = names_bytes(S) + align16(arena);
  return nb > work_min ? nb : work_min;
}
// worst case for a module of W words: hash mode in the global slot
__host__ __device__ inline size_t worst_bytes(uint32_t W, size_t work_min) {
  uint32_t I = W > 5 ? W - 5 : 0;
  uint32_t S = hash_capacity(W) + 1;
  return head_bytes(W) + inst_bytes(I) + word_bytes(W) + slot_bytes(S, true) +
         work_need(S, work_min, 5ull * W) + spill_bytes(I);
}

__device__ inline void layout_head(Mod& m, uint8_t* base, uint32_t W) {
  m.base = base;
  m.fill = reinterpret_cast<uint32_t*>(base);
  m.overflow = m.fill + 1;
  m.top_present = m.fill + 2;
  m.w = reinterpret_cast<uint32_t*>(base + 64);
  m.W = W;
  m.ioff = reinterpret_cast<uint32_t*>(base + 64 + align16(4ull * W));
  m.ovr = nullptr; m.ovr_text = nullptr; m.n_ovr = 0;
}

__device__ inline size_t tables_need(const Mod& m, bool direct, uint32_t S_or_C, size_t work_min) {
  const uint32_t S = direct ? S_or_C : S_or_C + 1;
  return head_used(m.W, m.I) + inst_bytes(m.I) + word_bytes(m.W) + slot_bytes(S, !direct) +
         work_need(S, work_min, m.arena_need);
}

// lay out per-instruction, per-slot and work arrays after the instruction offsets
__device__ inline void layout_tables(Mod& m, bool direct, uint32_t S_or_C, size_t region_bytes,
                                     size_t work_min) {
  uint8_t* p = m.base + head_used(m.W, m.I);
  const uint32_t I = m.I;
  auto take = [&](size_t bytes) { uint8_t* r = p; p += align16(bytes); return r; };
  m.idef = reinterpret_cast<uint16_t*>(take(2ull * I));
  m.iflag = take(I);
  m.ierr = take(I);
  m.isec = take(I);
  m.ia = reinterpret_cast<uint32_t*>(take(4ull * I));
  m.ib = reinterpret_cast<uint32_t*>(take(4ull * I));
  m.irl = reinterpret_cast<uint16_t*>(take(2ull * I));
  m.wk = reinterpret_cast<uint32_t*>(take(4ull * m.W));
  m.wl = reinterpret_cast<uint16_t*>(take(2ull * m.W));
  m.direct = direct;
  if (direct) {
    m.S = S_or_C; m.C = 0; m.shift = 0; m.hkey = nullptr;
  } else {
    m.C = S_or_C; m.S = S_or_C + 1;
    uint32_t lg = 0;
    while ((1u << lg) < m.C) ++lg;
    m.shift = 32 - lg;
    m.hkey = reinterpret_cast<uint32_t*>(take(4ull * m.S));
  }
  const uint32_t S = m.S;
  m.hdef = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.hti = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.hvt = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.hname = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.himp = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.hser = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.hrl = reinterpret_cast<uint16_t*>(take(2ull * S));
  m.hA = take(S);
  m.hfl = take(S);
  m.hpres = take(S);
  // work region: the friendly-name arrays live here during name resolution;
  // the render workspace reuses the same bytes afterwards
  m.work = p;
  const size_t used = (size_t)(p - m.base);
  size_t wb = work_need(S, work_min, m.arena_need);
  if (region_bytes > used + wb) wb = region_bytes - used;
  m.work_bytes = (uint32_t)wb;
  m.nH = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.nP = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.nLen = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.ndl = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.pos = reinterpret_cast<int32_t*>(take(4ull * (S + 2)));
  m.hnoff = reinterpret_cast<uint32_t*>(take(4ull * S));
  m.narena = take(m.arena_need);
  // the rest of the work region: the float repr cache, 16 bytes per word (disassembler)
  m.fpc = (size_t)(m.work + m.work_bytes - p) >= 16ull * m.W ? reinterpret_cast<uint4*>(p) : nullptr;
}

// -- warp helpers -------------------------------------------------------------
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint32_t warp_incl_sum(uint32_t v) {
  const uint32_t l = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t = __shfl_up_sync(FULL, v, d);
    if (l >= (uint32_t)d) v += t;
  }
  return v;
}

__device__ __forceinline__ int32_t warp_incl_max(int32_t v) {
  const uint32_t l = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int32_t t = __shfl_up_sync(FULL, v, d);
    if (l >= (uint32_t)d) v = max(v, t);
  }
  return v;
}

__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = max(v, __shfl_xor_sync(FULL, v, d));
  return v;
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
  return v;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// -- id table -------------------------------------------------------------------
__device__ __forceinline__ uint32_t ht_home(const Mod& m, uint32_t key) {
  return (key * 0x9E3779B1u) >> m.shift;
}

__device__ inline uint32_t ht_find(const Mod& m, uint32_t key) {
  if (m.direct) return (key < m.S && m.hpres[key]) ? key : NONE32;
  if (key == EMPTY) return *m.top_present ? m.C : NONE32;   // dedicated slot for 0xFFFFFFFF
  uint32_t s = ht_home(m, key);
  for (uint32_t probe = 0; probe < m.C; ++probe) {
    uint32_t k = m.hkey[s];
    if (k == key) return s;
    if (k == EMPTY) return NONE32;
    s = (s + 1) & (m.C - 1);
  }
  return NONE32;
}

__device__ inline uint32_t ht_insert(const Mod& m, uint32_t key) {
  if (m.direct) {
    if (key < m.S) { m.hpres[key] = 1; return key; }
    *m.overflow = 1;
    return NONE32;
  }
  if (key == EMPTY) {
    *m.top_present = 1;
    m.hpres[m.C] = 1;
    return m.C;
  }
  uint32_t s = ht_home(m, key);
  for (uint32_t probe = 0; probe < m.C; ++probe) {
    uint32_t k = m.hkey[s];
    if (k == key) return s;
    if (k == EMPTY) {
      uint32_t old = atomicCAS(&m.hkey[s], EMPTY, key);
      if (old == EMPTY) { m.hpres[s] = 1; return s; }
      if (old == key) return s;
    }
    s = (s + 1) & (m.C - 1);
  }
  *m.overflow = 1;
  return NONE32;
}

// key held by a slot (valid when hpres[slot])
__device__ __forceinline__ uint32_t slot_key(const Mod& m, uint32_t s) {
  if (m.direct) return s;
  return s < m.C ? m.hkey[s] : EMPTY;
}

// -- instruction accessors ------------------------------------------------------
__device__ __forceinline__ uint32_t inst_start(const Mod& m, uint32_t i) { return m.ioff[i]; }
__device__ __forceinline__ uint32_t inst_nops(const Mod& m, uint32_t i) { return (m.w[m.ioff[i]] >> 16) - 1; }
__device__ __forceinline__ uint32_t inst_opcode(const Mod& m, uint32_t i) { return m.w[m.ioff[i]] & 0xFFFF; }
__device__ __forceinline__ const uint32_t* inst_ops(const Mod& m, uint32_t i) { return m.w + m.ioff[i] + 1; }

// -- resolver (RenderContext.literal_resolver / validate._make_resolver) ---------
struct Resolver {
  const Mod* m;
  const Tables* T;
  __device__ __noinline__ Width rt(uint32_t id) const {
    uint32_t s = ht_find(*m, id);
    if (s == NONE32 || m->hti[s] == NONE32) return Width{0, false, false, false};
    uint32_t j = m->hti[s];
    const uint32_t* ops = inst_ops(*m, j);
    uint32_t d = m->idef[j];
    if (T->special(d) == SP_TYPEINT) return Width{ops[1], ops[2] == 1, false, true};
    return Width{ops[1], false, true, true};
  }
  __device__ __noinline__ Width sel(uint32_t selector) const {
    uint32_t s = ht_find(*m, selector);
    if (s == NONE32 || m->hvt[s] == NONE32) return Width{0, false, false, false};
    return rt(inst_ops(*m, m->hvt[s])[0]);
  }
};

struct NullVis {
  __device__ void id(uint32_t, uint32_t, int, uint32_t) {}
  __device__ void venum(uint32_t, uint32_t, uint32_t, uint32_t) {}
  __device__ void benum(uint32_t, uint32_t, bool, uint64_t, uint32_t) {}
  __device__ void str(const uint32_t*, uint32_t, uint32_t) {}
  __device__ void typed(const LitVal&, uint32_t, uint32_t) {}
  __device__ void lit(uint32_t, uint32_t, uint32_t) {}
  __device__ void comp_begin() {}
  __device__ void comp_end() {}
};

// -- error records --------------------------------------------------------------
struct ErrWriter {
  ErrRec* rec;
  int32_t n = 0;
  __device__ void put(uint8_t c) { if (n < (int32_t)sizeof(rec->msg) - 1) rec->msg[n] = (char)c; ++n; }
  __device__ void putn(const uint8_t* s, uint32_t len) { for (uint32_t i = 0; i < len; ++i) put(s[i]); }
  __device__ void fill(uint8_t c, uint32_t k) { for (uint32_t i = 0; i < k; ++i) put(c); }
};

// Batch-wide outputs common to all kernels
struct ErrSink {
  ErrRec* recs;
  uint32_t* count;
  uint32_t cap;
  __device__ ErrRec* alloc() {
    uint32_t k = atomicAdd(count, 1u);
    return k < cap ? recs + k : nullptr;
  }
};

// Compose the str(exc) text of a walk error (ops.py:351-374, codec.py:127-129,
// ops.py:420-422, CPython UnicodeDecodeError.__str__).
template <class S>
__device__ __noinline__ void put_walk_error(S& s, const Tables& T, uint32_t idef, const WalkErr& e) {
  auto opname = [&]() { s.putn(T.str + T.iname_off(idef), T.iname_len(idef)); };
  switch (e.code) {
    case W_EXHAUSTED: opname(); put_cstr(s, ": operand words exhausted mid-instruction"); break;
    case W_LEFTOVER: opname(); put_cstr(s, ": "); put_u64(s, e.a); put_cstr(s, " leftover operand word(s)"); break;
    case W_NONUL: put_cstr(s, "string literal is not NUL-terminated"); break;
    case W_UNRESOLVED: opname(); put_cstr(s, ": cannot resolve the width of a context-dependent literal"); break;
    case W_UNICODE:
      put_cstr(s, "'utf-8' codec can't decode ");
      if (e.b - e.a == 1) {
        put_cstr(s, "byte 0x"); put_hex2_lower(s, e.d); put_cstr(s, " in position "); put_u64(s, e.a);
      } else {
        put_cstr(s, "bytes in position "); put_u64(s, e.a); s.put('-'); put_u64(s, e.b - 1);
      }
      put_cstr(s, e.c == U8_START ? ": invalid start byte"
                  : e.c == U8_CONT ? ": invalid continuation byte" : ": unexpected end of data");
      break;
    case W_KEY: put_u64(s, e.a); break;
    case W_VALUE: put_cstr(s, "negative shift count"); break;
    default: break;
  }
}

__device__ inline int32_t walk_status(uint32_t code) {
  if (werr_is_codec(code)) return ST_CORRUPT;
  if (code == W_UNICODE) return ST_UNICODE;
  if (code == W_KEY) return ST_KEY;
  return ST_VALUE;
}



// ---------------------------------------------------------------------------
// load + boundary.  Returns ST_OK or an error class; on error fills `err`
// (on lane 0).  Words are loaded into m.w (already laid out via layout_head).
__device__ __noinline__ int32_t load_and_split(Mod& m, const uint8_t* src, uint64_t nbytes, ErrSink* es,
                                         int32_t module) {
  const uint32_t lane = lane_id();
  ErrRec* err = nullptr;
  if (nbytes % 4 != 0 || nbytes < 20) {
    if (lane == 0 && es) err = es->alloc();
    if (lane == 0 && err) {
      ErrWriter ew{err};
      put_u64(ew, nbytes);
      put_cstr(ew, " bytes is not a whole word stream of at least 5 words");
      err->module = module; err->cls = ST_TRUNCATED; err->len = ew.n;
    }
    return ST_TRUNCATED;
  }
  const uint32_t W = (uint32_t)(nbytes / 4);
#ifndef SKG_EXP_NO_PREFETCH
  prefetch_l2(src, nbytes);
#endif
  // little-endian, word-aligned input (the batch case): read the words in place
  // (the input arena is read-only for the kernel; no scratch copy)
  if ((reinterpret_cast<uintptr_t>(src) & 3) == 0 &&
      __ldg(reinterpret_cast<const uint32_t*>(src)) == MAGIC) {
    m.w = const_cast<uint32_t*>(reinterpret_cast<const uint32_t*>(src));
  } else if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {   // 16-byte vector loads
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(m.w);
    const uint32_t n4 = W / 4;
    for (uint32_t k = lane; k < n4; k += 32) d4[k] = __ldcs(s4 + k);   // read once: evict first
    for (uint32_t k = n4 * 4 + lane; k < W; k += 32) m.w[k] = __ldg(reinterpret_cast<const uint32_t*>(src) + k);
  } else {
    for (uint32_t k = lane; k < W; k += 32) {
      const uint8_t* p = src + 4ull * k;
      m.w[k] = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
    }
  }
  __syncwarp();
  const uint32_t w0 = m.w[0];
  if (w0 != MAGIC) {
    if (bswap32(w0) != MAGIC) {
      if (lane == 0 && es) err = es->alloc();
      if (lane == 0 && err) {
        ErrWriter ew{err};
        put_cstr(ew, "magic word 0x"); put_hex8_upper(ew, w0); put_cstr(ew, " is not SPIR-V");
        err->module = module; err->cls = ST_NOTSPIRV; err->len = ew.n;
      }
      return ST_NOTSPIRV;
    }
    for (uint32_t k = lane; k < W; k += 32) m.w[k] = bswap32(m.w[k]);
    __syncwarp();
  }
  m.major = (m.w[1] >> 16) & 0xFF;
  m.minor = (m.w[1] >> 8) & 0xFF;
  m.gen = m.w[2];
  m.bound = m.w[3];
  m.schema = m.w[4];
  // instruction-boundary walk (codec.py:212-229: pos += wc), warp-cooperative: the
  // window [p, p + 32) is loaded one word per lane (coalesced), the chase inside it
  // runs on shuffles (no dependent memory loads), and the lanes that hold a start
  // write their offsets; the next window starts at the next instruction.
  int32_t st = ST_OK;
  uint32_t I = 0, bad = 0, arena = 0;
  uint32_t p = 5;
  while (p < W) {
    const uint32_t base = p;
    const uint32_t x = base + lane < W ? m.w[base + lane] : 0;
    uint32_t starts = 0;
    while (p < W && p < base + 32) {   // p is warp-uniform
      const uint32_t wc = __shfl_sync(FULL, x, p - base) >> 16;
      if (wc == 0) { st = ST_CORRUPT; bad = p; break; }
      if (p + wc > W) { st = ST_TRUNCATED; bad = p; break; }
      starts |= 1u << (p - base);
      p += wc;
    }
    const bool mine = (starts >> lane) & 1;
    if (mine) {
      m.ioff[I + __popc(starts & ((1u << lane) - 1))] = base + lane;
      const uint32_t wc = x >> 16;
      if ((x & 0xFFFF) == 5 && wc > 2) arena += 4 * (wc - 2) + 1;   // OpName: sanitized name bound
    }
    I += __popc(starts);
    if (st != ST_OK) break;
  }
  arena = warp_sum_u32(arena);
  if (st != ST_OK && lane == 0) {
    if (es) err = es->alloc();
    if (err) {
      ErrWriter ew{err};
      put_cstr(ew, "instruction at word "); put_u64(ew, bad);
      put_cstr(ew, st == ST_CORRUPT ? " has word count 0" : " runs past the end of the stream");
      err->module = module; err->cls = st; err->len = ew.n;
    }
  }
  m.I = I;
  m.arena_need = arena;
  __syncwarp();
  return st;
}

__device__ __noinline__ void init_tables(Mod& m) {
  const uint32_t lane = lane_id();
  for (uint32_t s = lane; s < m.S; s += 32) {
    if (!m.direct) m.hkey[s] = EMPTY;
    m.hdef[s] = NONE32; m.hti[s] = NONE32; m.hvt[s] = NONE32; m.hname[s] = NONE32;
    m.himp[s] = NONE32; m.hser[s] = NONE32;
    m.hA[s] = 0; m.hfl[s] = 0; m.hpres[s] = 0;
  }
  if (lane == 0) { *m.fill = 0; *m.overflow = 0; *m.top_present = 0; }
  __syncwarp();
}

// move words + offsets from the shared slab to the global slot
__device__ inline void move_to_global(Mod& m, uint8_t* gslot) {
  Mod g;
  layout_head(g, gslot, m.W);
  for (uint32_t k = lane_id(); k < m.W; k += 32) g.w[k] = m.w[k];
  for (uint32_t k = lane_id(); k < m.I; k += 32) g.ioff[k] = m.ioff[k];
  g.I = m.I; g.arena_need = m.arena_need; g.major = m.major; g.minor = m.minor; g.gen = m.gen; g.bound = m.bound; g.schema = m.schema;
  g.ovr = m.ovr; g.ovr_text = m.ovr_text; g.n_ovr = m.n_ovr;
  __syncwarp();
  m = g;
}

// Lay out the id tables (direct when ids fit below the header bound, hash
// otherwise), moving to the global slot when the shared slab is too small.
// Returns false if even the global slot cannot hold the module.
__device__ __noinline__ bool place_tables(Mod& m, bool direct, bool& in_smem, uint8_t* gslot,
                                    uint64_t gslot_bytes, uint32_t slab_bytes, size_t work_min) {
  const size_t greg = gslot_bytes - spill_bytes(m.I);
  // the slot is sized for hash mode (worst_bytes); a direct table for a bound above the
  // hash capacity (small modules: bound <= 2W + 64) may not fit, hash mode always does
  if (direct && tables_need(m, true, m.bound, work_min) > greg) direct = false;
  const uint32_t SC = direct ? m.bound : hash_capacity(m.W);
  const size_t need = tables_need(m, direct, SC, work_min);
  if (in_smem && need > slab_bytes) {
    if (need > greg) return false;
    move_to_global(m, gslot);
    in_smem = false;
  }
  if (!in_smem && need > greg) return false;
  layout_tables(m, direct, SC, in_smem ? slab_bytes : greg, work_min);
  m.work_shared = in_smem;
  m.spill = gslot + greg;
  return true;
}

// last-writer / first-writer within a chunk for equal keys
__device__ __forceinline__ bool group_last(bool part, uint32_t key) {
  uint64_t k = part ? (uint64_t)key : (0x100000000ull + lane_id());
  unsigned g = __match_any_sync(FULL, k);
  return part && (31 - __clz(g)) == (int)lane_id();
}
__device__ __forceinline__ bool group_first(bool part, uint32_t key) {
  uint64_t k = part ? (uint64_t)key : (0x100000000ull + lane_id());
  unsigned g = __match_any_sync(FULL, k);
  return part && (__ffs(g) - 1) == (int)lane_id();
}

// prescan: returns whether any OpName was recorded
__device__ __noinline__ bool prescan(Mod& m, const Tables& T) {
  const uint32_t lane = lane_id();
  bool any_name = false;
  for (uint32_t base = 0; base < m.I; base += 32) {
    const uint32_t i = base + lane;
    const bool act = i < m.I;
    uint32_t d = NONE32, n = 0, sp = SP_NONE;
    const uint32_t* ops = nullptr;
    if (act) {
      ops = inst_ops(m, i);
      n = inst_nops(m, i);
      d = T.inst_of(inst_opcode(m, i));
      m.idef[i] = d == NONE32 ? NONE16 : (uint16_t)d;
      sp = d == NONE32 ? SP_NONE : T.special(d);
      m.iflag[i] = 0;
      m.ierr[i] = 0;
    }
    // type_info (last wins): OpTypeInt with exactly 3 words / OpTypeFloat >= 2
    {
      bool part = act && ((sp == SP_TYPEINT && n == 3) || (sp == SP_TYPEFLOAT && n >= 2));
      uint32_t key = part ? ops[0] : 0;
      uint32_t slot = part ? ht_insert(m, key) : NONE32;
      if (group_last(part, key) && slot != NONE32) m.hti[slot] = i;
    }
    __syncwarp();
    // value_type (last wins)
    {
      bool part = act && d != NONE32 && T.has_result(d) && T.has_rtype(d) && n >= 2;
      uint32_t key = part ? ops[1] : 0;
      uint32_t slot = part ? ht_insert(m, key) : NONE32;
      if (group_last(part, key) && slot != NONE32) m.hvt[slot] = i;
    }
    __syncwarp();
    // OpExtInstImport (last decodable wins) / OpName (first decodable wins)
    {
      bool part = act && (sp == SP_EXTINSTIMPORT || sp == SP_NAME) && n >= 2;
      if (part) {
        uint32_t nbytes, next;
        if (!string_span(ops, 1, n, nbytes, next)) part = false;
        else {
          WalkErr e;
          if (string_utf8(ops, 1, nbytes, e) != U8_OK) { part = false; m.iflag[i] |= IF_PRESCAN_UTF8; }
        }
      }
      bool imp = part && sp == SP_EXTINSTIMPORT, nam = part && sp == SP_NAME;
      uint32_t key = part ? ops[0] : 0;
      uint32_t slot = part ? ht_insert(m, key) : NONE32;
      if (group_last(imp, key) && slot != NONE32) m.himp[slot] = i;
      if (group_first(nam, key) && slot != NONE32 && m.hname[slot] == NONE32) m.hname[slot] = i;
      any_name |= nam;
    }
    __syncwarp();
    // first definition (definition order D)
    {
      bool part = false;
      uint32_t key = 0;
      if (act && d != NONE32 && T.has_result(d)) {
        uint32_t idx = T.has_rtype(d) ? 1 : 0;
        if (idx < n) { part = true; key = ops[idx]; }
      }
      uint32_t slot = part ? ht_insert(m, key) : NONE32;
      if (group_first(part, key) && slot != NONE32 && m.hdef[slot] == NONE32) m.hdef[slot] = i;
    }
    __syncwarp();
  }
  return __any_sync(FULL, any_name);
}

// Output placement: a bump allocator over the text arena.  Modules are
// independent, so each warp reserves its module's bytes with one atomic and
// never waits on another module (no ordering dependency between tickets).
// counters: [0] ticket, [1] error count, [2] overflow flag, [4..5] u64 cursor
__device__ inline uint64_t alloc_text(uint32_t* counters, uint64_t bytes, uint64_t cap, bool& fits) {
  uint64_t off = 0;
  if (lane_id() == 0 && bytes) {
    off = atomicAdd(reinterpret_cast<unsigned long long*>(counters + 4), (unsigned long long)bytes);
    if (off + bytes > cap) atomicExch(counters + 2, 1u);
  }
  off = __shfl_sync(FULL, off, 0);
  fits = off + bytes <= cap;
  return off;
}

}  // namespace skg
