// Device view of the grammar table blob built by paper_2305_09493_b200/tables.py.
// One little-endian uint32 array; the header (64 words) holds counts and word
// offsets of every section.  All lookups the reference performs through
// Python dicts (grammar.py:97-127, ops.py:376-409) become array indexing here.
#pragma once
#include <cstdint>

namespace skg {

constexpr uint32_t NONE32 = 0xFFFFFFFFu;
constexpr uint16_t NONE16 = 0xFFFFu;

// Barrier of one group of warps of the CTA (named barrier 1 + group; the
// phase-synchronised kernels sync per group of `warps` warps, not per CTA).
__device__ __forceinline__ void group_sync(uint32_t group, uint32_t warps) {
  asm volatile("bar.sync %0, %1;" :: "r"(1 + group), "r"(32 * warps) : "memory");
}


// Ask L2 for every 128-byte line of [p, p + n), one prefetch per lane per 4 KB:
// a module's bytes are then in flight at once instead of one load round trip per
// step of the (dependent) scans that read them.
__device__ __forceinline__ void prefetch_l2(const void* p, uint64_t n) {
  const uint64_t a = reinterpret_cast<uint64_t>(p) & ~127ull, e = reinterpret_cast<uint64_t>(p) + n;
  for (uint64_t q = a + 128ull * (threadIdx.x & 31); q < e; q += 128ull * 32)
    asm volatile("prefetch.global.L2 [%0];" :: "l"(q));
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" :: "l"(p));
}

// ---------------------------------------------------------------------------
// Cross-module work assignment inside one CTA (every warp of the CTA calls it;
// CTA barriers inside).  Warp w offers n entries in `in`, each entry carrying its
// warp in bits 27-31 and an item index below 2^27.  The entries of all warps are
// counting-sorted by key(e) (< CTA_KEYS) into the warps' `out` arrays -- sorted
// position p lives in the out array of the warp whose prefix range holds p, so a
// warp needs room for its own entries only -- and then every warp runs work(e)
// for 32 consecutive positions at a time: the lanes of a warp get items with equal
// or adjacent keys, mostly of different modules, and warps with few items of
// their own (or none: a finished module) take a share of the others'.
constexpr uint32_t CTA_KEYS = 1024;
constexpr uint32_t CTA_ITEM = (1u << 27) - 1;
struct CtaSort {
  uint32_t hist[CTA_KEYS];
  uint32_t pre[33];
  uint32_t* out[32];
};

__device__ __forceinline__ uint32_t cta_owner(const CtaSort& cs, uint32_t nwb, uint32_t p) {
  uint32_t o = 0;   // the largest warp o with pre[o] <= p (the non-empty range holding p)
#pragma unroll
  for (uint32_t step = 16; step; step >>= 1)
    if (o + step < nwb && cs.pre[o + step] <= p) o += step;
  return o;
}

template <class Key, class Work>
__device__ __forceinline__ void cta_dispatch(CtaSort& cs, const uint32_t* in, uint32_t* out, uint32_t n,
                                             Key&& key, Work&& work) {
  const uint32_t lane = threadIdx.x & 31, nwb = blockDim.x >> 5, wib = threadIdx.x >> 5;
  for (uint32_t k = threadIdx.x; k < CTA_KEYS; k += blockDim.x) cs.hist[k] = 0;
  __syncthreads();
  for (uint32_t i = lane; i < n; i += 32) atomicAdd(&cs.hist[min(key(in[i]), CTA_KEYS - 1)], 1u);
  if (lane == 0) { cs.out[wib] = out; cs.pre[wib + 1] = n; }
  __syncthreads();
  if (wib == 0) {   // bucket cursors (exclusive scan of the histogram), per-warp prefix
    auto incl_sum = [&](uint32_t v) {
#pragma unroll
      for (uint32_t d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, d);
        if (lane >= d) v += t;
      }
      return v;
    };
    uint32_t carry = 0;
    for (uint32_t base = 0; base < CTA_KEYS; base += 32) {
      const uint32_t c = cs.hist[base + lane];
      const uint32_t incl = incl_sum(c);
      cs.hist[base + lane] = carry + incl - c;
      carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
    const uint32_t c = lane < nwb ? cs.pre[lane + 1] : 0;
    const uint32_t incl = incl_sum(c);
    if (lane < nwb) cs.pre[lane + 1] = incl;
    if (lane == 0) cs.pre[0] = 0;
  }
  __syncthreads();
  for (uint32_t i = lane; i < n; i += 32) {   // scatter into sorted order
    const uint32_t e = in[i];
    const uint32_t p = atomicAdd(&cs.hist[min(key(e), CTA_KEYS - 1)], 1u);
    const uint32_t o = cta_owner(cs, nwb, p);
    cs.out[o][p - cs.pre[o]] = e;
  }
  __syncthreads();
  const uint32_t total = cs.pre[nwb];
  for (uint32_t c0 = 32 * wib; c0 < total; c0 += 32 * nwb) {
    const uint32_t p = c0 + lane;
    if (p < total) {
      const uint32_t o = cta_owner(cs, nwb, p);
      work(cs.out[o][p - cs.pre[o]]);
    }
  }
  __syncthreads();
}

// instruction special codes (tables.py SPECIAL)
enum : uint32_t {
  SP_NONE = 0, SP_TYPEINT = 1, SP_TYPEFLOAT = 2, SP_EXTINSTIMPORT = 3, SP_NAME = 4, SP_SWITCH = 5,
  SP_EXTINST = 6, SP_FUNCTION = 7, SP_FUNCTIONEND = 8, SP_CAPABILITY = 9, SP_MEMORYMODEL = 10,
  SP_ENTRYPOINT = 11, SP_LABEL = 12, SP_FUNCTIONPARAM = 13, SP_VARIABLE = 14, SP_UNDEF = 15,
  SP_LINE = 16, SP_NOLINE = 17
};
enum : uint32_t { CAT_ID = 0, CAT_BITENUM = 1, CAT_VALUEENUM = 2, CAT_LITERAL = 3, CAT_COMPOSITE = 4 };
enum : uint32_t { LIT_PLAIN = 0, LIT_STRING = 1, LIT_CTXNUM = 2, LIT_INTEGER = 3, LIT_EXTINST = 4, LIT_SPECOP = 5 };
enum : uint32_t { IDR_ID = 0, IDR_RESULT = 1, IDR_RESULT_TYPE = 2 };
enum : uint32_t { Q_ONE = 0, Q_OPT = 1, Q_VAR = 2 };
constexpr uint32_t SECTION_KEEP = 255;

struct Tables {
  const uint32_t* blob;
  uint32_t n_inst, max_opcode, n_kind, n_enum, n_slot, n_req, n_cap, cap_words, n_vsort;
  int32_t ext_max;
  uint32_t idref, linkage, ocl_off, ocl_len, req_stride, cap_kind;
  uint32_t width_req[5];
  uint32_t str_bytes;
  const uint32_t* inst;     // 8 words / instruction
  const uint16_t* opidx;    // max_opcode+1 entries
  const uint32_t* kind;     // 8 words / kind
  const uint32_t* enm;      // 8 words / enumerant
  const uint32_t* slot;     // kind | quant<<16 | spec_tail<<24
  const uint8_t* str;
  const uint32_t* req;      // req_stride words / requirement
  const uint64_t* closure;  // cap_words u64 / capability name
  const uint32_t* vsort;    // (value, enum index) pairs
  const uint32_t* ext;      // (name_off, name_len) per ext number

  // -- instructions ----------------------------------------------------------
  __device__ __forceinline__ uint32_t inst_of(uint32_t opcode) const {
    if (opcode > max_opcode) return NONE32;
    uint16_t v = __ldg(opidx + opcode);
    return v == NONE16 ? NONE32 : v;
  }
  __device__ __forceinline__ const uint32_t* irec(uint32_t i) const { return inst + 8 * i; }
  __device__ __forceinline__ uint32_t iname_off(uint32_t i) const { return __ldg(irec(i)); }
  __device__ __forceinline__ uint32_t iname_len(uint32_t i) const { return __ldg(irec(i) + 1) & 0xFFFF; }
  __device__ __forceinline__ uint32_t inslots(uint32_t i) const { return __ldg(irec(i) + 1) >> 16; }
  __device__ __forceinline__ uint32_t islot_off(uint32_t i) const { return __ldg(irec(i) + 2); }
  __device__ __forceinline__ uint32_t iflags(uint32_t i) const { return __ldg(irec(i) + 3); }
  __device__ __forceinline__ bool has_result(uint32_t i) const { return iflags(i) & 1; }
  __device__ __forceinline__ bool has_rtype(uint32_t i) const { return iflags(i) & 2; }
  __device__ __forceinline__ uint32_t special(uint32_t i) const { return (iflags(i) >> 8) & 0xFF; }
  __device__ __forceinline__ uint32_t section(uint32_t i) const { return (iflags(i) >> 16) & 0xFF; }
  __device__ __forceinline__ uint32_t ireq(uint32_t i) const { return __ldg(irec(i) + 4); }
  // some operand kind of the instruction can carry a capability requirement (tables.py)
  __device__ __forceinline__ bool ireqops(uint32_t i) const { return __ldg(irec(i) + 6) & 1; }

  // -- kinds -----------------------------------------------------------------
  __device__ __forceinline__ const uint32_t* krec(uint32_t k) const { return kind + 8 * k; }
  __device__ __forceinline__ uint32_t kcat(uint32_t k) const { return __ldg(krec(k)) & 0xFF; }
  __device__ __forceinline__ uint32_t ksub(uint32_t k) const { return (__ldg(krec(k)) >> 8) & 0xFF; }
  __device__ __forceinline__ uint32_t knbases(uint32_t k) const { return __ldg(krec(k)) >> 16; }
  __device__ __forceinline__ uint32_t kenum_off(uint32_t k) const { return __ldg(krec(k) + 1); }
  __device__ __forceinline__ uint32_t knenum(uint32_t k) const { return __ldg(krec(k) + 2); }
  __device__ __forceinline__ uint32_t kzero(uint32_t k) const { return __ldg(krec(k) + 3); }
  __device__ __forceinline__ uint32_t kbase_off(uint32_t k) const { return __ldg(krec(k) + 4); }
  __device__ __forceinline__ uint32_t kvs_off(uint32_t k) const { return __ldg(krec(k) + 5); }
  __device__ __forceinline__ uint32_t kvs_n(uint32_t k) const { return __ldg(krec(k) + 6); }

  // -- enumerants ----------------------------------------------------------------
  __device__ __forceinline__ const uint32_t* erec(uint32_t e) const { return enm + 8 * e; }
  __device__ __forceinline__ uint32_t evalue(uint32_t e) const { return __ldg(erec(e)); }
  __device__ __forceinline__ uint32_t ename_off(uint32_t e) const { return __ldg(erec(e) + 1); }
  __device__ __forceinline__ uint32_t ename_len(uint32_t e) const { return __ldg(erec(e) + 2) & 0xFFFF; }
  __device__ __forceinline__ uint32_t enparams(uint32_t e) const { return __ldg(erec(e) + 2) >> 16; }
  __device__ __forceinline__ uint32_t eparam_off(uint32_t e) const { return __ldg(erec(e) + 3); }
  __device__ __forceinline__ uint32_t ereq(uint32_t e) const { return __ldg(erec(e) + 4); }
  __device__ __forceinline__ uint32_t emerged(uint32_t e) const { return __ldg(erec(e) + 5); }
  __device__ __forceinline__ uint32_t ecapname(uint32_t e) const { return __ldg(erec(e) + 6); }

  // first enumerant of a ValueEnum kind with this value (ops.py:385-390)
  __device__ uint32_t venum_lookup(uint32_t k, uint32_t value) const {
    uint32_t lo = kvs_off(k), n = kvs_n(k);
    uint32_t hi = lo + n;
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      uint32_t v = __ldg(vsort + 2 * mid);
      if (v < value) lo = mid + 1; else hi = mid;
    }
    if (lo < kvs_off(k) + n && __ldg(vsort + 2 * lo) == value) return __ldg(vsort + 2 * lo + 1);
    return NONE32;
  }

  __device__ __forceinline__ uint32_t slot_kind(uint32_t s) const { return __ldg(slot + s) & 0xFFFF; }
  __device__ __forceinline__ uint32_t slot_quant(uint32_t s) const { return (__ldg(slot + s) >> 16) & 0xFF; }
  __device__ __forceinline__ bool slot_spec_tail(uint32_t s) const { return (__ldg(slot + s) >> 24) & 1; }

  // -- requirements / capabilities ---------------------------------------------
  __device__ __forceinline__ const uint32_t* rrec(uint32_t r) const { return req + req_stride * r; }

  // -- ext instructions -------------------------------------------------------
  __device__ __forceinline__ bool ext_name(uint32_t num, uint32_t& off, uint32_t& len) const {
    if (ext_max < 0 || num > (uint32_t)ext_max) return false;
    off = __ldg(ext + 2 * num);
    if (off == NONE32) return false;
    len = __ldg(ext + 2 * num + 1);
    return true;
  }
};

}  // namespace skg
