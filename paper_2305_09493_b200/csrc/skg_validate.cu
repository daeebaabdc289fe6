// Batch validator: binary modules -> diagnostics, bit-exact with the reference
// validate_module (validate.py:73-296).  Output per module is the
// diagnostics_text rendering, one "severity code location message" line per
// diagnostic, each terminated by '\n', in validate_module's order:
// module-level shape findings, then per instruction index i:
//   DuplicateResultId, BoundTooSmall*      (_check_ids, validate.py:139-168)
//   UnknownOpcode | OperandMismatch        (_check_operand_layout, :207-220)
//   MissingCapability (instruction, operands*, width)  (_closure_diagnostics, :237-267)
// Non-codec exceptions raised by the operand walk escape validate_module in the
// reference; they are reported as the module status like the disassembler does.
#include "skg_module.cuh"

namespace skg {

struct ValidateArgs {
  Tables T;
  const uint8_t* data;
  const int64_t* mod_off;
  const int64_t* mod_len;
  uint32_t n_mod;
  uint8_t* text;
  uint64_t text_cap;
  int64_t* text_span;
  int32_t* status;
  uint32_t* ticket;
  ErrRec* errs;
  uint32_t err_cap;
  uint8_t* gscratch;
  uint64_t gslot_bytes;
  uint32_t smem_slab;
  const uint32_t* order;      // ticket -> module index (skg_sched.cuh)
  uint32_t group_warps;       // warps per phase-barrier group
};

constexpr int MAX_CAPW = 6;

template <class S>
__device__ inline void diag_head(S& s, bool error, const char* code, uint32_t loc) {
  put_cstr(s, error ? "error " : "warning ");
  put_cstr(s, code);
  s.put(' ');
  if (loc == NONE32) put_cstr(s, "module"); else put_u64(s, loc);
  s.put(' ');
}

__device__ inline bool unsatisfied(const Tables& T, uint32_t r, const uint64_t* eff) {
  if (r == NONE32) return false;
  const uint32_t* rec = T.rrec(r);
  for (uint32_t k = 0; k < T.cap_words; ++k) {
    uint64_t bits = (uint64_t)__ldg(rec + 2 + 2 * k) | ((uint64_t)__ldg(rec + 3 + 2 * k) << 32);
    if (bits & eff[k]) return false;
  }
  return true;
}

template <class S>
__device__ inline void put_req_repr(S& s, const Tables& T, uint32_t r) {
  const uint32_t* rec = T.rrec(r);
  s.putn(T.str + __ldg(rec), __ldg(rec + 1));
}



template <class S>
struct BoundVis : NullVis {
  S* s;
  uint32_t i, bound;
  __device__ __noinline__ void id(uint32_t, uint32_t v, int, uint32_t) {
    if (v >= bound) {
      diag_head(*s, true, "BoundTooSmall", i);
      s->put('%'); put_u64(*s, v); put_cstr(*s, " is not below the header bound "); put_u64(*s, bound);
      s->put('\n');
    }
  }
};

template <class S>
struct ReqVis : NullVis {
  S* s;
  const Tables* T;
  const uint64_t* eff;
  uint32_t i, d;
  __device__ __noinline__ void line(uint32_t r) {
    diag_head(*s, true, "MissingCapability", i);
    s->putn(T->str + T->iname_off(d), T->iname_len(d));
    put_cstr(*s, " operand requires one of ");
    put_req_repr(*s, *T, r);
    s->put('\n');
  }
  __device__ __noinline__ void venum(uint32_t, uint32_t, uint32_t e, uint32_t) {
    if (e == NONE32) return;
    uint32_t r = T->emerged(e);
    if (unsatisfied(*T, r, eff)) line(r);
  }
  __device__ __noinline__ void benum(uint32_t k, uint32_t mask, bool full, uint64_t comp, uint32_t) {
    if (!full) return;
    uint32_t eo = T->kenum_off(k);
    for (uint64_t rest = comp; rest; rest &= rest - 1) {
      const int j = __ffsll((long long)rest) - 1;
      uint32_t r = T->ereq(eo + j);
      if (unsatisfied(*T, r, eff)) line(r);
    }
  }
};

// inst_diags shortcuts (fused pass): the walk status is already in m.ierr (the
// disassembler's classification walk), no id operand reaches the header bound
enum : uint32_t { VF_IERR_KNOWN = 1, VF_NO_BIG_IDS = 2 };

// all located diagnostics of instruction i; returns the walk status
template <class S>
__device__ __noinline__ WalkErr inst_diags(S& s, const Mod& m, const Tables& T, uint32_t i,
                                     const uint64_t* eff, uint32_t fast = 0) {
  const uint32_t d = m.idef[i];
  const uint32_t* ops = inst_ops(m, i);
  const uint32_t n = inst_nops(m, i);
  if (d == NONE16) {
    diag_head(s, false, "UnknownOpcode", i);
    put_cstr(s, "opcode "); put_u64(s, inst_opcode(m, i)); put_cstr(s, " is not in the loaded grammar\n");
    return WalkErr{};
  }
  if (T.has_result(d)) {
    uint32_t idx = T.has_rtype(d) ? 1 : 0;
    if (idx < n) {
      uint32_t slot = ht_find(m, ops[idx]);
      if (slot != NONE32 && m.hdef[slot] != i) {
        diag_head(s, true, "DuplicateResultId", i);
        s.put('%'); put_u64(s, ops[idx]); put_cstr(s, " already defined at instruction ");
        put_u64(s, m.hdef[slot]); s.put('\n');
      }
    }
  }
  Resolver res{&m, &T};
  NullVis nv;
  WalkErr e{};
  if (!(fast & VF_IERR_KNOWN) || m.ierr[i] != W_OK) e = walk(T, d, ops, n, nv, res);
  if (e.code != W_OK && !werr_is_codec(e.code)) return e;
  if (e.code == W_OK) {
    if (!(fast & VF_NO_BIG_IDS)) {
      BoundVis<S> bv;
      bv.s = &s; bv.i = i; bv.bound = m.bound;
      walk(T, d, ops, n, bv, res);
    }
  } else {
    diag_head(s, true, "OperandMismatch", i);
    put_walk_error(s, T, d, e);
    s.put('\n');
  }
  const uint32_t sp = T.special(d);
  if (sp == SP_CAPABILITY) return e;
  uint32_t r = T.ireq(d);
  if (unsatisfied(T, r, eff)) {
    diag_head(s, true, "MissingCapability", i);
    s.putn(T.str + T.iname_off(d), T.iname_len(d));
    put_cstr(s, " requires one of ");
    put_req_repr(s, T, r);
    s.put('\n');
  }
  if (e.code != W_OK) return e;
  if (T.ireqops(d)) {
    ReqVis<S> rv;
    rv.s = &s; rv.T = &T; rv.eff = eff; rv.i = i; rv.d = d;
    walk(T, d, ops, n, rv, res);
  }
  uint32_t wr = NONE32;
  if ((sp == SP_TYPEINT || sp == SP_TYPEFLOAT) && n >= 2) {
    uint32_t wd = ops[1];
    if (sp == SP_TYPEINT) wr = wd == 8 ? T.width_req[0] : wd == 16 ? T.width_req[1] : wd == 64 ? T.width_req[2] : NONE32;
    else wr = wd == 16 ? T.width_req[3] : wd == 64 ? T.width_req[4] : NONE32;
  }
  if (unsatisfied(T, wr, eff)) {
    diag_head(s, true, "MissingCapability", i);
    s.putn(T.str + T.iname_off(d), T.iname_len(d));
    put_cstr(s, " with this width requires one of ");
    put_req_repr(s, T, wr);
    s.put('\n');
  }
  return e;
}

struct Shape {
  bool has_fn, has_cap, has_ep;
  uint32_t n_mm;
  bool linkage;
};

template <class S>
__device__ __noinline__ void shape_diags(S& s, const Shape& sh) {
  if (!sh.has_fn) { diag_head(s, true, "MissingFunction", NONE32); put_cstr(s, "module declares no function\n"); }
  if (!sh.has_cap) { diag_head(s, true, "MissingCapability", NONE32); put_cstr(s, "module declares no capability\n"); }
  if (sh.n_mm == 0) { diag_head(s, true, "MissingMemoryModel", NONE32); put_cstr(s, "module has no memory model\n"); }
  else if (sh.n_mm > 1) {
    diag_head(s, true, "MultipleMemoryModels", NONE32);
    put_cstr(s, "module has "); put_u64(s, sh.n_mm); put_cstr(s, " memory model instructions\n");
  }
  if (!sh.has_ep) {
    diag_head(s, !sh.linkage, "MissingEntryPoint", NONE32);
    put_cstr(s, "module declares no entry point\n");
  }
}

// the validator's single diagnostic for a module that does not decode (validate.py:76-83):
// its code and the decode error's message, identical to load_and_split's
__device__ inline const char* decode_code(int32_t decode_status) {
  return decode_status == ST_NOTSPIRV ? "NotSpirv" : decode_status == ST_TRUNCATED ? "TruncatedStream"
                                                                                  : "CorruptStream";
}

template <class S>
__device__ __noinline__ void put_decode_msg(S& ew, const Mod& m, int64_t nbytes, int32_t decode_status) {
  if (nbytes % 4 != 0 || nbytes < 20) {
    put_u64(ew, (uint64_t)nbytes); put_cstr(ew, " bytes is not a whole word stream of at least 5 words");
  } else if (decode_status == ST_NOTSPIRV) {
    put_cstr(ew, "magic word 0x"); put_hex8_upper(ew, m.w[0]); put_cstr(ew, " is not SPIR-V");
  } else {
    uint32_t p = 5;   // re-walk to the failing position
    while (p < m.W) {
      uint32_t wc = m.w[p] >> 16;
      if (wc == 0 || p + wc > m.W) break;
      p += wc;
    }
    put_cstr(ew, "instruction at word "); put_u64(ew, p);
    put_cstr(ew, decode_status == ST_CORRUPT ? " has word count 0" : " runs past the end of the stream");
  }
}

// V2 (warp), in three parts: module shape + effective capabilities
// (validate.py:101-136); the per-instruction diagnostic sizes (one grammar walk per
// instruction: per warp here, or across the CTA's modules in val_walk_cta); then
// the first escaping exception (status, error record) and the per-instruction
// offsets in m.ia.  val_sizes returns the module's diagnostics bytes.
__device__ __noinline__ void val_shape(const Mod& m, const Tables& T, uint64_t* eff, Shape& sh) {
  const uint32_t lane = lane_id();
  bool fn = false, cap = false, ep = false;
  uint32_t mm = 0;
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane;
    if (i >= m.I || m.idef[i] == NONE16) continue;
    uint32_t sp = T.special(m.idef[i]);
    fn |= sp == SP_FUNCTION;
    ep |= sp == SP_ENTRYPOINT;
    mm += sp == SP_MEMORYMODEL;
    if (sp == SP_CAPABILITY) {
      cap = true;
      if (inst_nops(m, i) >= 1 && T.cap_kind != NONE32) {
        uint32_t e = T.venum_lookup(T.cap_kind, inst_ops(m, i)[0]);
        uint32_t cn = e == NONE32 ? NONE32 : T.ecapname(e);
        if (cn != NONE32)
          for (uint32_t k = 0; k < T.cap_words && k < MAX_CAPW; ++k) eff[k] |= __ldg(T.closure + cn * T.cap_words + k);
      }
    }
  }
  sh.has_fn = __any_sync(FULL, fn);
  sh.has_cap = __any_sync(FULL, cap);
  sh.has_ep = __any_sync(FULL, ep);
  sh.n_mm = warp_sum_u32(mm);
  for (int k = 0; k < MAX_CAPW; ++k) {
#pragma unroll
    for (int dd = 16; dd > 0; dd >>= 1) eff[k] |= __shfl_xor_sync(FULL, eff[k], dd);
  }
  sh.linkage = T.linkage != NONE32 && ((eff[T.linkage / 64] >> (T.linkage % 64)) & 1);
}

__device__ __forceinline__ void val_walk_one(Mod& m, const Tables& T, uint32_t i, const uint64_t* eff, uint32_t fast) {
  CountSink cs;
  WalkErr e = inst_diags(cs, m, T, i, eff, fast);
  m.ierr[i] = (uint8_t)e.code;
  m.ia[i] = cs.n;
}

__device__ __noinline__ uint64_t val_finish(Mod& m, const Tables& T, const uint64_t* eff, const Shape& sh,
                                            int32_t& status, ErrSink& es, int32_t t) {
  const uint32_t lane = lane_id();
  uint32_t bad = NONE32;
  for (uint32_t base = 0; base < m.I && bad == NONE32; base += 32) {
    uint32_t i = base + lane;
    unsigned b = __ballot_sync(FULL, i < m.I && m.ierr[i] != W_OK && !werr_is_codec(m.ierr[i]));
    if (b) bad = base + __ffs(b) - 1;
  }
  if (bad != NONE32) {
    if (lane == 0) {
      ErrRec* rec = es.alloc();
      CountSink cs;
      WalkErr e = inst_diags(cs, m, T, bad, eff);
      status = walk_status(e.code);
      if (rec) {
        ErrWriter ew{rec};
        put_walk_error(ew, T, m.idef[bad], e);
        rec->module = t; rec->cls = status; rec->len = ew.n;
        rec->a = e.a; rec->b = e.b; rec->c = e.c; rec->d = e.d;
      }
    }
    status = __shfl_sync(FULL, status, 0);
    return 0;
  }
  CountSink hs;
  shape_diags(hs, sh);
  uint64_t run = hs.n;
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane;
    uint32_t len = i < m.I ? m.ia[i] : 0;
    uint32_t incl = warp_incl_sum(len);
    if (i < m.I) m.ia[i] = (uint32_t)(run + incl - len);
    run += __shfl_sync(FULL, incl, 31);
  }
  __syncwarp();
  return run;
}

__device__ __noinline__ uint64_t val_sizes(Mod& m, const Tables& T, uint64_t* eff, Shape& sh, int32_t& status,
                                           ErrSink& es, int32_t t, uint32_t fast = 0) {
  val_shape(m, T, eff, sh);
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane_id();
    if (i < m.I) val_walk_one(m, T, i, eff, fast);
  }
  __syncwarp();
  return val_finish(m, T, eff, sh, status, es, t);
}

// The V2 walks or the V3 writes of all the CTA's modules (every warp calls it;
// `mine` = this warp's module takes part): instructions sorted by grammar entry
// (cta_dispatch; lists in each module's spill area), each walked with its own
// module's capabilities.  write == false: sizes (val_walk_one); write == true: the
// diagnostics text at out[module] + m.ia[i] (val_write's per-instruction part).
__device__ __noinline__ void val_walk_cta(Mod* all, const Tables& T, CtaSort& cs, const uint64_t (*effs)[MAX_CAPW],
                                          const uint32_t* fasts, uint8_t* const* outs, bool mine, bool write) {
  const uint32_t wib = threadIdx.x >> 5;
  Mod& m = all[wib];
  const uint32_t n = mine ? m.I : 0;
  uint32_t* in = reinterpret_cast<uint32_t*>(m.spill);
  uint32_t* out = in + n + 4;
  for (uint32_t i = lane_id(); i < n; i += 32) in[i] = (wib << 27) | i;
  cta_dispatch(cs, in, out, n, [&](uint32_t e) { return (uint32_t)m.idef[e & CTA_ITEM]; },
               [&](uint32_t e) {
                 const uint32_t mi = e >> 27, i = e & CTA_ITEM;
                 Mod& mm = all[mi];
                 if (write) {
                   MemSink ms(outs[mi] + mm.ia[i]);
                   inst_diags(ms, mm, T, i, effs[mi], fasts[mi]);
                 } else {
                   val_walk_one(mm, T, i, effs[mi], fasts[mi]);
                 }
               });
}

// V3 (warp): the diagnostics text at the offsets val_sizes left in m.ia
__device__ __noinline__ void val_write(uint8_t* out, const Mod& m, const Tables& T, const uint64_t* eff,
                                       const Shape& sh, uint32_t fast = 0) {
  if (lane_id() == 0) { MemSink ms(out); shape_diags(ms, sh); }
  for (uint32_t base = 0; base < m.I; base += 32) {
    uint32_t i = base + lane_id();
    if (i >= m.I) continue;
    MemSink ms(out + m.ia[i]);
    inst_diags(ms, m, T, i, eff, fast);
  }
}

// One module per warp; the CTA's warps run each phase together (CTA barrier
// between phases), like disasm_kernel.  Scratch in the per-warp global slot.
__device__ __noinline__ void validate_one(const ValidateArgs& a, uint32_t ticket, uint8_t* gslot, ErrSink& es,
                                          uint32_t gid, uint32_t gw, Mod& m, Mod* all, CtaSort& cs) {
  const uint32_t lane = lane_id();
  const Tables& T = a.T;
  const bool live = ticket < a.n_mod;
  const uint32_t t = live ? a.order[ticket] : 0;
  int32_t status = live ? ST_OK : ST_INTERNAL;
  int32_t decode_status = ST_OK;
  uint64_t total = 0;
  Shape sh{};
  uint64_t eff[MAX_CAPW] = {0, 0, 0, 0, 0, 0};
  int64_t nbytes = 0;
  // -- V0: load + boundary
  if (live) {
    nbytes = a.mod_len[t];
    const uint8_t* src = a.data + a.mod_off[t];
    const uint32_t W = (nbytes >= 0 && nbytes % 4 == 0) ? (uint32_t)(nbytes / 4) : 0;
    if (worst_bytes(W, 0) > a.gslot_bytes) {
      status = ST_INTERNAL;
      ErrRec* drec = nullptr;
      if (lane == 0 && (drec = es.alloc())) {
        ErrWriter ew{drec};
        put_cstr(ew, "internal: module exceeds the per-warp scratch slot");
        drec->module = (int32_t)t; drec->cls = ST_INTERNAL; drec->len = ew.n;
      }
    } else {
      layout_head(m, gslot, W);
      decode_status = load_and_split(m, src, (uint64_t)nbytes, nullptr, (int32_t)t);
    }
  }
  group_sync(gid, gw);
  // -- V1: id tables + prescan (hash tables when an id is at/above the bound)
  const bool go = status == ST_OK && decode_status == ST_OK;
  if (go) {
    bool in_smem = false;
    bool direct = m.bound <= 2 * m.W + 64;
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (!place_tables(m, direct, in_smem, gslot, a.gslot_bytes, 0, 0)) { status = ST_INTERNAL; break; }
      init_tables(m);
      prescan(m, T);
      if (*m.overflow && direct) { __syncwarp(); direct = false; continue; }
      break;
    }
  }
  group_sync(gid, gw);
  // -- V2: module shape + effective capabilities (validate.py:101-136), sizes,
  //        escaping exceptions, offsets
  // (the barrier group is the whole CTA: the per-instruction walks of V2 and V3 run
  //  across the CTA's modules, sorted by grammar entry -- val_walk_cta)
  __shared__ uint64_t s_veff[32][MAX_CAPW];
  __shared__ uint32_t s_vfast[32];
  __shared__ uint8_t* s_vout[32];
  const uint32_t wib = threadIdx.x >> 5;
  const bool vcross = gw == (blockDim.x >> 5);
  const bool vgo = go && status == ST_OK;
  if (vcross) {
    if (vgo) val_shape(m, T, eff, sh);
    if (lane == 0) {
      for (int k = 0; k < MAX_CAPW; ++k) s_veff[wib][k] = eff[k];
      s_vfast[wib] = 0;
    }
    val_walk_cta(all, T, cs, s_veff, s_vfast, nullptr, vgo, false);
    if (vgo) total = val_finish(m, T, eff, sh, status, es, (int32_t)t);
  } else if (vgo) {
    total = val_sizes(m, T, eff, sh, status, es, (int32_t)t);
  }
  group_sync(gid, gw);
  // -- V3: output
  bool vwrite = false;
  uint8_t* vout = nullptr;
  if (live && status == ST_OK && decode_status != ST_OK) {
    // the decode error of the module is its only diagnostic line
    const char* code = decode_code(decode_status);
    CountSink cs;
    diag_head(cs, true, code, NONE32);
    ErrRec tmp;
    {
      ErrWriter ew{&tmp};
      put_decode_msg(ew, m, nbytes, decode_status);
      tmp.len = ew.n;
    }
    total = cs.n + (uint32_t)tmp.len + 1;
    bool fits;
    uint64_t off = alloc_text(a.ticket, total, a.text_cap, fits);
    if (lane == 0) {
      a.text_span[2 * t] = (int64_t)off;
      a.text_span[2 * t + 1] = (int64_t)total;
      a.status[t] = ST_OK;
      if (fits) {
        MemSink ms(a.text + off);
        diag_head(ms, true, code, NONE32);
        ms.putn((const uint8_t*)tmp.msg, (uint32_t)tmp.len);
        ms.put('\n');
      }
    }
  } else if (live) {
    if (status != ST_OK) total = 0;
    bool fits;
    uint64_t off = alloc_text(a.ticket, total, a.text_cap, fits);
    if (lane == 0) {
      a.text_span[2 * t] = (int64_t)off;
      a.text_span[2 * t + 1] = (int64_t)total;
      a.status[t] = status;
    }
    vwrite = status == ST_OK && total > 0 && fits;
    vout = a.text + off;
  }
  if (vcross) {
    if (vwrite && lane == 0) { MemSink ms(vout); shape_diags(ms, sh); }
    if (lane == 0) s_vout[wib] = vout;
    val_walk_cta(all, T, cs, s_veff, s_vfast, s_vout, vwrite, true);
  } else if (vwrite) {
    val_write(vout, m, T, eff, sh);
  }
  __syncwarp();
  group_sync(gid, gw);
}

#ifndef SKG_VAL_MAXT
#define SKG_VAL_MAXT 1024
#endif
__global__ void __launch_bounds__(SKG_VAL_MAXT) validate_kernel(const __grid_constant__ ValidateArgs a) {
  __shared__ ValidateArgs s_args;   // one copy per CTA: field reads are shared loads
  if (threadIdx.x == 0) s_args = a;
  __syncthreads();
  __shared__ uint32_t s_base[16];
  __shared__ Mod s_mod[32];   // module descriptor, one per warp (not 32 per-thread local copies)
  __shared__ CtaSort s_cs;    // cross-module work assignment (V2 / V3 walks)
  const uint32_t warps = blockDim.x >> 5;
  const uint32_t warp_in_block = threadIdx.x >> 5;
  const uint32_t gw = a.group_warps;
  const uint32_t gid = warp_in_block / gw, gwarp_in = warp_in_block % gw;
  const uint32_t gwarp = blockIdx.x * warps + warp_in_block;
  uint8_t* gslot = a.gscratch + (size_t)gwarp * a.gslot_bytes;
  ErrSink es{a.errs, a.ticket + 1, a.err_cap};
  while (true) {
    if (gwarp_in == 0 && lane_id() == 0) s_base[gid] = atomicAdd(a.ticket, gw);
    group_sync(gid, gw);
    const uint32_t base = s_base[gid];
    group_sync(gid, gw);
    if (base >= a.n_mod) break;
    validate_one(s_args, base + gwarp_in, gslot, es, gid, gw, s_mod[warp_in_block], s_mod, s_cs);
  }
}

}  // namespace skg

// ---------------------------------------------------------------------------
// One large module over the whole GPU (skg_big.cuh): shape + effective
// capabilities, per-instruction diagnostic sizes, scan, write.
namespace skg {

__global__ void big_val_shape(const Mod* mp, Tables T, uint32_t* ctl) {
  const Mod m = *mp;
  unsigned long long* eff = reinterpret_cast<unsigned long long*>(ctl + BC_EFF);
  uint32_t fl = 0, mm = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m.I; i += gridDim.x * blockDim.x) {
    if (m.idef[i] == NONE16) continue;
    const uint32_t sp = T.special(m.idef[i]);
    fl |= sp == SP_FUNCTION ? BF_FN : 0;
    fl |= sp == SP_ENTRYPOINT ? BF_EP : 0;
    mm += sp == SP_MEMORYMODEL;
    if (sp == SP_CAPABILITY) {
      fl |= BF_CAP;
      if (inst_nops(m, i) >= 1 && T.cap_kind != NONE32) {
        const uint32_t e = T.venum_lookup(T.cap_kind, inst_ops(m, i)[0]);
        const uint32_t cn = e == NONE32 ? NONE32 : T.ecapname(e);
        if (cn != NONE32)
          for (uint32_t k = 0; k < T.cap_words && k < MAX_CAPW; ++k)
            atomicOr(eff + k, (unsigned long long)__ldg(T.closure + cn * T.cap_words + k));
      }
    }
  }
  if (fl) atomicOr(&ctl[BC_FLAGS], fl);
  if (mm) atomicAdd(&ctl[BC_NMM], mm);
}

__device__ inline Shape big_shape(const Tables& T, const uint32_t* ctl, uint64_t* eff) {
  const unsigned long long* e = reinterpret_cast<const unsigned long long*>(ctl + BC_EFF);
  for (int k = 0; k < MAX_CAPW; ++k) eff[k] = e[k];
  Shape sh;
  sh.has_fn = ctl[BC_FLAGS] & BF_FN;
  sh.has_cap = ctl[BC_FLAGS] & BF_CAP;
  sh.has_ep = ctl[BC_FLAGS] & BF_EP;
  sh.n_mm = ctl[BC_NMM];
  sh.linkage = T.linkage != NONE32 && ((eff[T.linkage / 64] >> (T.linkage % 64)) & 1);
  return sh;
}

__global__ void big_val_sizes(const Mod* mp, Tables T, uint32_t* ctl) {
  const Mod m = *mp;
  uint64_t eff[MAX_CAPW];
  const Shape sh = big_shape(T, ctl, eff);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    CountSink hs;
    shape_diags(hs, sh);
    ctl[BC_TOTAL] = hs.n;
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m.I; i += gridDim.x * blockDim.x) {
    CountSink cs;
    const WalkErr e = inst_diags(cs, m, T, i, eff);
    m.ia[i] = cs.n;
    m.ierr[i] = (uint8_t)e.code;
    if (e.code != W_OK && !werr_is_codec(e.code)) atomicMin(&ctl[BC_BAD], i);
  }
}

// the exception of the first instruction whose walk escapes (validate.py:88-94)
__global__ void big_val_error(const Mod* mp, Tables T, const uint32_t* ctl, ErrRec* rec, int32_t* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const Mod m = *mp;
  uint64_t eff[MAX_CAPW];
  big_shape(T, ctl, eff);
  const uint32_t bad = ctl[BC_BAD];
  CountSink cs;
  const WalkErr e = inst_diags(cs, m, T, bad, eff);
  *status = walk_status(e.code);
  if (rec) {
    ErrWriter ew{rec};
    put_walk_error(ew, T, m.idef[bad], e);
    rec->module = 0; rec->cls = *status; rec->len = ew.n;
    rec->a = e.a; rec->b = e.b; rec->c = e.c; rec->d = e.d;
  }
}

__global__ void big_val_write(const Mod* mp, Tables T, const uint32_t* ctl, uint8_t* out) {
  const Mod m = *mp;
  uint64_t eff[MAX_CAPW];
  const Shape sh = big_shape(T, ctl, eff);
  if (blockIdx.x == 0 && threadIdx.x == 0) { MemSink ms(out); shape_diags(ms, sh); }
  const uint32_t head = ctl[BC_TOTAL];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m.I; i += gridDim.x * blockDim.x) {
    MemSink ms(out + head + m.ia[i]);
    inst_diags(ms, m, T, i, eff);
  }
}

}  // namespace skg
