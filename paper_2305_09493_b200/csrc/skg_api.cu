// C-ABI entry points of libskgpu (include/skgpu.h).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <cub/device/device_radix_sort.cuh>
#ifdef W_OK   // <unistd.h> access() mode (via CUB): the walk status enum uses the name
#undef W_OK
#endif
#include "../../include/skgpu.h"
#include "skg_module.cuh"
#include "skg_sched.cuh"
#include "skg_bigdecode.cuh"
#include "skg_big.cuh"
#include "skg_codec.cuh"

namespace skg {
struct DisasmArgs;
struct ValidateArgs;
struct DecodeArgs;
}

#include "skg_validate.cu"
#include "skg_disasm.cu"
#include "skg_decode.cu"
#include "skg_asm.cu"

struct skg_tables {
  skg::Tables t;
  skg::Uni u;
  skg::AsmTables a;
  uint32_t* d_blob;
};

namespace {


int g_sms[64] = {};

int sm_count() {
  int dev = 0;
  cudaGetDevice(&dev);
  int& n = g_sms[dev & 63];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// true the first time it is called for the current device (function attributes are
// per device)
bool first_on_device(uint64_t& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done & bit) return false;
  done |= bit;
  return true;
}

uint64_t gslot_bytes(uint32_t max_words) {
  return (skg::worst_bytes(max_words, skg::RENDER_MIN) + 255) & ~(uint64_t)255;
}


struct WsLayout {
  uint64_t state, counters, sched, scratch, total, slot, gtext;
  uint32_t n_warps;
};

// scheduling region: hist[1024], cursor[1024], perm[n]
uint64_t sched_bytes(uint32_t n_mod) { return (skg::SCHED_PERM_OFF + 4ull * n_mod + 255) & ~255ull; }

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// module processing order (largest first; region-major for big batches of modules
// in caller order, see skg_sched.cuh) into sched + SCHED_PERM_OFF
uint32_t sched_regions(uint32_t n) {
  const int want = env_int("SKG_SCHED_REGIONS", -1);         // experiments: fixed count
  uint32_t r = want > 0 ? (uint32_t)want : std::min<uint32_t>(16, n / 50000);
  uint32_t p = 1;
  while (p * 2 <= r && p * 2 <= 16) p *= 2;                  // a power of two <= 16
  return p;
}

int launch_sched(const int64_t* len, uint32_t stride, uint32_t n, uint8_t* sched, cudaStream_t s,
                 bool regions = false, uint32_t shift = skg::SCHED_SHIFT) {
  uint32_t* hist = reinterpret_cast<uint32_t*>(sched);
  uint32_t* cursor = hist + skg::SCHED_BUCKETS;
  uint32_t* perm = cursor + skg::SCHED_BUCKETS;
  if (n <= 1)   // one module (single-module calls): the order is [0], no sort kernels
    return n ? (int)cudaMemsetAsync(perm, 0, 4, s) : 0;
  if (cudaError_t e = cudaMemsetAsync(hist, 0, 4 * skg::SCHED_BUCKETS, s)) return (int)e;
  uint32_t blocks = (n + 4095) / 4096;
  if (blocks > (uint32_t)sm_count() * 2) blocks = (uint32_t)sm_count() * 2;
  if (blocks == 0) blocks = 1;
  const skg::SchedKey key{regions ? sched_regions(n) : 1u, n, shift};   // size classes of 2^shift units
  skg::sched_hist<<<blocks, 1024, 0, s>>>(len, stride, n, hist, key);
  skg::sched_scan<<<1, 1024, 0, s>>>(hist, cursor);
  skg::sched_scatter<<<blocks, 1024, 0, s>>>(len, stride, n, cursor, perm, key);
  return (int)cudaGetLastError();
}


// disassembler: phase-synchronised CTAs of kDisWarps warps (one module per warp),
// one CTA per SM, kDisSlab bytes of shared memory per warp
int kDisWarps = env_int("SKG_DIS_WARPS", 32);
uint32_t kDisStage = (uint32_t)env_int("SKG_DIS_STAGE", 1024);
// module slab in shared memory (default 0: all module scratch in the per-warp
// global slot -- measured faster, the L1 that the carve-out leaves caches it)
uint32_t kDisSlab = (uint32_t)env_int("SKG_DIS_SLAB", 0);
uint32_t dis_blocks() {
  const int g = env_int("SKG_DIS_GRID", 0);   // experiments: explicit grid
  return g > 0 ? (uint32_t)g : (uint32_t)sm_count() * env_int("SKG_DIS_BLOCKS_PER_SM", 1);
}

// warps per named-barrier group: a divisor of the CTA's warps, at most 15 groups
uint32_t group_warps(int warps, int want) {
  int g = want < 1 ? 1 : (want > warps ? warps : want);
  while (warps % g || warps / g > 15) ++g;
  return (uint32_t)g;
}

// Launch geometry: the persistent grid, shrunk for batches with fewer modules
// than resident warps (a single huge module gets one warp and one scratch slot).
struct Geom { uint32_t blocks, warps; };
Geom fit_geom(uint32_t blocks, uint32_t warps, uint32_t n_mod, bool shrink_warps) {
  if ((uint64_t)blocks * warps > n_mod) {
    blocks = n_mod ? (n_mod + warps - 1) / warps : 1;
    if (blocks == 1 && shrink_warps) warps = n_mod ? (n_mod < warps ? n_mod : warps) : 1;
  }
  return {blocks, warps};
}
Geom dis_geom(uint32_t n_mod) { return fit_geom(dis_blocks(), (uint32_t)kDisWarps, n_mod, true); }
Geom val_geom(uint32_t n_mod) { return fit_geom(dis_blocks(), (uint32_t)kDisWarps, n_mod, true); }

// the fused validator's counters (error records, overflow, cursor) inside the
// 256-byte counter block, after the disassembler's
constexpr uint32_t kValCounters = 128;

WsLayout ws_layout(uint32_t n_mod, uint32_t max_words) {
  WsLayout l;
  (void)n_mod;
  const Geom gv = val_geom(n_mod), gd = dis_geom(n_mod);
  l.n_warps = gv.blocks * gv.warps;
  if (gd.blocks * gd.warps > l.n_warps) l.n_warps = gd.blocks * gd.warps;
  l.slot = gslot_bytes(max_words);
  l.counters = 0;
  l.state = 0;
  l.sched = 256;
  l.scratch = l.sched + sched_bytes(n_mod);
  l.gtext = 0;
  l.total = l.scratch + l.slot * l.n_warps;
  return l;
}

int check(cudaError_t e) {
  if (e != cudaSuccess) {
    fprintf(stderr, "skgpu: CUDA error %s\n", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

}  // namespace

namespace skg {
// device -> mapped pinned host words (skg_store_counters)
__global__ void store_words_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
}
// device -> mapped pinned host bytes by SM stores (skg_copy_to_host): 16-byte
// loads and stores, a grid-stride loop over 16-byte blocks, the tail by bytes
__global__ void __launch_bounds__(256) copy_to_host_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                                           uint64_t n) {
  const uint64_t nb = n >> 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nb; k += stride)
    reinterpret_cast<uint4*>(dst)[k] = __ldcs(reinterpret_cast<const uint4*>(src) + k);
  if (blockIdx.x == 0)
    for (uint64_t i = (nb << 4) + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
}
}  // namespace skg

extern "C" {

const char* skg_version(void) { return "skgpu 0.1 (sm_100a)"; }

#ifdef SKG_PHASE_TIMING
int skg_debug_disasm_phases(unsigned long long* out16) {
  return check(cudaMemcpyFromSymbol(out16, skg::g_dis_phase, 16 * sizeof(unsigned long long)));
}
int skg_debug_asm_phases(unsigned long long* out16) {
  return check(cudaMemcpyFromSymbol(out16, skg::g_asm_phase, 16 * sizeof(unsigned long long)));
}
#endif

int skg_tables_create(const uint32_t* host_blob, uint64_t n_words, skg_tables** out) {
  if (!host_blob || n_words < 64 || !out) return -1;
  if (host_blob[0] != 0x54474B53u) return -2;
  skg_tables* t = new skg_tables();
  if (int e = check(cudaMalloc(&t->d_blob, n_words * 4))) { delete t; return e; }
  if (int e = check(cudaMemcpy(t->d_blob, host_blob, n_words * 4, cudaMemcpyHostToDevice))) {
    cudaFree(t->d_blob); delete t; return e;
  }
  const uint32_t* h = host_blob;
  skg::Tables& T = t->t;
  const uint32_t* b = t->d_blob;
  T.blob = b;
  T.n_inst = h[2]; T.inst = b + h[3];
  T.max_opcode = h[4]; T.opidx = reinterpret_cast<const uint16_t*>(b + h[5]);
  T.n_kind = h[6]; T.kind = b + h[7];
  T.n_enum = h[8]; T.enm = b + h[9];
  T.n_slot = h[10]; T.slot = b + h[11];
  T.str = reinterpret_cast<const uint8_t*>(b + h[12]); T.str_bytes = h[13];
  T.n_req = h[14]; T.req = b + h[15];
  T.n_cap = h[16]; T.cap_words = h[17];
  T.closure = reinterpret_cast<const uint64_t*>(b + h[18]);
  T.vsort = b + h[19]; T.n_vsort = h[20];
  T.ext_max = (int32_t)h[21]; T.ext = b + h[22];
  T.idref = h[23];
  for (int j = 0; j < 5; ++j) T.width_req[j] = h[24 + j];
  T.linkage = h[29];
  T.ocl_off = h[30]; T.ocl_len = h[31];
  T.req_stride = h[32];
  T.cap_kind = h[33];
  skg::AsmTables& A = t->a;
  A.info = b + h[34];
  A.ophash = b + h[35]; A.ophash_cap = h[36];
  A.enhash = b + h[37]; A.enhash_cap = h[38];
  A.exhash = b + h[39]; A.exhash_cap = h[40];
  A.storage_fn = h[49]; A.op_label = h[50]; A.op_fnend = h[51];
  A.op_typeint = h[53]; A.op_typefloat = h[54];
  t->u = skg::Uni{b + h[41], h[42], b + h[43], h[44], b + h[45], h[46], b + h[47], h[48]};
  *out = t;
  return 0;
}

void skg_tables_destroy(skg_tables* t) {
  if (!t) return;
  cudaFree(t->d_blob);
  delete t;
}

uint64_t skg_workspace_bytes(uint32_t n_mod, uint32_t max_words) {
  return ws_layout(n_mod, max_words).total;
}

int skg_store_counters(void* host_dst, const void* dev_src, uint32_t n_words, void* stream) {
  if (!host_dst || !dev_src || n_words == 0 || n_words > 1024) return -1;
  void* dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, host_dst, 0) != cudaSuccess || !dptr) {
    cudaGetLastError();   // not mapped: a plain async copy
    return check(cudaMemcpyAsync(host_dst, dev_src, 4ull * n_words, cudaMemcpyDeviceToHost,
                                 static_cast<cudaStream_t>(stream)));
  }
  skg::store_words_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint32_t*>(dptr), static_cast<const uint32_t*>(dev_src), n_words);
  return check(cudaGetLastError());
}

int skg_copy_to_host(void* host_dst, const void* dev_src, uint64_t n_bytes, uint32_t n_ctas, void* stream) {
  if (!host_dst || !dev_src) return -1;
  if (n_bytes == 0) return 0;
  void* dptr = nullptr;
  if ((reinterpret_cast<uintptr_t>(host_dst) | reinterpret_cast<uintptr_t>(dev_src)) & 15 ||
      cudaHostGetDevicePointer(&dptr, host_dst, 0) != cudaSuccess || !dptr) {
    cudaGetLastError();   // not mapped / not aligned: a plain async copy
    return check(cudaMemcpyAsync(host_dst, dev_src, n_bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
  }
  const uint32_t g = n_ctas ? n_ctas : 64;
  skg::copy_to_host_kernel<<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint8_t*>(dptr), static_cast<const uint8_t*>(dev_src), n_bytes);
  return check(cudaGetLastError());
}

int skg_last_counts(const void* workspace, uint32_t* n_errors, uint32_t* text_overflow,
                    uint64_t* text_bytes, void* stream) {
  uint32_t c[6];
  cudaStream_t s = (cudaStream_t)stream;
  if (int e = check(cudaMemcpyAsync(c, workspace, 24, cudaMemcpyDeviceToHost, s))) return e;
  if (int e = check(cudaStreamSynchronize(s))) return e;
  if (n_errors) *n_errors = c[1];
  if (text_overflow) *text_overflow = c[2];
  if (text_bytes) *text_bytes = (uint64_t)c[4] | ((uint64_t)c[5] << 32);
  return 0;
}

int skg_disasm(const skg_tables* t, const uint8_t* data, const int64_t* mod_off,
               const int64_t* mod_len, uint32_t n_mod, uint32_t opts, uint32_t max_words,
               uint8_t* text, uint64_t text_cap, int64_t* text_span, int32_t* status,
               skg_error* errors, uint32_t err_cap, void* workspace, uint64_t workspace_bytes,
               void* stream) {
  return skg_disasm_refs(t, data, mod_off, mod_len, n_mod, opts, max_words, text, text_cap, text_span, status,
                         errors, err_cap, workspace, workspace_bytes, stream, nullptr, nullptr, 0);
}

namespace {
struct ValOut {   // the fused validator's outputs (skg_disasm_validate)
  uint8_t* text; uint64_t cap; int64_t* span; int32_t* status; skg_error* errors; uint32_t err_cap;
};

int disasm_launch(const skg_tables* t, const uint8_t* data, const int64_t* mod_off, const int64_t* mod_len,
                  uint32_t n_mod, uint32_t opts, uint32_t max_words, uint8_t* text, uint64_t text_cap,
                  int64_t* text_span, int32_t* status, skg_error* errors, uint32_t err_cap, void* workspace,
                  uint64_t workspace_bytes, void* stream, const uint32_t* ref_ids, const uint8_t* ref_text,
                  uint32_t n_refs, const ValOut* vo) {
  if (!t || !workspace || (n_refs && (!ref_ids || !ref_text))) return -1;
  if (vo && (!vo->span || !vo->status || !vo->text)) return -1;
  WsLayout l = ws_layout(n_mod, max_words);
  if (workspace_bytes < l.total) return -3;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* ws = (uint8_t*)workspace;
  if (int e = check(cudaMemsetAsync(ws, 0, l.scratch, s))) return e;
  if (n_mod == 0) return 0;
  skg::DisasmArgs a;
  a.T = t->t;
  a.data = data; a.mod_off = mod_off; a.mod_len = mod_len; a.n_mod = n_mod; a.opts = opts;
  a.text = text; a.text_cap = text_cap; a.text_span = text_span; a.status = status;
  a.ticket = reinterpret_cast<uint32_t*>(ws + l.counters);
  a.errs = reinterpret_cast<skg::ErrRec*>(errors);
  a.err_cap = err_cap;
  a.gscratch = ws + l.scratch;
  a.gslot_bytes = l.slot;
  a.smem_slab = kDisSlab;
  a.ovr = ref_ids; a.ovr_text = ref_text; a.n_ovr = n_refs;
  a.vtext = vo ? vo->text : nullptr; a.vtext_cap = vo ? vo->cap : 0;
  a.vspan = vo ? vo->span : nullptr; a.vstatus = vo ? vo->status : nullptr;
  a.vctr = reinterpret_cast<uint32_t*>(ws + l.counters + kValCounters);
  a.verrs = reinterpret_cast<skg::ErrRec*>(vo ? vo->errors : nullptr);
  a.verr_cap = vo ? vo->err_cap : 0;
  if (int e = check((cudaError_t)launch_sched(mod_len, 1, n_mod, ws + l.sched, s, true,
                                               (uint32_t)env_int("SKG_DIS_SHIFT", 6)))) return e;
  a.order = reinterpret_cast<const uint32_t*>(ws + l.sched + skg::SCHED_PERM_OFF);
  a.stage_bytes = kDisStage;
  const Geom g = dis_geom(n_mod);
  a.group_warps = group_warps((int)g.warps, env_int("SKG_DIS_GROUP", (int)g.warps));
  const size_t smem_max = (size_t)(kDisSlab + kDisStage) * kDisWarps;
  const size_t smem = (size_t)(kDisSlab + kDisStage) * g.warps;
  static uint64_t attr = 0;
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(skg::disasm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    cudaFuncSetAttribute(skg::pipeline_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
  }
  static uint64_t carve = 0;
  if (first_on_device(carve)) {   // smallest shared-memory carveout that fits: the rest is L1 for the scratch
    const int pct = env_int("SKG_CARVEOUT", -2);
    if (pct != -2) {
      cudaFuncSetAttribute(skg::disasm_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      cudaFuncSetAttribute(skg::pipeline_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    }
  }
  if (vo) skg::pipeline_kernel<<<g.blocks, 32 * g.warps, smem, s>>>(a);
  else skg::disasm_kernel<<<g.blocks, 32 * g.warps, smem, s>>>(a);
  return check(cudaGetLastError());
}
}  // namespace

int skg_disasm_refs(const skg_tables* t, const uint8_t* data, const int64_t* mod_off,
                    const int64_t* mod_len, uint32_t n_mod, uint32_t opts, uint32_t max_words,
                    uint8_t* text, uint64_t text_cap, int64_t* text_span, int32_t* status,
                    skg_error* errors, uint32_t err_cap, void* workspace, uint64_t workspace_bytes,
                    void* stream, const uint32_t* ref_ids, const uint8_t* ref_text, uint32_t n_refs) {
  return disasm_launch(t, data, mod_off, mod_len, n_mod, opts, max_words, text, text_cap, text_span, status, errors,
                       err_cap, workspace, workspace_bytes, stream, ref_ids, ref_text, n_refs, nullptr);
}

int skg_disasm_validate(const skg_tables* t, const uint8_t* data, const int64_t* mod_off,
                        const int64_t* mod_len, uint32_t n_mod, uint32_t opts, uint32_t max_words,
                        uint8_t* text, uint64_t text_cap, int64_t* text_span, int32_t* status,
                        skg_error* errors, uint32_t err_cap, uint8_t* vtext, uint64_t vtext_cap,
                        int64_t* vtext_span, int32_t* vstatus, skg_error* verrors, uint32_t verr_cap,
                        void* workspace, uint64_t workspace_bytes, void* stream) {
  const ValOut vo{vtext, vtext_cap, vtext_span, vstatus, verrors, verr_cap};
  return disasm_launch(t, data, mod_off, mod_len, n_mod, opts, max_words, text, text_cap, text_span, status, errors,
                       err_cap, workspace, workspace_bytes, stream, nullptr, nullptr, 0, &vo);
}

int skg_validate(const skg_tables* t, const uint8_t* data, const int64_t* mod_off,
                 const int64_t* mod_len, uint32_t n_mod, uint32_t max_words, uint8_t* text,
                 uint64_t text_cap, int64_t* text_span, int32_t* status, skg_error* errors,
                 uint32_t err_cap, void* workspace, uint64_t workspace_bytes, void* stream) {
  if (!t || !workspace) return -1;
  WsLayout l = ws_layout(n_mod, max_words);
  if (workspace_bytes < l.total) return -3;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* ws = (uint8_t*)workspace;
  if (int e = check(cudaMemsetAsync(ws, 0, l.scratch, s))) return e;
  if (n_mod == 0) return 0;
  skg::ValidateArgs a;
  a.T = t->t;
  a.data = data; a.mod_off = mod_off; a.mod_len = mod_len; a.n_mod = n_mod;
  a.text = text; a.text_cap = text_cap; a.text_span = text_span; a.status = status;
  a.ticket = reinterpret_cast<uint32_t*>(ws + l.counters);
  a.errs = reinterpret_cast<skg::ErrRec*>(errors);
  a.err_cap = err_cap;
  a.gscratch = ws + l.scratch;
  a.gslot_bytes = l.slot;
  a.smem_slab = 0;
  // size order only: region-major measured 53.3 -> 54.6 ms on the 1M-module batch here
  if (int e = check((cudaError_t)launch_sched(mod_len, 1, n_mod, ws + l.sched, s, env_int("SKG_VAL_REGIONS", 0) != 0,
                                               (uint32_t)env_int("SKG_VAL_SHIFT", 6)))) return e;
  a.order = reinterpret_cast<const uint32_t*>(ws + l.sched + skg::SCHED_PERM_OFF);
  const Geom g = val_geom(n_mod);
  a.group_warps = group_warps((int)g.warps, env_int("SKG_VAL_GROUP", (int)g.warps));
  static uint64_t carve = 0;
  if (first_on_device(carve)) {
    const int pct = env_int("SKG_CARVEOUT", -2);
    if (pct != -2) cudaFuncSetAttribute(skg::validate_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  }
  skg::validate_kernel<<<g.blocks, 32 * g.warps, 0, s>>>(a);
  return check(cudaGetLastError());
}

uint64_t skg_asm_slot_hint(uint64_t max_text_bytes) {
  return ((32ull * max_text_bytes + 65536) + 255) & ~255ull;
}

// assembler: phase-synchronised CTAs of kAsmWarps warps (one module per warp), 2 per SM
int kAsmWarps = env_int("SKG_ASM_WARPS", 32);
uint32_t asm_blocks() {
  const int g = env_int("SKG_ASM_GRID", 0);   // experiments: explicit grid
  return g > 0 ? (uint32_t)g : (uint32_t)sm_count() * env_int("SKG_ASM_BLOCKS_PER_SM", 1);
}

Geom asm_geom(uint32_t n_mod) { return fit_geom(asm_blocks(), (uint32_t)kAsmWarps, n_mod, true); }

uint64_t skg_asm_workspace_bytes(uint64_t slot_bytes, uint32_t n_mod) {
  const Geom g = asm_geom(n_mod);
  return 256 + sched_bytes(n_mod) + (uint64_t)g.blocks * g.warps * slot_bytes;
}

int skg_asm(const skg_tables* t, const uint8_t* text, const int64_t* mod_off, const int64_t* mod_len,
            uint32_t mod_stride, uint32_t n_mod, uint64_t slot_bytes, uint8_t* out, uint64_t out_cap, int64_t* out_span,
            int32_t* status, void* workspace, uint64_t workspace_bytes, void* stream,
            uint32_t default_version) {
  if (!t || !workspace) return -1;
  if (t->a.op_label == 0xFFFFFFFFu || t->a.op_fnend == 0xFFFFFFFFu) return -4;
  if (workspace_bytes < skg_asm_workspace_bytes(slot_bytes, n_mod)) return -3;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* ws = (uint8_t*)workspace;
  if (int e = check(cudaMemsetAsync(ws, 0, 256, s))) return e;
  if (n_mod == 0) return 0;
  skg::AsmArgs a;
  a.T = t->t; a.U = t->u; a.A = t->a;
  a.text = text; a.mod_off = mod_off; a.mod_len = mod_len; a.n_mod = n_mod;
  a.mod_stride = mod_stride ? mod_stride : 1;
  a.out = out; a.out_cap = out_cap; a.out_span = out_span; a.status = status;
  a.counters = reinterpret_cast<uint32_t*>(ws);
  // Size order (text bytes), not region-major: the texts already lie in the disassembler's
  // processing order (region-major measured 159 -> 169 ms on the bench's 1M-module batch).
  // A work key of 4 x lines + tokens per text (counted by a SWAR kernel) balanced the CTAs'
  // lines/tokens far better on paper (max/mean 1.41 -> 1.06) but measured 159 -> 161 ms.
  if (int e = check((cudaError_t)launch_sched(mod_len, a.mod_stride, n_mod, ws + 256, s,
                                               env_int("SKG_ASM_REGIONS", 0) != 0,
                                               (uint32_t)env_int("SKG_ASM_SHIFT", 6)))) return e;
  a.order = reinterpret_cast<const uint32_t*>(ws + 256 + skg::SCHED_PERM_OFF);
  a.gscratch = ws + 256 + sched_bytes(n_mod);
  a.gslot_bytes = slot_bytes;
  a.default_version = default_version;
  const Geom g = asm_geom(n_mod);
  a.group_warps = group_warps((int)g.warps, env_int("SKG_ASM_GROUP", (int)g.warps));
  static uint64_t carve = 0;
  if (first_on_device(carve)) {
    const int pct = env_int("SKG_CARVEOUT", -2);
    if (pct != -2) cudaFuncSetAttribute(skg::asm_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  }
  skg::asm_kernel<<<g.blocks, 32 * g.warps, 0, s>>>(a);
  return check(cudaGetLastError());
}

namespace {
// the link arrays after entry / count (skg_decode_large_workspace_bytes)
void bd_link_layout(skg::BigDecode& b, uint32_t* q) {
  const uint64_t N = (uint64_t)b.ntiles * skg::BD_K;
  uint32_t levels = 1;
  while ((1ull << levels) <= b.ntiles) ++levels;
  b.levels = levels;
  b.next = q; q += N;
  b.tpos = q; q += N;
  b.tcode = q; q += N;
  b.jump = q;
}
// the tiles linked in parallel (successors, doubling, path); the sequential link only
// if some speculative exit on the true chain landed on an unmarked position
void bd_link(const skg::BigDecode& b, cudaStream_t s) {
  const uint32_t N = b.ntiles * skg::BD_K;
  skg::tile_entry_init<<<(b.ntiles + 255) / 256, 256, 0, s>>>(b);
  skg::tile_land<<<(N + 127) / 128, 128, 0, s>>>(b);
  for (uint32_t r = 1; r < b.levels; ++r) skg::tile_jump<<<(N + 255) / 256, 256, 0, s>>>(b, r);
  skg::tile_path<<<(b.ntiles + 1 + 255) / 256, 256, 0, s>>>(b);
  skg::tile_link_if_raw<<<1, 32, 0, s>>>(b);
}
}  // namespace

uint64_t skg_decode_large_workspace_bytes(uint64_t n_words) {
  const uint64_t nt = (n_words + skg::BD_TILE - 1) / skg::BD_TILE;
  uint64_t levels = 1;
  while ((1ull << levels) <= nt) ++levels;
  // chain maps, speculative exits / errors, entries + counts (+1 spare), then the
  // parallel link's successor / terminal arrays and doubled maps (u32 per node per level)
  return 256 + nt * skg::BD_TILE + 3 * 4 * skg::BD_K * nt + 3 * 4 * nt +
         (3 + levels) * 4 * skg::BD_K * nt + 256;
}

int skg_decode_large(const uint8_t* data, uint64_t nbytes, uint32_t max_opcode, uint32_t* header,
                     uint32_t* inst_off, uint32_t* inst_count, uint32_t* words_out, int32_t* status,
                     skg_error* error, void* workspace, uint64_t workspace_bytes, void* stream) {
  const uint64_t W64 = nbytes / 4;
  if (!workspace || !data || W64 > 0xFFFFFFF0ull) return -1;
  if (workspace_bytes < skg_decode_large_workspace_bytes(W64)) return -3;
  cudaStream_t s = (cudaStream_t)stream;
  skg::BigDecode b;
  b.src = data; b.nbytes = nbytes; b.W = (uint32_t)W64; b.words = words_out; b.inst_off = inst_off;
  b.ntiles = (uint32_t)((W64 + skg::BD_TILE - 1) / skg::BD_TILE);
  uint8_t* ws = (uint8_t*)workspace;
  b.result = reinterpret_cast<uint32_t*>(ws);
  b.max_opcode = max_opcode ? max_opcode : 0xFFFFu;
  b.chain = ws + 256;
  uint32_t* q = reinterpret_cast<uint32_t*>(ws + 256 + (uint64_t)b.ntiles * skg::BD_TILE);
  b.spec_exit = q; q += (uint64_t)b.ntiles * skg::BD_K;
  b.spec_err = q; q += (uint64_t)b.ntiles * skg::BD_K;
  b.spec_errc = q; q += (uint64_t)b.ntiles * skg::BD_K;
  b.entry = q; q += b.ntiles;
  b.count = q; q += b.ntiles;
  q += b.ntiles;
  bd_link_layout(b, q);
  const uint32_t tb = 128, tg = (b.ntiles + tb - 1) / tb;
  skg::big_prologue<<<1, 32, 0, s>>>(b);
  if (b.W >= 5) {
    skg::big_copy<<<sm_count() * 8, 256, 0, s>>>(b);
    cudaMemsetAsync(b.chain, 0, (size_t)b.ntiles * skg::BD_TILE, s);   // chain maps (a memset beats a thread per tile)
    skg::tile_spec<<<tg, tb, 0, s>>>(b);
    bd_link(b, s);
    skg::tile_count<<<tg, tb, 0, s>>>(b);
    skg::tile_scan<<<1, 1024, 0, s>>>(b);
    skg::tile_write<<<tg, tb, 0, s>>>(b);
  }
  skg::big_epilogue<<<1, 32, 0, s>>>(b, header, inst_count, status, reinterpret_cast<skg::ErrRec*>(error));
  return check(cudaGetLastError());
}

// -- one large module over the whole GPU (skg_big.cuh) ----------------------------
namespace {
struct LargeWs {
  uint32_t* ctl;
  uint8_t* dec;
  skg::Mod* mod;
  uint8_t* slot;
  uint32_t* sums;
  uint64_t total;
};
uint64_t al256(uint64_t x) { return (x + 255) & ~255ull; }
LargeWs large_ws(uint8_t* ws, uint64_t W, uint32_t bound) {
  LargeWs l;
  uint64_t o = 0;
  l.ctl = reinterpret_cast<uint32_t*>(ws + o); o += 256;
  l.dec = ws + o; o += al256(skg_decode_large_workspace_bytes(W));
  l.mod = reinterpret_cast<skg::Mod*>(ws + o); o += al256(sizeof(skg::Mod));
  l.slot = ws + o; o += al256(skg::big_slot_bytes((uint32_t)W, bound));
  l.sums = reinterpret_cast<uint32_t*>(ws + o); o += al256(4 * (3 * W / skg::BS_BLOCK + 4));   // N <= 2W + 64
  l.total = o;
  return l;
}

// tiled boundary pass into the module scratch + layout; returns the decode status
// (host-synchronous) or -1 on a CUDA error
int large_front(const uint8_t* data, uint64_t nbytes, uint32_t max_opcode, const LargeWs& l, skg::ErrRec* derr,
                cudaStream_t s, uint32_t min_table) {
  skg::BigDecode b;
  const uint64_t W = nbytes / 4;
  b.src = data; b.nbytes = nbytes; b.W = (uint32_t)W;
  b.words = reinterpret_cast<uint32_t*>(l.slot + 64);
  b.inst_off = reinterpret_cast<uint32_t*>(l.slot + 64 + skg::align16(4 * W));
  b.ntiles = (uint32_t)((W + skg::BD_TILE - 1) / skg::BD_TILE);
  b.result = l.ctl;
  b.max_opcode = max_opcode ? max_opcode : 0xFFFFu;
  b.chain = l.dec + 256;
  uint32_t* q = reinterpret_cast<uint32_t*>(l.dec + 256 + (uint64_t)b.ntiles * skg::BD_TILE);
  b.spec_exit = q; q += (uint64_t)b.ntiles * skg::BD_K;
  b.spec_err = q; q += (uint64_t)b.ntiles * skg::BD_K;
  b.spec_errc = q; q += (uint64_t)b.ntiles * skg::BD_K;
  b.entry = q; q += b.ntiles;
  b.count = q; q += b.ntiles;
  q += b.ntiles;
  bd_link_layout(b, q);
  const uint32_t tb = 128, tg = (b.ntiles + tb - 1) / tb;
  uint32_t* hdr = reinterpret_cast<uint32_t*>(l.dec);          // scratch for the epilogue outputs
  skg::big_prologue<<<1, 32, 0, s>>>(b);
  if (b.W >= 5) {
    skg::big_copy<<<sm_count() * 8, 256, 0, s>>>(b);
    cudaMemsetAsync(b.chain, 0, (size_t)b.ntiles * skg::BD_TILE, s);   // chain maps (a memset beats a thread per tile)
    skg::tile_spec<<<tg, tb, 0, s>>>(b);
    bd_link(b, s);
    skg::tile_count<<<tg, tb, 0, s>>>(b);
    skg::tile_scan<<<1, 1024, 0, s>>>(b);
    skg::tile_write<<<tg, tb, 0, s>>>(b);
  }
  skg::big_epilogue<<<1, 32, 0, s>>>(b, hdr, hdr + 8, reinterpret_cast<int32_t*>(hdr + 9), derr);
  uint32_t st = 0;
  if (check(cudaMemcpyAsync(&st, l.ctl, 4, cudaMemcpyDeviceToHost, s)) || check(cudaStreamSynchronize(s))) return -1;
  if (st != 0) return (int)st;
  skg::big_setup<<<1, 1, 0, s>>>(l.mod, l.slot, (uint32_t)W, l.ctl, min_table);
  return check(cudaGetLastError()) ? -1 : 0;
}

uint32_t grid_for(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  const uint64_t cap = (uint64_t)sm_count() * 8;
  return (uint32_t)(b < 1 ? 1 : (b > cap ? cap : b));
}
}  // namespace

namespace {
int64_t large_scan_total(uint32_t* a, uint32_t n, const LargeWs& l, cudaStream_t s);
}

uint64_t skg_large_workspace_bytes(uint64_t n_words, uint32_t bound) {
  return large_ws(nullptr, n_words, bound).total;
}

int skg_validate_large(const skg_tables* t, const uint8_t* data, uint64_t nbytes, uint8_t* text,
                       uint64_t text_cap, uint64_t* text_bytes, int32_t* status, skg_error* error,
                       void* workspace, uint64_t workspace_bytes, void* stream, uint32_t min_table) {
  if (!t || !workspace || !data || !text_bytes || nbytes / 4 > 0xFFFFFFF0ull) return -1;
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t W = nbytes / 4;
  // the header bound sizes the direct id tables
  uint32_t hdr[5] = {0, 0, 0, 0, 0};
  if (W >= 5 && check(cudaMemcpyAsync(hdr, data, 20, cudaMemcpyDeviceToHost, s))) return -1;
  if (check(cudaStreamSynchronize(s))) return -1;
  uint32_t bound = hdr[3];
  if (hdr[0] == 0x03022307u) bound = __builtin_bswap32(bound);
  if (min_table > bound) bound = min_table;                         // direct table size
  if ((uint64_t)bound > 2 * W + 64) return 2;                      // not direct: use skg_validate
  const LargeWs l = large_ws((uint8_t*)workspace, W, bound);
  if (workspace_bytes < l.total) return -3;
  *text_bytes = 0;
  const int dst = large_front(data, nbytes, t->t.max_opcode, l, reinterpret_cast<skg::ErrRec*>(error), s, min_table);
  if (dst < 0) return -1;
  if (dst > 0) return 10 + dst;                                    // decode error: caller formats it
  skg::big_init_tables<<<grid_for(bound), 256, 0, s>>>(l.mod);
  uint32_t I = 0;
  if (check(cudaMemcpyAsync(&I, l.ctl + skg::BC_COUNT, 4, cudaMemcpyDeviceToHost, s))) return -1;
  skg::big_prescan<<<grid_for(W), 256, 0, s>>>(l.mod, t->t, l.ctl);
  skg::big_fix_tables<<<grid_for(bound), 256, 0, s>>>(l.mod);
  skg::big_val_shape<<<grid_for(W), 256, 0, s>>>(l.mod, t->t, l.ctl);
  skg::big_val_sizes<<<grid_for(W), 256, 0, s>>>(l.mod, t->t, l.ctl);
  uint32_t ctl[64];
  if (check(cudaMemcpyAsync(ctl, l.ctl, sizeof(ctl), cudaMemcpyDeviceToHost, s)) || check(cudaStreamSynchronize(s)))
    return -1;
  if (ctl[skg::BC_OVER]) return 2;                                 // an id at/above the bound
  if (ctl[skg::BC_BAD] != 0xFFFFFFFFu) {                           // an exception escapes
    skg::big_val_error<<<1, 32, 0, s>>>(l.mod, t->t, l.ctl, reinterpret_cast<skg::ErrRec*>(error), status);
    return check(cudaStreamSynchronize(s)) ? -1 : 1;
  }
  // per-instruction offsets: ia (I entries) lives in the module scratch
  skg::Mod m;
  if (check(cudaMemcpyAsync(&m, l.mod, sizeof(m), cudaMemcpyDeviceToHost, s))) return -1;
  if (check(cudaStreamSynchronize(s))) return -1;
  const int64_t body = large_scan_total(m.ia, I, l, s);
  if (body < 0) return (int)body;
  uint32_t tot[4];
  if (check(cudaMemcpyAsync(tot, l.ctl + skg::BC_TOTAL, 16, cudaMemcpyDeviceToHost, s)) ||
      check(cudaStreamSynchronize(s)))
    return -1;
  const uint64_t total = (uint64_t)tot[0] + (uint64_t)body;
  if (total > 0xFFFFFFFFull) return -4;                            // diagnostics offsets are 32-bit
  *text_bytes = total;
  if (total > text_cap) return 3;                                  // grow the arena and call again
  skg::big_val_write<<<grid_for(W), 256, 0, s>>>(l.mod, t->t, l.ctl, text);
  const int32_t ok = 0;
  if (check(cudaMemcpyAsync(status, &ok, 4, cudaMemcpyHostToDevice, s))) return -1;
  return check(cudaStreamSynchronize(s)) ? -1 : 0;
}

namespace {
// exclusive scan of n uint32 in place; returns the total (host-synchronous)
// returns -1 on a CUDA error, -4 when the total does not fit the 32-bit offsets
int64_t large_scan_total(uint32_t* a, uint32_t n, const LargeWs& l, cudaStream_t s) {
  unsigned long long* sum = reinterpret_cast<unsigned long long*>(l.ctl + skg::BC_SUM);
  unsigned long long tot64 = 0;
  if (check(cudaMemsetAsync(sum, 0, 8, s))) return -1;
  if (n) skg::sum_u64<<<grid_for(n), 256, 0, s>>>(a, n, sum);
  if (check(cudaMemcpyAsync(&tot64, sum, 8, cudaMemcpyDeviceToHost, s)) || check(cudaStreamSynchronize(s)))
    return -1;
  if (tot64 > 0xFFFFFFFFull) return -4;
  const uint32_t nb = (n + skg::BS_BLOCK - 1) / skg::BS_BLOCK;
  if (nb) skg::scan_blocks<<<nb, skg::BS_BLOCK, 0, s>>>(a, n, l.sums);
  skg::scan_top<<<1, skg::BS_BLOCK, 0, s>>>(l.sums, nb, l.ctl + skg::BC_SCAN);
  if (nb) skg::scan_apply<<<nb, skg::BS_BLOCK, 0, s>>>(a, n, l.sums);
  uint32_t tot = 0;
  if (check(cudaMemcpyAsync(&tot, l.ctl + skg::BC_SCAN, 4, cudaMemcpyDeviceToHost, s)) ||
      check(cudaStreamSynchronize(s)))
    return -1;
  return tot;
}
int read_ctl(const LargeWs& l, uint32_t* out64, cudaStream_t s) {
  return check(cudaMemcpyAsync(out64, l.ctl, 256, cudaMemcpyDeviceToHost, s)) || check(cudaStreamSynchronize(s));
}
}  // namespace

namespace {
// closed-form name de-duplication (skg_disasm.cu bnc_*): stable radix sorts of the
// named idents by group leader and of the child list by (parent, serial), group and
// child ranges, one kernel per level of the parent / child tree, then the serials
int name_dedup_closed(const LargeWs& l, uint32_t nd, const uint32_t* clist, uint32_t nc, cudaStream_t s) {
  using namespace skg;
  if (nd == 0) return 0;
  const uint32_t ncx = nc ? nc : 1;
  int bits = 1;
  while (bits < 32 && (1ull << bits) < nd) ++bits;
  const bool dbg = getenv("SKG_DEBUG_SYNC") != nullptr;
  size_t tmp_sort = 0, tmp_csort = 0;
  const cudaError_t q1 = cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, (const uint32_t*)nullptr,
                                                         (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                                         (uint32_t*)nullptr, (int)nd, 0, bits, s);
  const cudaError_t q2 = cub::DeviceRadixSort::SortPairs(nullptr, tmp_csort, (const unsigned long long*)nullptr,
                                                         (unsigned long long*)nullptr, (const uint32_t*)nullptr,
                                                         (uint32_t*)nullptr, (int)ncx, 0, 64, s);
  if (int e = check(q1 != cudaSuccess ? q1 : q2)) return e;
  const size_t tmp = std::max(tmp_sort, tmp_csort);
  // buffers: 4 x nd members, 6 x nd per-leader arrays, nd flags, 4 x nc children, skips
  // (+ 256-byte alignment of each of the 17 pieces)
  const size_t bytes = 16ull * nd + 24ull * nd + ((nd + 15) & ~15ull) + 24ull * ncx + 4ull * ncx + tmp + 17 * 256;
  // a per-device buffer kept across calls (grow-only): a cudaMalloc / cudaFree of a few
  // hundred MB per call synchronises the device and costs milliseconds; the lock keeps
  // concurrent host threads on one device from sharing it mid-call
  int dev = 0;
  if (int e = check(cudaGetDevice(&dev))) return e;
  static std::mutex locks[64];
  static uint8_t* bufs[64] = {};
  static size_t caps[64] = {};
  if (dev < 0 || dev >= 64) return -1;
  std::lock_guard<std::mutex> guard(locks[dev]);
  if (caps[dev] < bytes) {
    if (bufs[dev]) cudaFree(bufs[dev]);
    bufs[dev] = nullptr; caps[dev] = 0;
    const size_t grow = bytes + bytes / 4;
    if (int e = check(cudaMalloc(reinterpret_cast<void**>(&bufs[dev]), grow))) return e;
    caps[dev] = grow;
  }
  uint8_t* buf = bufs[dev];
  uint8_t* p = buf;
  auto take = [&](size_t b) { uint8_t* r = p; p += (b + 255) & ~255ull; return r; };
  uint32_t* keys = reinterpret_cast<uint32_t*>(take(4ull * nd));
  uint32_t* vals = reinterpret_cast<uint32_t*>(take(4ull * nd));
  uint32_t* skeys = reinterpret_cast<uint32_t*>(take(4ull * nd));
  uint32_t* svals = reinterpret_cast<uint32_t*>(take(4ull * nd));
  uint8_t* zero0 = p;                                              // zero-initialised from here
  uint32_t* gstart = reinterpret_cast<uint32_t*>(take(4ull * nd));
  uint32_t* gend = reinterpret_cast<uint32_t*>(take(4ull * nd));
  uint32_t* cstart = reinterpret_cast<uint32_t*>(take(4ull * nd));
  uint32_t* cend = reinterpret_cast<uint32_t*>(take(4ull * nd));
  uint32_t* depth = reinterpret_cast<uint32_t*>(take(4ull * nd));
  uint32_t* nskip = reinterpret_cast<uint32_t*>(take(4ull * nd));
  uint8_t* btaken = take(nd);
  uint8_t* zero1 = p;
  auto* ckeys = reinterpret_cast<unsigned long long*>(take(8ull * ncx));
  auto* sckeys = reinterpret_cast<unsigned long long*>(take(8ull * ncx));
  uint32_t* cvals = reinterpret_cast<uint32_t*>(take(4ull * ncx));
  uint32_t* scvals = reinterpret_cast<uint32_t*>(take(4ull * ncx));
  uint32_t* skipq = reinterpret_cast<uint32_t*>(take(4ull * ncx));
  void* ctmp = take(tmp);
  int rc = 0;
  const uint32_t gN = grid_for(nd), gC = grid_for(ncx);
  auto step_ok = [&](const char* what) -> bool {   // SKG_DEBUG_SYNC: synchronise and name a failing step
    if (!dbg) return true;
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { fprintf(stderr, "skgpu: name_dedup_closed %s: %s\n", what, cudaGetErrorString(e)); rc = (int)e; }
    return e == cudaSuccess;
  };
  do {
    if ((rc = check(cudaMemsetAsync(zero0, 0, (size_t)(zero1 - zero0), s)))) break;
    if (!step_ok("memset")) break;
    bnc_keys<<<gN, 256, 0, s>>>(l.mod, nd, keys, vals, clist, nc, ckeys, cvals);
    if (!step_ok("keys")) break;
    size_t t1 = tmp;
    if ((rc = check(cub::DeviceRadixSort::SortPairs(ctmp, t1, keys, skeys, vals, svals, (int)nd, 0, bits, s)))) break;
    if (nc) {
      size_t t2 = tmp;
      if ((rc = check(cub::DeviceRadixSort::SortPairs(ctmp, t2, ckeys, sckeys, cvals, scvals, (int)nc, 0, 64, s))))
        break;
    }
    if (!step_ok("sorts")) break;
    bnc_ranges<<<gN, 256, 0, s>>>(l.mod, nd, skeys, gstart, gend, nc, sckeys, cstart, cend, depth, l.ctl);
    uint32_t maxd = 0;
    if ((rc = check(cudaMemcpyAsync(&maxd, l.ctl + BC_DEPTH, 4, cudaMemcpyDeviceToHost, s)))) break;
    if ((rc = check(cudaStreamSynchronize(s)))) break;
    if (nc)
      for (uint32_t lv = 0; lv <= maxd; ++lv)
        bnc_level<<<gC, 256, 0, s>>>(nc, sckeys, scvals, svals, gstart, gend, cstart, cend, depth, lv, btaken, skipq,
                                     nskip);
    if (!step_ok("levels")) break;
    bnc_assign<<<gN, 256, 0, s>>>(l.mod, nd, skeys, svals, gstart, btaken, cstart, skipq, nskip);
    rc = check(cudaGetLastError());
    step_ok("assign");
  } while (false);
  if (!rc) rc = check(cudaStreamSynchronize(s));
  return rc;
}
}  // namespace

int skg_disasm_large(const skg_tables* t, const uint8_t* data, uint64_t nbytes, uint32_t opts, uint8_t* text,
                     uint64_t text_cap, uint64_t* text_bytes, int32_t* status, skg_error* error,
                     void* workspace, uint64_t workspace_bytes, void* stream, uint32_t min_table) {
  using namespace skg;
  if (!t || !workspace || !data || !text_bytes || nbytes / 4 > 0xFFFFFFF0ull) return -1;
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t W = nbytes / 4;
  uint32_t hdr[5] = {0, 0, 0, 0, 0};
  if (W >= 5 && check(cudaMemcpyAsync(hdr, data, 20, cudaMemcpyDeviceToHost, s))) return -1;
  if (check(cudaStreamSynchronize(s))) return -1;
  uint32_t bound = hdr[3];
  if (hdr[0] == 0x03022307u) bound = __builtin_bswap32(bound);
  if (min_table > bound) bound = min_table;                         // direct table size
  if ((uint64_t)bound > 2 * W + 64) return 2;
  const LargeWs l = large_ws((uint8_t*)workspace, W, bound);
  if (workspace_bytes < l.total) return -3;
  *text_bytes = 0;
  ErrRec* rec = reinterpret_cast<ErrRec*>(error);
  const int dst = large_front(data, nbytes, t->t.max_opcode, l, rec, s, min_table);
  if (dst < 0) return -1;
  if (dst > 0) return 10 + dst;                                    // decode exception (record in *error)
  const Tables& T = t->t;
  const uint32_t gW = grid_for(W), gS = grid_for(bound);
  uint32_t ctl[64];
  big_init_tables<<<gS, 256, 0, s>>>(l.mod);
  big_prescan<<<gW, 256, 0, s>>>(l.mod, T, l.ctl);
  big_fix_tables<<<gS, 256, 0, s>>>(l.mod);
  bd_classify<<<gW, 256, 0, s>>>(l.mod, T);
  if (read_ctl(l, ctl, s)) return -1;
  if (ctl[BC_OVER]) return 2;
  const bool names_mode = (opts & OPT_INLINE) && ctl[BC_ANYNAME];
  Mod m;
  if (check(cudaMemcpyAsync(&m, l.mod, sizeof(m), cudaMemcpyDeviceToHost, s))) return -1;
  if (names_mode) bd_collect<<<gW, 256, 0, s>>>(l.mod);
  bd_errors<<<gW, 256, 0, s>>>(l.mod, l.ctl, opts, names_mode);
  uint32_t ovf = 0;
  if (check(cudaMemcpyAsync(&ovf, m.overflow, 4, cudaMemcpyDeviceToHost, s))) return -1;
  if (read_ctl(l, ctl, s)) return -1;
  if (ovf) return 2;                                               // a referenced id at/above the bound
  const uint32_t bad1 = ctl[BC_E1], bad2 = ctl[BC_E2], bad3 = ctl[BC_E3];
  if (bad1 != NONE32 || bad2 != NONE32 || bad3 != NONE32) {
    const uint32_t which = bad1 != NONE32 ? 1 : (bad2 != NONE32 ? 2 : 3);
    bd_error_rec<<<1, 32, 0, s>>>(l.mod, T, which, which == 1 ? bad1 : (which == 2 ? bad2 : bad3), rec, status);
    return check(cudaStreamSynchronize(s)) ? -1 : 1;
  }
  const uint32_t I = m.I;
  if (names_mode) {
    bn_flags<<<gS, 256, 0, s>>>(l.mod, l.ctl);
    bn_mark<<<gW, 256, 0, s>>>(l.mod, T);
    const int64_t cj = large_scan_total(m.ib, I, l, s);
    const int64_t nd64 = large_scan_total(m.ia, I, l, s);
    if (cj < 0 || nd64 < 0) return (int)std::min(cj, nd64);
    if (read_ctl(l, ctl, s)) return -1;
    const uint32_t nd = (uint32_t)nd64, N = ctl[BC_NP0] + (uint32_t)cj;
    bn_ndl<<<gW, 256, 0, s>>>(l.mod, T);
    for (uint32_t step = 0; step < 3; ++step) bn_pos<<<grid_for(std::max<uint64_t>(N + 1, std::max<uint64_t>(I, bound))), 256, 0, s>>>(l.mod, T, N, step);
    if (N >= 1) {   // inclusive prefix max over pos[1..N] from -2
      int32_t* a = m.pos + 1;
      const uint32_t nb = (N + BS_BLOCK - 1) / BS_BLOCK;
      int32_t* maxes = reinterpret_cast<int32_t*>(l.sums);
      maxscan_blocks<<<nb, BS_BLOCK, 0, s>>>(a, N, maxes);
      maxscan_top<<<1, 32, 0, s>>>(maxes, nb, -2);
      maxscan_apply<<<nb, BS_BLOCK, 0, s>>>(a, N, maxes);
    }
    bn_kept<<<gW, 256, 0, s>>>(l.mod, T, N);
    uint32_t C = 4;
    while (C < 2 * nd) C <<= 1;
    uint32_t* htab = reinterpret_cast<uint32_t*>(m.spill);
    const uint32_t gN = grid_for(nd), gC = grid_for(C);
    bn_step<<<gN, 256, 0, s>>>(l.mod, htab, C, nd, 0);
    bn_step<<<gC, 256, 0, s>>>(l.mod, htab, C, nd, 1);
    for (uint32_t step = 2; step <= 5; ++step) bn_step<<<gN, 256, 0, s>>>(l.mod, htab, C, nd, step);
    uint32_t* clist = reinterpret_cast<uint32_t*>(m.spill);       // the table is no longer needed
    uint32_t* flags = clist + 4ull * nd;                            // spill holds >= 32 nd bytes
    bn_children<<<gN, 256, 0, s>>>(l.mod, flags, clist, nd, 0);
    const int64_t nc = large_scan_total(flags, nd, l, s);
    if (nc < 0) return (int)nc;
    bn_children<<<gN, 256, 0, s>>>(l.mod, flags, clist, nd, 1);
    if (int e = name_dedup_closed(l, nd, clist, (uint32_t)nc, s)) return e;
    bn_arena<<<gN, 256, 0, s>>>(l.mod, flags, nd, 0);
    const int64_t arena = large_scan_total(flags, nd, l, s);
    if (arena < 0) return (int)arena;
    bn_arena<<<gN, 256, 0, s>>>(l.mod, flags, nd, 1);
  }
  bd_refs<<<gS, 256, 0, s>>>(l.mod, T, l.ctl, 0);
  bd_refs<<<gW, 256, 0, s>>>(l.mod, T, l.ctl, 1);
  if (opts & OPT_GROUP) {
    bd_sections<<<1, 32, 0, s>>>(l.mod, T);
    bd_blanks<<<gW, 256, 0, s>>>(l.mod);
  }
  bd_header_len<<<1, 32, 0, s>>>(l.mod, opts, l.ctl);
  if (read_ctl(l, ctl, s)) return -1;
  const uint32_t width = (opts & OPT_NO_INDENT) ? 0 : ctl[BC_WIDTH];
  const uint32_t head = ctl[BC_TOTAL];
  const uint32_t nr = (uint32_t)((W - 5 + BD_RANGE - 1) / BD_RANGE);
  uint32_t* rsum = reinterpret_cast<uint32_t*>(m.spill);           // names are done with the spill area
  bd_lengths<<<grid_for((uint64_t)nr * 32), 256, 0, s>>>(l.mod, T, opts, width, rsum);
  const int64_t body = nr ? large_scan_total(rsum, nr, l, s) : 0;
  if (body < 0) return (int)body;
  const uint64_t total = (uint64_t)head + (uint64_t)body;
  if (total > 0xFFFFFFFFull) return -4;                            // text offsets are 32-bit
  *text_bytes = total;
  if (total > text_cap) return 3;
  bd_render<<<grid_for((uint64_t)nr * 32 + 32), 256, 8 * 1024, s>>>(l.mod, T, opts, width, text, rsum, head);
  const int32_t ok = 0;
  if (check(cudaMemcpyAsync(status, &ok, 4, cudaMemcpyHostToDevice, s))) return -1;
  return check(cudaStreamSynchronize(s)) ? -1 : 0;
}

int skg_decode(const uint8_t* data, const int64_t* mod_off, const int64_t* mod_len, uint32_t n_mod,
               uint32_t* header, uint32_t* inst_off, const int64_t* inst_base, uint32_t* inst_count,
               uint32_t* words_out, const int64_t* words_base, int32_t* status, skg_error* errors,
               uint32_t err_cap, void* workspace, uint64_t workspace_bytes, void* stream) {
  if (!workspace) return -1;
  if (workspace_bytes < 256) return -3;
  cudaStream_t s = (cudaStream_t)stream;
  if (int e = check(cudaMemsetAsync(workspace, 0, 256, s))) return e;
  if (n_mod == 0) return 0;
  skg::DecodeArgs a;
  a.data = data; a.mod_off = mod_off; a.mod_len = mod_len; a.n_mod = n_mod;
  a.header = header; a.inst_off = inst_off; a.inst_base = inst_base; a.inst_count = inst_count;
  a.words_out = words_out; a.words_base = words_base; a.status = status;
  a.counters = reinterpret_cast<uint32_t*>(workspace);
  a.errs = reinterpret_cast<skg::ErrRec*>(errors);
  a.err_cap = err_cap;
  const uint32_t threads = 256;
  uint32_t blocks = (n_mod + threads - 1) / threads;
  skg::decode_kernel<<<blocks, threads, 0, s>>>(a);
  return check(cudaGetLastError());
}


// -- standalone codec / tokenizer entries (skg_codec.cuh) --------------------------------
namespace {
uint32_t item_grid(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  const uint64_t cap = (uint64_t)sm_count() * 16;
  return (uint32_t)(b < 1 ? 1 : (b > cap ? cap : b));
}
}  // namespace

int skg_tokenize(const uint8_t* text, const int64_t* line_off, const int64_t* line_len, uint32_t n_lines,
                 uint64_t* tok_off, uint32_t* tok_len, uint32_t* tok_col, uint8_t* tok_flags, uint8_t* esc,
                 int32_t* kind, int32_t* ntok, uint32_t* err_col, void* stream) {
  if (n_lines == 0) return 0;
  if (!text || !line_off || !line_len || !tok_off || !tok_len || !tok_col || !tok_flags || !esc || !kind ||
      !ntok || !err_col)
    return -1;
  skg::tokenize_kernel<<<item_grid(n_lines), 256, 0, (cudaStream_t)stream>>>(
      text, line_off, line_len, n_lines, tok_off, tok_len, tok_col, tok_flags, esc, kind, ntok, err_col);
  return check(cudaGetLastError());
}

int skg_encode_modules(const int64_t* header, uint32_t n_mod, const int64_t* inst_base, const int64_t* opcode,
                       uint64_t n_inst, const int64_t* op_off, const uint32_t* ops, uint64_t n_ops,
                       uint32_t* out, uint64_t* err, void* stream) {
  if (n_mod == 0) return 0;
  if (!header || !inst_base || !op_off || !out || !err || n_inst >= 0xFFFFFFFFull) return -1;
  cudaStream_t s = (cudaStream_t)stream;
  auto* e = reinterpret_cast<unsigned long long*>(err);
  skg::encode_headers_kernel<<<item_grid(n_mod), 256, 0, s>>>(header, n_mod, inst_base, op_off, out, e);
  if (n_inst) skg::encode_insts_kernel<<<item_grid(n_inst), 256, 0, s>>>(opcode, op_off, n_inst, inst_base,
                                                                          n_mod, out, e);
  if (n_ops) skg::encode_operands_kernel<<<item_grid(n_ops), 256, 0, s>>>(ops, n_ops, op_off, (uint32_t)n_inst,
                                                                           inst_base, n_mod, out);
  return check(cudaGetLastError());
}

int skg_pack_strings(const uint8_t* bytes, const int64_t* off, const int64_t* len, const int64_t* word_off,
                     uint32_t n_str, uint64_t n_words, uint32_t* out, int32_t* bad, void* stream) {
  if (n_str == 0 || n_words == 0) return 0;
  if (!bytes || !off || !len || !word_off || !out || !bad) return -1;
  skg::pack_strings_kernel<<<item_grid(n_words), 256, 0, (cudaStream_t)stream>>>(bytes, off, len, word_off, n_str,
                                                                                  n_words, out, bad);
  return check(cudaGetLastError());
}

int skg_ctx_literals(const int64_t* width, const uint32_t* flags, const uint64_t* val, uint32_t n,
                     uint32_t* words, int32_t* nwords, int32_t* status, void* stream) {
  if (n == 0) return 0;
  if (!width || !flags || !val || !words || !nwords || !status) return -1;
  skg::ctx_literals_kernel<<<item_grid(n), 256, 0, (cudaStream_t)stream>>>(width, flags, val, n, words, nwords,
                                                                            status);
  return check(cudaGetLastError());
}

int skg_selftest_repr_f32(const skg_tables* t, uint64_t start, uint64_t count, uint64_t* fails,
                          uint32_t* first_fail, void* stream) {
  if (!t || !fails || !first_fail || start + count > (1ull << 32)) return -1;
  if (count == 0) return 0;
  skg::selftest_repr_f32_kernel<<<sm_count() * 8, 256, 0, (cudaStream_t)stream>>>(
      t->u, start, count, reinterpret_cast<unsigned long long*>(fails), first_fail);
  return check(cudaGetLastError());
}

}  // extern "C"
