// One large module (config 3) spread over the whole GPU: grid-wide kernels per
// phase instead of one warp per module.  The boundary pass is the tiled one of
// skg_bigdecode.cuh (writing the words and instruction offsets straight into
// the module's scratch layout), and every later phase is a grid-stride loop
// over instructions / words / ids calling the same per-item device functions
// as the batch kernels (the grammar walk, inst_diags, ...).  Where the batch
// kernels resolve "first wins" / "last wins" per id by document-order warp
// chunks, these use atomicMin / atomicMax on the instruction index; ordered
// outputs use a device-wide exclusive scan.  Direct-indexed id tables only
// (ids below the header bound, i.e. the canonical case); anything else is
// reported back so the host runs the one-warp batch path instead.
#pragma once
#include <cstdint>

namespace skg {

// control words (workspace offset 0, 256 bytes)
enum : uint32_t {
  BC_STATUS = 0, BC_ERRPOS = 1, BC_COUNT = 2, BC_SWAP = 3,        // shared with BigDecode.result
  BC_FLAGS = 8, BC_NMM = 9, BC_BAD = 10, BC_OVER = 11, BC_ANYNAME = 12, BC_ARENA = 13,
  BC_TOTAL = 14, BC_SCAN = 16,                                     // BC_SCAN: u64 total of the last scan
  BC_NP0 = 18, BC_E1 = 19, BC_E2 = 20, BC_E3 = 21, BC_WIDTH = 22, BC_SUM = 24,   // BC_SUM: u64
  BC_DEPTH = 26,                                                   // closed-form name dedup: max tree depth
  BC_EFF = 32                                                      // eff: 8 x u64 at word 32
};
enum : uint32_t { BF_FN = 1, BF_CAP = 2, BF_EP = 4 };

// module scratch bytes for W words and header bound `bound` (direct tables)
__host__ __device__ inline size_t big_slot_bytes(uint32_t W, uint32_t bound) {
  const uint32_t I = W > 5 ? W - 5 : 1;
  return head_bytes(W) + inst_bytes(I) + word_bytes(W) + slot_bytes(bound, false) +
         work_need(bound, 0, 5ull * W) + spill_bytes(I) + 256;
}

// layout of the module scratch once I is known (one thread)
// min_table: direct id tables of at least this many slots (a module whose ids reach
// its header bound is redone with tables for every id below 2W + 64)
__global__ void big_setup(Mod* mp, uint8_t* slot, uint32_t W, uint32_t* ctl, uint32_t min_table) {
  Mod m;
  layout_head(m, slot, W);
  m.I = ctl[BC_COUNT];
  m.major = (m.w[1] >> 16) & 0xFF;
  m.minor = (m.w[1] >> 8) & 0xFF;
  m.gen = m.w[2];
  m.bound = m.w[3];
  m.schema = m.w[4];
  m.arena_need = 0;
  for (uint32_t k = BC_FLAGS; k < 64; ++k) ctl[k] = 0;
  ctl[BC_BAD] = NONE32; ctl[BC_E1] = NONE32; ctl[BC_E2] = NONE32; ctl[BC_E3] = NONE32;
  const uint32_t S = m.bound > min_table ? m.bound : min_table;
  if (S > 2 * m.W + 64) { ctl[BC_OVER] = 1; *mp = m; return; }   // not direct: host falls back
  layout_tables(m, true, S, 0, 0);
  m.fpc = nullptr;
  m.work_shared = false;
  const uint32_t Imax = W > 5 ? W - 5 : 1;
  m.spill = slot + big_slot_bytes(W, S) - 256 - spill_bytes(Imax);
  *m.fill = 0; *m.overflow = 0; *m.top_present = 0;
  *mp = m;
}

__global__ void big_init_tables(const Mod* mp) {
  const Mod m = *mp;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < m.S; s += gridDim.x * blockDim.x) {
    m.hdef[s] = NONE32; m.hname[s] = NONE32;
    m.hti[s] = 0; m.hvt[s] = 0; m.himp[s] = 0;      // last-wins tables hold index + 1 until big_fix
    m.hser[s] = NONE32;
    m.hA[s] = 0; m.hfl[s] = 0; m.hpres[s] = 0;
  }
}

// disasm.py:131-157 / validate.py:179-192 maps, first / last wins by index
__global__ void big_prescan(const Mod* mp, Tables T, uint32_t* ctl) {
  const Mod m = *mp;
  bool any_name = false, over = false;
  uint32_t arena = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m.I; i += gridDim.x * blockDim.x) {
    const uint32_t* ops = inst_ops(m, i);
    const uint32_t n = inst_nops(m, i);
    const uint32_t opc = inst_opcode(m, i);
    const uint32_t d = T.inst_of(opc);
    m.idef[i] = d == NONE32 ? NONE16 : (uint16_t)d;
    m.iflag[i] = 0;
    m.ierr[i] = 0;
    if (opc == 5 && n + 1 > 2) arena += 4 * (n - 1) + 1;   // OpName: sanitized name bound
    if (d == NONE32) continue;
    const uint32_t sp = T.special(d);
    auto mark = [&](uint32_t key) -> bool {
      if (key >= m.S) { over = true; return false; }
      m.hpres[key] = 1;
      return true;
    };
    if (((sp == SP_TYPEINT && n == 3) || (sp == SP_TYPEFLOAT && n >= 2)) && mark(ops[0]))
      atomicMax(&m.hti[ops[0]], i + 1);
    if (T.has_result(d) && T.has_rtype(d) && n >= 2 && mark(ops[1])) atomicMax(&m.hvt[ops[1]], i + 1);
    if ((sp == SP_EXTINSTIMPORT || sp == SP_NAME) && n >= 2) {
      uint32_t nbytes, next;
      if (string_span(ops, 1, n, nbytes, next)) {
        WalkErr e;
        if (string_utf8(ops, 1, nbytes, e) != U8_OK) {
          m.iflag[i] |= IF_PRESCAN_UTF8;
        } else if (mark(ops[0])) {
          if (sp == SP_EXTINSTIMPORT) atomicMax(&m.himp[ops[0]], i + 1);
          else { atomicMin(&m.hname[ops[0]], i); any_name = true; }
        }
      }
    }
    if (T.has_result(d)) {
      const uint32_t idx = T.has_rtype(d) ? 1 : 0;
      if (idx < n && mark(ops[idx])) atomicMin(&m.hdef[ops[idx]], i);
    }
  }
  if (any_name) atomicOr(&ctl[BC_ANYNAME], 1u);
  if (over) atomicOr(&ctl[BC_OVER], 1u);
  if (arena) atomicAdd(&ctl[BC_ARENA], arena);
}

__global__ void big_fix_tables(const Mod* mp) {
  const Mod m = *mp;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < m.S; s += gridDim.x * blockDim.x) {
    m.hti[s] = m.hti[s] ? m.hti[s] - 1 : NONE32;
    m.hvt[s] = m.hvt[s] ? m.hvt[s] - 1 : NONE32;
    m.himp[s] = m.himp[s] ? m.himp[s] - 1 : NONE32;
  }
}

// -- device-wide exclusive scan of uint32 (in place), total -> *total (u64) ----------
constexpr uint32_t BS_BLOCK = 1024;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t& total) {
  __shared__ uint32_t wsum[32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = lane < (blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, d);
      if (lane >= (uint32_t)d) s += y;
    }
    wsum[lane] = s;
  }
  __syncthreads();
  total = wsum[31];
  const uint32_t r = x - v + (warp ? wsum[warp - 1] : 0);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(BS_BLOCK) scan_blocks(uint32_t* a, uint32_t n, uint32_t* sums) {
  const uint32_t i = blockIdx.x * BS_BLOCK + threadIdx.x;
  uint32_t tot;
  const uint32_t v = i < n ? a[i] : 0;
  const uint32_t r = block_excl_scan(v, tot);
  if (i < n) a[i] = r;
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(BS_BLOCK) scan_top(uint32_t* sums, uint32_t nb, uint32_t* total_u64) {
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < nb; base += BS_BLOCK) {
    const uint32_t i = base + threadIdx.x;
    uint32_t tot;
    const uint32_t v = i < nb ? sums[i] : 0;
    const uint32_t r = block_excl_scan(v, tot);
    const uint32_t c0 = carry;
    if (i < nb) sums[i] = c0 + r;
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) { total_u64[0] = carry; total_u64[1] = 0; }
}

// 64-bit sum of n uint32 (the exclusive scans above are 32-bit: the host refuses totals
// that do not fit instead of letting the offsets wrap)
__global__ void sum_u64(const uint32_t* a, uint32_t n, unsigned long long* out) {
  unsigned long long v = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v += a[i];
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}

__global__ void __launch_bounds__(BS_BLOCK) scan_apply(uint32_t* a, uint32_t n, const uint32_t* sums) {
  const uint32_t i = blockIdx.x * BS_BLOCK + threadIdx.x;
  if (i < n) a[i] += sums[blockIdx.x];
}

// -- device-wide inclusive max-scan of int32 (in place), starting from `init` ------
__device__ __forceinline__ int32_t block_incl_max(int32_t v, int32_t& total) {
  __shared__ int32_t wmax[32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
    if (lane >= (uint32_t)d) x = max(x, y);
  }
  if (lane == 31) wmax[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t s = wmax[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t y = __shfl_up_sync(0xFFFFFFFFu, s, d);
      if (lane >= (uint32_t)d) s = max(s, y);
    }
    wmax[lane] = s;
  }
  __syncthreads();
  total = wmax[31];
  const int32_t r = warp ? max(x, wmax[warp - 1]) : x;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(BS_BLOCK) maxscan_blocks(int32_t* a, uint32_t n, int32_t* maxes) {
  const uint32_t i = blockIdx.x * BS_BLOCK + threadIdx.x;
  int32_t tot;
  const int32_t r = block_incl_max(i < n ? a[i] : INT32_MIN, tot);
  if (i < n) a[i] = r;
  if (threadIdx.x == 0) maxes[blockIdx.x] = tot;
}

// maxes[b] := max(init, maxes[0..b)) (exclusive); one thread (a few thousand blocks)
__global__ void maxscan_top(int32_t* maxes, uint32_t nb, int32_t init) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int32_t c = init;
  for (uint32_t b = 0; b < nb; ++b) {
    const int32_t v = maxes[b];
    maxes[b] = c;
    c = max(c, v);
  }
}

__global__ void __launch_bounds__(BS_BLOCK) maxscan_apply(int32_t* a, uint32_t n, const int32_t* maxes) {
  const uint32_t i = blockIdx.x * BS_BLOCK + threadIdx.x;
  if (i < n) a[i] = max(a[i], maxes[blockIdx.x]);
}

}  // namespace skg
