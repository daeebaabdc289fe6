// Instruction-boundary pass for ONE large module (decode_module on config-3
// sizes; reference codec.py:199-231), parallel over tiles of the word stream.
//
// The boundary chain p -> p + (w[p] >> 16) is a linked list, not a prefix sum,
// so it is split speculatively (hard part 1):
//   1. big_copy      byte-order-normalised words, grid-stride
//   2. tile_spec     per tile (thread per tile): walk the chains from the tile's
//                    first BD_K plausible starts (word count >= 1, opcode <= the
//                    grammar's largest) to the tile end, marking the positions
//                    each visits (a later chain stops where it joins an earlier
//                    one) -> per chain the exit X and the first error on it
//   3. tile_land / tile_jump / tile_path: the tiles linked in parallel -- every
//                    (tile, chain) node's successor is the chain its exit lands on
//                    (the exact walk from the exit to the next marked position: from
//                    there that speculative chain IS the true chain, so its exit and
//                    recorded first error are the true ones); the successor map is
//                    doubled and thread d reads the d-th node of the true chain.  A walk
//                    that crosses 64 K words unmarked sends the whole link to tile_link
//                    (one warp, tiles in order, the same rule sequentially).
//   4. tile_count    per tile: instructions on the true chain in the tile
//   5. tile_scan     exclusive scan of the counts (one CTA)
//   6. tile_write    per tile: the instruction offsets
// Errors are the first wc == 0 / overrun on the true chain, with the word
// position and message the reference raises.
#pragma once
#include <cstdint>

namespace skg {

#ifndef SKG_BD_TILE
#define SKG_BD_TILE 1024   // 4096 measured 2 ms slower per call (fewer threads in the per-tile passes)
#endif
constexpr uint32_t BD_TILE = SKG_BD_TILE;   // words per tile
constexpr uint32_t BD_K = 4;                // speculative chains per tile
constexpr uint32_t BD_SCAN = 64;            // words searched for plausible starts
constexpr uint32_t BD_NONE = 0xFFFFFFFFu;

struct BigDecode {
  const uint8_t* src;
  uint32_t W;
  uint32_t* words;           // W normalised words
  uint32_t ntiles;
  uint8_t* chain;            // ntiles * BD_TILE: 1 + speculative chain visiting the word, or 0
  uint32_t* spec_exit;       // per tile and chain: first chain position >= tile end (BD_NONE: error)
  uint32_t* spec_err;        // per tile and chain: first error position on the chain (BD_NONE: none)
  uint32_t* spec_errc;       // per tile and chain: ST_CORRUPT / ST_TRUNCATED
  uint32_t max_opcode;       // plausibility filter for speculative starts (0xFFFF: none)
  uint32_t* entry;           // per tile: first true-chain position in the tile (BD_NONE: none)
  // parallel link (tile_land / tile_jump / tile_path): one node per (tile, chain)
  uint32_t* next;            // node -> the node the true chain continues on, or BD_TERM | node
  uint32_t* tpos;            // node: where the walk into the next tile ended (error position)
  uint32_t* tcode;           // node: terminal kind (TK_END / TK_RAW / an error status)
  uint32_t* jump;            // levels x nodes: next composed 2^r times
  uint32_t levels;
  uint32_t* count;           // per tile: instructions, then exclusive offsets
  uint32_t* result;          // [0] status, [1] error position, [2] instruction count, [3] byte swap
  uint32_t* inst_off;
  uint64_t nbytes;
};

// length and magic checks (codec.py:199-216); result[0] gates every later kernel
__global__ void big_prologue(BigDecode b) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t st = ST_OK, swap = 0;
  if (b.nbytes % 4 != 0 || b.nbytes < 20) {
    st = ST_TRUNCATED;
  } else {
    const uint8_t* p = b.src;
    const uint32_t w0 = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
    if (w0 != MAGIC) {
      if (__byte_perm(w0, 0, 0x0123) == MAGIC) swap = 1; else { st = ST_NOTSPIRV; b.result[1] = w0; }
    }
  }
  b.result[0] = st;
  b.result[2] = 0;
  b.result[3] = swap;
}

__global__ void big_copy(BigDecode b) {
  if (b.result[0] != ST_OK) return;
  const bool swap = b.result[3] != 0;
  const uint32_t* s = reinterpret_cast<const uint32_t*>(b.src);
  const bool aligned = (reinterpret_cast<uintptr_t>(b.src) & 3) == 0;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < b.W; k += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v;
    if (aligned) {
      v = __ldcs(s + k);
    } else {
      const uint8_t* p = b.src + 4 * k;
      v = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
    }
    b.words[k] = swap ? __byte_perm(v, 0, 0x0123) : v;
  }
}

__global__ void tile_spec(BigDecode b) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= b.ntiles || b.result[0] != ST_OK) return;
  const uint32_t lo = t * BD_TILE, hi = min(lo + BD_TILE, b.W);
  uint8_t* cm = b.chain + (uint64_t)t * BD_TILE;   // zeroed by the host (cudaMemsetAsync)
  uint32_t* ex = b.spec_exit + (uint64_t)t * BD_K;
  uint32_t* er = b.spec_err + (uint64_t)t * BD_K;
  uint32_t* ec = b.spec_errc + (uint64_t)t * BD_K;
  uint32_t s = t == 0 ? 5 : lo;   // tile 0: the true chain itself
  for (uint32_t k = 0; k < BD_K; ++k) {
    ex[k] = BD_NONE; er[k] = BD_NONE; ec[k] = 0;
    if (t != 0 || k != 0) {       // next plausible start
      while (s < hi && s < lo + BD_SCAN) {
        const uint32_t x = b.words[s];
        if ((x >> 16) != 0 && (x & 0xFFFF) <= b.max_opcode && cm[s - lo] == 0) break;
        ++s;
      }
      if (s >= hi || s >= lo + BD_SCAN) break;
    }
    uint32_t p = s;
    ++s;
    while (p < hi) {
      const uint32_t c = cm[p - lo];
      if (c) { ex[k] = ex[c - 1]; er[k] = er[c - 1]; ec[k] = ec[c - 1]; break; }   // joins chain c-1
      cm[p - lo] = (uint8_t)(k + 1);
      const uint32_t wc = b.words[p] >> 16;
      if (wc == 0) { er[k] = p; ec[k] = ST_CORRUPT; break; }
      if ((uint64_t)p + wc > b.W) { er[k] = p; ec[k] = ST_TRUNCATED; break; }
      p += wc;
    }
    if (p >= hi) ex[k] = p;
    if (t == 0) break;
  }
}

// One warp.  The walk is sequential over tiles, so its cost is latency: the
// lanes first load 32 tiles' speculative results (exits, errors, and the first
// 16 bytes of their chain maps, where an entry nearly always lands) in one
// round, then every lane runs the same walk, taking tile j's data from lane j by
// shuffles; only an entry past those 16 bytes, or an unmarked one, reads memory.
__device__ __forceinline__ void tile_link_body(BigDecode& b);
__global__ void tile_link(BigDecode b) { tile_link_body(b); }
__global__ void tile_link_if_raw(BigDecode b) {
  if (b.result[4] == 0) return;   // the parallel link was complete
  if (threadIdx.x < 32) b.result[0] = ST_OK;   // tile_path may have set nothing else
  __syncwarp();
  tile_link_body(b);
}
__device__ __forceinline__ void tile_link_body(BigDecode& b) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  if (b.result[0] != ST_OK) return;   // (the same value for every lane)
  const uint32_t lane = threadIdx.x;
  uint32_t e = 5, status = ST_OK, errpos = 0;
  for (uint32_t t0 = 0; t0 < b.ntiles; t0 += 32) {
    const uint32_t tl = t0 + lane;
    uint32_t ex[BD_K], er[BD_K], ec[BD_K];
    uint4 c16 = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (uint32_t k = 0; k < BD_K; ++k) { ex[k] = BD_NONE; er[k] = BD_NONE; ec[k] = 0; }
    if (tl < b.ntiles) {
#pragma unroll
      for (uint32_t k = 0; k < BD_K; ++k) {
        ex[k] = b.spec_exit[(uint64_t)tl * BD_K + k];
        er[k] = b.spec_err[(uint64_t)tl * BD_K + k];
        ec[k] = b.spec_errc[(uint64_t)tl * BD_K + k];
      }
      c16 = *reinterpret_cast<const uint4*>(b.chain + (uint64_t)tl * BD_TILE);
    }
    const uint32_t nt = min(32u, b.ntiles - t0);
#pragma unroll 1
    for (uint32_t j = 0; j < nt; ++j) {
      const uint32_t t = t0 + j;
      const uint32_t lo = t * BD_TILE, hi = min(lo + BD_TILE, b.W);
      const uint32_t w0 = __shfl_sync(0xFFFFFFFFu, c16.x, j), w1 = __shfl_sync(0xFFFFFFFFu, c16.y, j);
      const uint32_t w2 = __shfl_sync(0xFFFFFFFFu, c16.z, j), w3 = __shfl_sync(0xFFFFFFFFu, c16.w, j);
      if (status != ST_OK || e >= hi) { if (lane == 0) b.entry[t] = BD_NONE; continue; }
      if (lane == 0) b.entry[t] = e;
      const uint8_t* cm = b.chain + (uint64_t)t * BD_TILE;
      uint32_t p = e, c = 0;
#pragma unroll 1
      while (p < hi) {
        const uint32_t o = p - lo;
        if (o < 16) {
          const uint32_t w = o < 8 ? (o < 4 ? w0 : w1) : (o < 12 ? w2 : w3);
          c = (w >> (8 * (o & 3))) & 0xFF;
        } else {
          c = cm[o];
        }
        if (c) break;
        const uint32_t wc = b.words[p] >> 16;
        if (wc == 0) { status = ST_CORRUPT; errpos = p; break; }
        if ((uint64_t)p + wc > b.W) { status = ST_TRUNCATED; errpos = p; break; }
        p += wc;
      }
      // chain c - 1's exit / first error, from lane j (selected without a dynamic register index)
      const uint32_t kk = c ? c - 1 : 0;
      uint32_t sx = ex[0], sr = er[0], sc = ec[0];
#pragma unroll
      for (uint32_t k = 1; k < BD_K; ++k) if (kk == k) { sx = ex[k]; sr = er[k]; sc = ec[k]; }
      sx = __shfl_sync(0xFFFFFFFFu, sx, j);
      sr = __shfl_sync(0xFFFFFFFFu, sr, j);
      sc = __shfl_sync(0xFFFFFFFFu, sc, j);
      if (status != ST_OK) continue;
      if (c) {   // on speculative chain c - 1 from here on
        if (sr != BD_NONE) { status = sc; errpos = sr; continue; }
        e = sx;
      } else {
        e = p;
      }
    }
  }
  if (lane == 0) { b.result[0] = status; b.result[1] = errpos; }
}

// ---------------------------------------------------------------------------
// Parallel link.  Node n = 4 t + k stands for "the true chain follows speculative
// chain k of tile t".  tile_land computes each node's successor independently:
// chain k's first error makes the node terminal (that is the true chain's first
// error: it lies at or after any point where the true chain joins chain k); its
// exit e (the first position past tile t, possibly several tiles on) is walked
// by the exact rule in e's tile until it lands on a marked position (node of that
// tile's chain), reaches the end of the stream (terminal END), hits a word count
// 0 / overrun (terminal error) or leaves the tile unmarked (terminal RAW: the
// sequential tile_link then does the whole link).  tile_jump composes the
// successor map by doubling; tile_path gives thread d the d-th node of the chain
// from node 0 (bits of d through the doubled maps), which sets that tile's entry
// (the exit of node d-1) and, for the first terminal, the status.
constexpr uint32_t BD_TERM = 0x80000000u;
constexpr uint32_t TK_END = 100, TK_RAW = 101;

// tiles a successor walk may cross before giving up (TK_RAW): 64 K words, one maximal instruction
constexpr uint32_t BD_MAXHOP = 65536 / BD_TILE;

__global__ void tile_land(BigDecode b) {
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= b.ntiles * BD_K || b.result[0] != ST_OK) return;
  const uint32_t er = b.spec_err[n], ex = b.spec_exit[n];
  uint32_t nxt = BD_TERM | n, code = TK_RAW, pos = 0;
  if (er != BD_NONE) {
    code = b.spec_errc[n]; pos = er;
  } else if (ex != BD_NONE) {
    // the exact walk from the exit until it meets a marked position (chain maps are
    // contiguous: chain[p] for absolute p), the stream end, or an error
    uint32_t p = ex, t0 = ex / BD_TILE;
    code = TK_END;
    while (p < b.W) {
      const uint32_t c = b.chain[p];
      if (c) { nxt = BD_K * (p / BD_TILE) + c - 1; code = 0; break; }
      const uint32_t wc = b.words[p] >> 16;
      if (wc == 0) { code = ST_CORRUPT; pos = p; break; }
      if ((uint64_t)p + wc > b.W) { code = ST_TRUNCATED; pos = p; break; }
      p += wc;
      if (p / BD_TILE > t0 + BD_MAXHOP) { code = TK_RAW; break; }
    }
  }
  b.next[n] = nxt;
  b.jump[n] = nxt;
  b.tpos[n] = pos;
  b.tcode[n] = code;
}

// level r from level r - 1 (a terminal maps to itself)
__global__ void tile_jump(BigDecode b, uint32_t r) {
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t N = b.ntiles * BD_K;
  if (n >= N || b.result[0] != ST_OK) return;
  const uint32_t* prev = b.jump + (uint64_t)(r - 1) * N;
  const uint32_t x = prev[n];
  b.jump[(uint64_t)r * N + n] = (x & BD_TERM) ? x : prev[x];
}

__device__ __forceinline__ uint32_t path_node(const BigDecode& b, uint32_t d) {
  const uint32_t N = b.ntiles * BD_K;
  uint32_t x = 0;
  for (uint32_t r = 0; d && r < b.levels; ++r, d >>= 1)
    if ((d & 1) && !(x & BD_TERM)) x = b.jump[(uint64_t)r * N + x];
  return x;
}

// the tiles a true-chain walk from p enters before it meets a marked position or the
// stream end: each gets its first position as entry (tile_land validated the walk)
__device__ __forceinline__ void path_entries(const BigDecode& b, uint32_t p) {
  uint32_t last = BD_NONE;
  while (p < b.W) {
    const uint32_t t = p / BD_TILE;
    if (t != last) { b.entry[t] = p; last = t; }
    if (b.chain[p]) return;
    p += b.words[p] >> 16;
  }
}

// thread d: the d-th node on the true chain (d <= ntiles: at most one node per tile)
__global__ void tile_path(BigDecode b) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d > b.ntiles || b.result[0] != ST_OK) return;
  const uint32_t x = path_node(b, d);
  const uint32_t pv = d ? path_node(b, d - 1) : BD_TERM;
  if (!(x & BD_TERM)) {   // node x: the walk into its tile from the previous node's exit
    if (d == 0) b.entry[0] = 5u;
    else path_entries(b, b.spec_exit[pv]);
    return;
  }
  if (d && (pv & BD_TERM)) return;   // not the first terminal
  const uint32_t n = x & ~BD_TERM;   // the node whose successor is terminal
  const uint32_t code = b.tcode[n];
  if (code == TK_END) {              // the chain ends with the stream: the tiles it still enters
    if (b.spec_exit[n] != BD_NONE) path_entries(b, b.spec_exit[n]);
    return;
  }
  if (code == TK_RAW) { b.result[4] = 1; return; }   // the sequential link decides
  b.result[0] = code;
  b.result[1] = b.tpos[n];
}

// entries default to BD_NONE before the path sets the tiles it visits
__global__ void tile_entry_init(BigDecode b) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < b.ntiles) b.entry[t] = BD_NONE;
  if (t == 0) b.result[4] = 0;
}

// the sequential link only when the parallel one met an unmarked exit (TK_RAW)
__global__ void tile_link_if_raw(BigDecode b);

__global__ void tile_count(BigDecode b) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= b.ntiles) return;
  uint32_t c = 0;
  if (b.result[0] == ST_OK && b.entry[t] != BD_NONE) {
    const uint32_t hi = min(t * BD_TILE + BD_TILE, b.W);
    for (uint32_t p = b.entry[t]; p < hi; p += b.words[p] >> 16) ++c;
  }
  b.count[t] = c;
}

// exclusive scan of count[0..ntiles) in place; total into result[2] (one CTA of 1024)
__global__ void __launch_bounds__(1024) tile_scan(BigDecode b) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t base = 0; base < b.ntiles; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < b.ntiles ? b.count[i] : 0;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
      if (lane >= (uint32_t)d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t s = wsum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, d);
        if (lane >= (uint32_t)d) s += y;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    const uint32_t c0 = carry;
    if (i < b.ntiles) b.count[i] = c0 + x - v + (warp ? wsum[warp - 1] : 0);
    __syncthreads();
    if (threadIdx.x == 1023) carry = c0 + wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) b.result[2] = carry;
}

__global__ void tile_write(BigDecode b) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= b.ntiles || b.result[0] != ST_OK || b.entry[t] == BD_NONE) return;
  const uint32_t hi = min(t * BD_TILE + BD_TILE, b.W);
  uint32_t k = b.count[t];
  for (uint32_t p = b.entry[t]; p < hi; p += b.words[p] >> 16) b.inst_off[k++] = p;
}

// header, count, status and the exact error text (codec.py:82-89, 199-231)
__global__ void big_epilogue(BigDecode b, uint32_t* header, uint32_t* inst_count, int32_t* status, ErrRec* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const uint32_t st = b.result[0];
  *status = (int32_t)st;
  *inst_count = st == ST_OK ? b.result[2] : 0;
  if (st == ST_OK) {
    header[0] = (b.words[1] >> 16) & 0xFF;
    header[1] = (b.words[1] >> 8) & 0xFF;
    header[2] = b.words[2];
    header[3] = b.words[3];
    header[4] = b.words[4];
    return;
  }
  if (!err) return;
  ErrWriter ew{err};
  if (st == ST_TRUNCATED && (b.nbytes % 4 != 0 || b.nbytes < 20)) {
    put_u64(ew, b.nbytes); put_cstr(ew, " bytes is not a whole word stream of at least 5 words");
  } else if (st == ST_NOTSPIRV) {
    put_cstr(ew, "magic word 0x"); put_hex8_upper(ew, b.result[1]); put_cstr(ew, " is not SPIR-V");
  } else {
    put_cstr(ew, "instruction at word "); put_u64(ew, b.result[1]);
    put_cstr(ew, st == ST_CORRUPT ? " has word count 0" : " runs past the end of the stream");
  }
  err->module = 0; err->cls = (int32_t)st; err->len = ew.n;
}

}  // namespace skg
