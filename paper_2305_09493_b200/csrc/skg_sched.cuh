// Module scheduling order: a device counting sort of module indices by size,
// largest first.  The phase-synchronised kernels hand consecutive tickets to
// the warps of one CTA, and a CTA waits at every phase barrier for its slowest
// module; sorting by size makes the modules of one CTA similar in size (and
// puts the largest first, so the tail of the grid is filled by small ones).
// Only the processing order changes: outputs are addressed by module index.
#pragma once
#include <cstdint>

namespace skg {

constexpr uint32_t SCHED_BUCKETS = 4096;
constexpr uint32_t SCHED_PER_THREAD = SCHED_BUCKETS / 1024;   // buckets per thread of sched_scan
constexpr uint32_t SCHED_PERM_OFF = 8 * SCHED_BUCKETS;         // bytes: hist[], cursor[], then perm[]
constexpr uint32_t SCHED_SHIFT = 6;        // 64-byte size classes

// Region-major order (regions > 1): the modules are cut into `regions` contiguous
// index ranges, processed one range after the other, each largest first (in
// SCHED_BUCKETS/regions size classes of 2^shift bytes).  The modules in flight at any time
// then come from one range of the input instead of from all of it.  Over the
// bench's 1M-module (2.7 GB) batch: disassembly 133.1 -> 115.8 ms with 16 regions
// of 64 128-byte classes (4: 127.2, 8: 119.6, 32: 118.4, 64: 119.7 ms; 16 regions of
// 64 64-byte classes, i.e. everything over 4 KB in one class: 121.6 ms), 115.2 ms
// with 4096 buckets (16 regions of 256 64-byte classes); the fused
// disassemble+validate pass 156.5 -> 135.4 ms.
// Used where the modules arrive in caller order (disassembler, fused pass).
struct SchedKey {
  uint32_t regions, n, shift;
};

__device__ __forceinline__ uint32_t sched_bucket(int64_t len, uint32_t i, SchedKey k) {
  const uint64_t c = len <= 0 ? 0 : ((uint64_t)len >> k.shift);
  const uint32_t per = SCHED_BUCKETS / k.regions;
  const uint32_t r = (uint32_t)(((uint64_t)i * k.regions) / k.n);
  return r * per + per - 1 - (uint32_t)(c < per - 1 ? c : per - 1);
}

// hist[b] += number of modules in bucket b
__global__ void __launch_bounds__(1024) sched_hist(const int64_t* len, uint32_t stride, uint32_t n,
                                                   uint32_t* hist, SchedKey k) {
  __shared__ uint32_t h[SCHED_BUCKETS];
  for (uint32_t b = threadIdx.x; b < SCHED_BUCKETS; b += blockDim.x) h[b] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(&h[sched_bucket(len[(size_t)i * stride], i, k)], 1u);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < SCHED_BUCKETS; b += blockDim.x)
    if (h[b]) atomicAdd(&hist[b], h[b]);
}

// cursor = exclusive scan of hist (one CTA of 1024 threads, SCHED_PER_THREAD
// consecutive buckets each)
__global__ void __launch_bounds__(1024) sched_scan(const uint32_t* hist, uint32_t* cursor) {
  __shared__ uint32_t wsum[32];
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint32_t v[SCHED_PER_THREAD], own = 0;
#pragma unroll
  for (uint32_t j = 0; j < SCHED_PER_THREAD; ++j) { v[j] = hist[t * SCHED_PER_THREAD + j]; own += v[j]; }
  uint32_t x = own;
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
  uint32_t c = x - own + (warp ? wsum[warp - 1] : 0);
#pragma unroll
  for (uint32_t j = 0; j < SCHED_PER_THREAD; ++j) { cursor[t * SCHED_PER_THREAD + j] = c; c += v[j]; }
}

// perm[cursor[b]++] = i; each CTA owns a contiguous chunk of module indices
__global__ void __launch_bounds__(1024) sched_scatter(const int64_t* len, uint32_t stride, uint32_t n,
                                                      uint32_t* cursor, uint32_t* perm, SchedKey k) {
  __shared__ uint32_t h[SCHED_BUCKETS];
  const uint32_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const uint32_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  for (uint32_t b = threadIdx.x; b < SCHED_BUCKETS; b += blockDim.x) h[b] = 0;
  __syncthreads();
  for (uint32_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&h[sched_bucket(len[(size_t)i * stride], i, k)], 1u);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < SCHED_BUCKETS; b += blockDim.x)
    if (h[b]) h[b] = atomicAdd(&cursor[b], h[b]);
  __syncthreads();
  for (uint32_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint32_t b = sched_bucket(len[(size_t)i * stride], i, k);
    perm[atomicAdd(&h[b], 1u)] = i;
  }
}

}  // namespace skg
