// Device-side helpers shared by the kernels (warp/block scans, cache hints).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bfb {

__device__ __forceinline__ int64_t warp_inclusive_i64(int64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Block-wide sum; `red` holds blockDim.x/32 entries.  Result valid in all threads.
__device__ __forceinline__ int64_t block_sum_i64(int64_t v, int64_t* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum_i64(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int64_t t = (lane < nw) ? red[lane] : 0;
  t = warp_sum_i64(t);
  __syncthreads();
  return t;
}

// Block-wide exclusive scan; `wsum` holds 33 entries.  *total = block sum.
__device__ __forceinline__ int64_t block_exclusive_i64(int64_t v, int64_t* wsum, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t inc = warp_inclusive_i64(v);
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < nw ? wsum[lane] : 0;
    int64_t wi = warp_inclusive_i64(w);
    if (lane < nw) wsum[lane] = wi - w;
    if (lane == 31) wsum[32] = wi;
  }
  __syncthreads();
  int64_t off = wsum[warp];
  *total = wsum[32];
  int64_t res = off + inc - v;
  __syncthreads();
  return res;
}

// Streaming read (evict-first): adjacency is touched once per BFS.
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) { return __ldcs(p); }

}  // namespace bfb
