// Device-wide exclusive scans used by the graph build (degree -> offsets,
// flag words -> compaction positions).  Reduce-then-scan over 4096-item
// tiles; int64 results so |E| > 2^32 works.
#include "bfb_internal.cuh"
#include "bfb_device.cuh"

namespace bfb {
namespace {

constexpr int kBlock = 256;
constexpr int kItems = 16;
constexpr int64_t kTile = (int64_t)kBlock * kItems;

struct LoadU32 {
  const uint32_t* p;
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return (int64_t)p[i]; }
};
struct LoadPopc {
  const uint32_t* p;
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return (int64_t)__popc(p[i]); }
};

template <class L>
__global__ void __launch_bounds__(kBlock) k_tile_reduce(L load, int64_t n, int64_t* tile_sums) {
  int64_t base = (int64_t)blockIdx.x * kTile;
  int64_t acc = 0;
#pragma unroll 4
  for (int k = 0; k < kItems; ++k) {
    int64_t i = base + (int64_t)k * kBlock + threadIdx.x;
    if (i < n) acc += load(i);
  }
  __shared__ int64_t red[kBlock / 32];
  acc = block_sum_i64(acc, red);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = acc;
}

// Single block: exclusive scan of tile sums in place.
__global__ void __launch_bounds__(1024) k_tiles_scan(int64_t* sums, int64_t ntiles) {
  __shared__ int64_t wsum[33];
  __shared__ int64_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int64_t base = 0; base < ntiles; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < ntiles ? sums[i] : 0;
    int64_t total;
    int64_t ex = block_exclusive_i64(v, wsum, &total);
    int64_t carry = carry_s;
    if (i < ntiles) sums[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + total;
    __syncthreads();
  }
}

template <class L>
__global__ void __launch_bounds__(kBlock) k_tile_apply(L load, int64_t n, const int64_t* tile_pref,
                                                       int64_t* out) {
  int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
  int64_t v[kItems];
  int64_t acc = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    int64_t i = base + k;
    v[k] = i < n ? load(i) : 0;
    acc += v[k];
  }
  __shared__ int64_t wsum[33];
  int64_t total;
  int64_t ex = block_exclusive_i64(acc, wsum, &total) + tile_pref[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    int64_t i = base + k;
    if (i < n) out[i] = ex;
    ex += v[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) out[n] = ex;
}

template <class L>
int scan_impl(L load, int64_t n, int64_t* out, int64_t* tmp, cudaStream_t s) {
  int64_t ntiles = (n + kTile - 1) / kTile;
  if (ntiles == 0) {
    BFB_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
    return BFB_OK;
  }
  k_tile_reduce<<<(unsigned)ntiles, kBlock, 0, s>>>(load, n, tmp);
  k_tiles_scan<<<1, 1024, 0, s>>>(tmp, ntiles);
  k_tile_apply<<<(unsigned)ntiles, kBlock, 0, s>>>(load, n, tmp, out);
  BFB_CUDA(cudaGetLastError());
  return BFB_OK;
}

}  // namespace

size_t scan_tmp_words(int64_t n) { return (size_t)((n + kTile - 1) / kTile + 1); }

int scan_u32_to_i64(const uint32_t* in, int64_t n, int64_t* out, int64_t* tmp, cudaStream_t s) {
  return scan_impl(LoadU32{in}, n, out, tmp, s);
}

int scan_popc_to_i64(const uint32_t* words, int64_t n, int64_t* out, int64_t* tmp,
                     cudaStream_t s) {
  return scan_impl(LoadPopc{words}, n, out, tmp, s);
}

}  // namespace bfb
