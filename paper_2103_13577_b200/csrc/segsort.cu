// Per-row ascending sort of a CSR-shaped array (the np.unique / lexsort
// ordering of graphs.py:226,250 and the relabel's re-sorted rows):
// rows[rowstart[v] .. rowstart[v+1]) sorted into out, every row independent.
//
//   rows of 1          copied by the warp kernel
//   rows of 2..32      one warp, bitonic network in registers (shfl_xor)
//   rows of 33..2048   one warp, bitonic network in an 8 KB shared-memory slab
//   rows > 2048        one 256-thread block, LSD radix sort over 8-bit digits
//                      through global memory (stable per-tile ranking by
//                      match_any), `rows` used as the ping-pong buffer
//
// The warp kernel reads 32 rows' bounds per step (coalesced) and walks the
// rows of its class; the radix kernel takes the long rows from a list built
// by an append pass.  `rows` is clobbered (callers pass a scratch buffer).
#include <algorithm>

#include "bfb_device.cuh"
#include "bfb_internal.cuh"

namespace bfb {
namespace {

constexpr int kWarpMax = 2048;      // longest row sorted by one warp
constexpr int kSortWarps = 4;       // warps per block of the warp kernel (32 KB slab)
constexpr int kRadixBlock = 256;
constexpr int kRadixWarps = kRadixBlock / 32;
constexpr uint32_t kPad = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t bitonic32(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      x = (lower == up) ? min(x, y) : max(x, y);
    }
  }
  return x;
}

// bitonic sort of buf[0, p) (p a power of two <= kWarpMax) by one warp
__device__ __forceinline__ void bitonic_smem(uint32_t* buf, int p) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= p; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int lj = __ffs(j) - 1;
      for (int i = lane; i < (p >> 1); i += 32) {
        const int a = ((i >> lj) << (lj + 1)) + (i & (j - 1));
        const int b = a + j;
        const uint32_t x = buf[a], y = buf[b];
        const bool up = (a & k) == 0;
        if ((x > y) == up) {
          buf[a] = y;
          buf[b] = x;
        }
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kSortWarps * 32) k_sort_rows_warp(const int64_t* __restrict__ rowstart,
                                                                    int64_t n,
                                                                    const uint32_t* __restrict__ rows,
                                                                    uint32_t* __restrict__ out,
                                                                    uint32_t* big,
                                                                    unsigned long long* nbig) {
  __shared__ uint32_t slab[kSortWarps][kWarpMax];
  const int lane = threadIdx.x & 31;
  uint32_t* buf = slab[threadIdx.x >> 5];
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < n;
       base += nw * 32) {
    const int64_t v = base + lane;
    const int64_t b = v < n ? __ldg(rowstart + v) : 0;
    const int64_t d = v < n ? __ldg(rowstart + v + 1) - b : 0;
    if (d == 1) out[b] = __ldg(rows + b);
    if (d > kWarpMax) {
      const unsigned long long k = atomicAdd(nbig, 1ull);
      big[k] = (uint32_t)v;
    }
    for (unsigned m = __ballot_sync(0xffffffffu, d >= 2 && d <= kWarpMax); m; m &= m - 1) {
      const int j = __ffs(m) - 1;
      const int64_t rb = __shfl_sync(0xffffffffu, b, j);
      const int len = (int)__shfl_sync(0xffffffffu, d, j);
      if (len <= 32) {
        uint32_t x = lane < len ? __ldg(rows + rb + lane) : kPad;
        x = bitonic32(x);
        if (lane < len) out[rb + lane] = x;
      } else {
        const int p = 1 << (32 - __clz(len - 1));  // next power of two
        for (int i = lane; i < p; i += 32) buf[i] = i < len ? __ldg(rows + rb + i) : kPad;
        __syncwarp();
        bitonic_smem(buf, p);
        for (int i = lane; i < len; i += 32) out[rb + i] = buf[i];
        __syncwarp();
      }
    }
  }
}

// One long row per block at a time (rows from the list): LSD radix sort,
// `passes` 8-bit digits.  Pass q reads src and writes dst, alternating
// rows -> out -> rows ...; an even pass count ends with a copy into out.
__global__ void __launch_bounds__(kRadixBlock) k_sort_rows_radix(const int64_t* __restrict__ rowstart,
                                                                 uint32_t* rows, uint32_t* out,
                                                                 const uint32_t* __restrict__ big,
                                                                 const unsigned long long* nbig,
                                                                 int passes) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t run[256];
  __shared__ uint32_t wcnt[kRadixWarps][256];
  __shared__ int64_t wsum[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t cnt = (int64_t)*nbig;
  for (int64_t k = blockIdx.x; k < cnt; k += gridDim.x) {
    const uint32_t v = big[k];
    const int64_t b = rowstart[v];
    const int64_t d = rowstart[v + 1] - b;
    for (int q = 0; q < passes; ++q) {
      const uint32_t* src = (q & 1) ? out + b : rows + b;
      uint32_t* dst = (q & 1) ? rows + b : out + b;
      const int shift = 8 * q;
      hist[tid] = 0;
      __syncthreads();
      for (int64_t i = tid; i < d; i += kRadixBlock) atomicAdd(&hist[(src[i] >> shift) & 255u], 1u);
      __syncthreads();
      int64_t tot;
      const int64_t ex = block_exclusive_i64((int64_t)hist[tid], wsum, &tot);
      run[tid] = (uint32_t)ex;
      __syncthreads();
      for (int64_t t0 = 0; t0 < d; t0 += kRadixBlock) {
        const int64_t i = t0 + tid;
        const bool valid = i < d;
        const uint32_t key = valid ? src[i] : 0u;
        const int dig = valid ? (int)((key >> shift) & 255u) : 256;
        const unsigned peers = __match_any_sync(0xffffffffu, dig);
        const int rank = __popc(peers & lt);
#pragma unroll
        for (int w = 0; w < kRadixWarps; ++w) wcnt[w][tid] = 0;
        __syncthreads();
        if (valid && rank == 0) wcnt[warp][dig] = __popc(peers);
        __syncthreads();
        {  // thread = digit: exclusive prefix over the warps, continuing run[]
          uint32_t acc = run[tid];
#pragma unroll
          for (int w = 0; w < kRadixWarps; ++w) {
            const uint32_t c = wcnt[w][tid];
            wcnt[w][tid] = acc;
            acc += c;
          }
          run[tid] = acc;
        }
        __syncthreads();
        if (valid) dst[wcnt[warp][dig] + rank] = key;
        __syncthreads();
      }
    }
    if ((passes & 1) == 0)
      for (int64_t i = tid; i < d; i += kRadixBlock) out[b + i] = rows[b + i];
    __syncthreads();
  }
}

}  // namespace

int sort_rows(bfb_ctx* ctx, const int64_t* rowstart, int64_t n, int64_t total, uint32_t* rows,
              uint32_t* out, int64_t key_bound) {
  if (n <= 0 || total <= 0) return BFB_OK;
  cudaStream_t s = ctx->stream;
  const int sms = ctx->num_sms;
  DevBuf<uint32_t> big;
  DevBuf<unsigned long long> nbig;
  BFB_TRY(big.alloc(total / (kWarpMax + 1) + 1));
  BFB_TRY(nbig.alloc(1));
  BFB_CUDA(cudaMemsetAsync(nbig.p, 0, sizeof(unsigned long long), s));
  int occ = 1;
  BFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sort_rows_warp, kSortWarps * 32, 0));
  const int64_t want = (n + 32 * kSortWarps - 1) / (32 * kSortWarps);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * std::max(1, occ)));
  k_sort_rows_warp<<<grid, kSortWarps * 32, 0, s>>>(rowstart, n, rows, out, big.p, nbig.p);
  // key bits: the rows hold vertex ids < key_bound
  int bits = 1;
  while (bits < 32 && ((int64_t)1 << bits) < key_bound) ++bits;
  const int passes = (bits + 7) / 8;
  int occr = 1;
  BFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occr, k_sort_rows_radix, kRadixBlock, 0));
  k_sort_rows_radix<<<(unsigned)sms * std::max(1, occr), kRadixBlock, 0, s>>>(rowstart, rows, out,
                                                                              big.p, nbig.p, passes);
  BFB_CUDA(cudaGetLastError());
  BFB_CUDA(cudaStreamSynchronize(s));
  return BFB_OK;
}

}  // namespace bfb
