// Measurement kernel: the random-probe ceiling of phase 1.
//
// Top-down expansion is bound by its visited-bitmap probes -- one random
// 4-byte load per edge into an n/8-byte bitmap that lives in L2 -- not by
// the 4 bytes of streamed adjacency.  k_probe_peak issues only such loads
// (8 independent ones per thread per step, plain ld.global like the probe in
// k_expand_w) over a buffer of the bitmap's size, so probes/s here is the
// ceiling bench.py reports the expand kernel against (roofline "l2_probe").
#include <algorithm>
#include <cstdlib>

#include "bfb_internal.cuh"

namespace bfb {
namespace {

constexpr int kProbeItems = 8;

// kNC: the loads go through the non-coherent path (ld.global.nc, what a
// const __restrict__ pointer compiles to); the expand's probes are plain
// ld.global (the bitmap is written during the kernel), so the ceiling is
// measured with kNC = false.
template <bool kNC>
__global__ void __launch_bounds__(256) k_probe_peak(const uint32_t* buf, uint32_t nwords, int steps,
                                                    uint32_t* __restrict__ sink) {
  uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  uint32_t acc = 0;
  for (int s = 0; s < steps; ++s) {
    uint32_t w[kProbeItems];
#pragma unroll
    for (int k = 0; k < kProbeItems; ++k) {
      x ^= x << 13;
      x ^= x >> 7;
      x ^= x << 17;
      const uint32_t* p = buf + __umulhi((uint32_t)(x >> 32), nwords);  // uniform in [0, nwords)
      if (kNC) {
        w[k] = __ldg(p);
      } else {
        asm volatile("ld.global.u32 %0, [%1];" : "=r"(w[k]) : "l"(p));
      }
    }
#pragma unroll
    for (int k = 0; k < kProbeItems; ++k) acc ^= w[k];
  }
  if (acc == 0x12345678u) sink[0] = acc;  // keeps the loads live
}

__global__ void k_fill(uint32_t* buf, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    buf[i] = (uint32_t)(i * 2654435761u);
}

}  // namespace

int probe_peak(bfb_ctx* ctx, int64_t bytes, int64_t* probes_out, double* ms_out) {
  const uint32_t nwords = (uint32_t)std::min<int64_t>(std::max<int64_t>(1, bytes / 4), 0xFFFFFFFFll);
  DevBuf<uint32_t> buf, sink;
  BFB_TRY(buf.alloc(nwords));
  BFB_TRY(sink.alloc(1));
  cudaStream_t s = ctx->stream;
  k_fill<<<ctx->num_sms * 8, 256, 0, s>>>(buf.p, nwords);
  const int grid = ctx->num_sms * 8, steps = 256;
  const char* nc_env = std::getenv("BFB_PROBE_NC");  // developer switch: the .nc path instead
  auto kernel = nc_env && nc_env[0] == '1' ? k_probe_peak<true> : k_probe_peak<false>;
  kernel<<<grid, 256, 0, s>>>(buf.p, nwords, steps, sink.p);  // warm L2
  cudaEvent_t e0, e1;
  BFB_CUDA(cudaEventCreate(&e0));
  BFB_CUDA(cudaEventCreate(&e1));
  BFB_CUDA(cudaEventRecord(e0, s));
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kernel<<<grid, 256, 0, s>>>(buf.p, nwords, steps, sink.p);
  BFB_CUDA(cudaEventRecord(e1, s));
  BFB_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  BFB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  BFB_CUDA(cudaGetLastError());
  *probes_out = (int64_t)reps * grid * 256 * (int64_t)steps * kProbeItems;
  *ms_out = ms;
  return BFB_OK;
}

}  // namespace bfb
