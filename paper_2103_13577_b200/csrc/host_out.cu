// Result read-out: d_local (levels) and parents from HBM into the caller's
// host arrays.
//
// The reference hands node 0's DistanceArray back as uint32 per vertex
// (engine.py `run`), i.e. 2 GB at scale 29, and at PCIe
// speed that copy costs as much as the BFS itself.  Levels are small
// integers, so the device packs them first -- 4 bits per vertex when the BFS
// has at most 15 levels (15 = UNREACHED), 8 bits when it has at most 255,
// else the uint32 array as is -- and the packed array crosses PCIe in chunks
// while host threads widen each landed chunk into the caller's uint32 array
// (non-temporal stores, no read-for-ownership).  Parents (uint32 on device,
// int64 with -1 in the reference's output) take the same pipeline.
#include <emmintrin.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>

#include "bfb_internal.cuh"

namespace bfb {
namespace {

constexpr uint32_t kNoLevel = 0xFFFFFFFFu;

// Eight vertices per thread: two 16-byte loads, one packed word.
__global__ void k_pack_levels4(const uint32_t* __restrict__ level, int64_t n,
                               uint32_t* __restrict__ out) {
  const int64_t nw = (n + 7) / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = i * 8;
    uint32_t v[8];
    if (u + 8 <= n) {
      const uint4 a = __ldcs(reinterpret_cast<const uint4*>(level + u));
      const uint4 b = __ldcs(reinterpret_cast<const uint4*>(level + u) + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = u + j < n ? level[u + j] : kNoLevel;
    }
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) w |= min(v[j], 15u) << (4 * j);
    out[i] = w;
  }
}

// Four vertices per thread: one 16-byte load, one packed word.
__global__ void k_pack_levels8(const uint32_t* __restrict__ level, int64_t n,
                               uint32_t* __restrict__ out) {
  const int64_t nw = (n + 3) / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = i * 4;
    uint32_t v[4];
    if (u + 4 <= n) {
      const uint4 a = __ldcs(reinterpret_cast<const uint4*>(level + u));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = u + j < n ? level[u + j] : kNoLevel;
    }
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) w |= min(v[j], 255u) << (8 * j);
    out[i] = w;
  }
}

// Host threads for the widening: BFB_HOST_THREADS, else the CPUs this
// process may run on, at most 32.
int host_threads() {
  if (const char* e = std::getenv("BFB_HOST_THREADS")) {
    const int t = std::atoi(e);
    if (t > 0) return std::min(t, 64);
  }
  cpu_set_t set;
  int t = 1;
  if (sched_getaffinity(0, sizeof(set), &set) == 0) t = CPU_COUNT(&set);
  return std::max(1, std::min(t, 32));
}

uint64_t g_nib[256];  // packed byte -> two uint32 levels (low nibble first)
std::once_flag g_nib_once;

inline uint32_t widen4(uint32_t x) { return x == 15u ? kNoLevel : x; }

void init_tables() {
  std::call_once(g_nib_once, [] {
    for (int b = 0; b < 256; ++b)
      g_nib[b] = (uint64_t)widen4(b & 15) | ((uint64_t)widen4(b >> 4) << 32);
  });
}

// Elements [e0, e1) of a nibble-packed array into out (e0 even).
void widen_nibbles(const uint8_t* in, int64_t e0, int64_t e1, uint32_t* out) {
  int64_t e = e0;
  auto one = [&](int64_t i) { out[i] = widen4((in[i >> 1] >> ((i & 1) * 4)) & 15u); };
  while (e < e1 && ((reinterpret_cast<uintptr_t>(out + e) & 15) || (e & 1))) one(e++);
  for (; e + 4 <= e1; e += 4) {
    const uint8_t* b = in + (e >> 1);
    _mm_stream_si128(reinterpret_cast<__m128i*>(out + e),
                     _mm_set_epi64x((long long)g_nib[b[1]], (long long)g_nib[b[0]]));
  }
  for (; e < e1; ++e) one(e);
}

// Elements [e0, e1) of a byte-packed array (255 = UNREACHED).
void widen_bytes(const uint8_t* in, int64_t e0, int64_t e1, uint32_t* out) {
  int64_t e = e0;
  auto one = [&](int64_t i) { out[i] = in[i] == 255 ? kNoLevel : in[i]; };
  while (e < e1 && (reinterpret_cast<uintptr_t>(out + e) & 15)) one(e++);
  const __m128i zero = _mm_setzero_si128(), ff = _mm_set1_epi32(255);
  for (; e + 4 <= e1; e += 4) {
    uint32_t w;
    std::memcpy(&w, in + e, 4);
    __m128i x = _mm_unpacklo_epi16(_mm_unpacklo_epi8(_mm_cvtsi32_si128((int)w), zero), zero);
    x = _mm_or_si128(x, _mm_cmpeq_epi32(x, ff));
    _mm_stream_si128(reinterpret_cast<__m128i*>(out + e), x);
  }
  for (; e < e1; ++e) one(e);
}

// Elements [e0, e1) of a uint32 parent array into int64 (UNREACHED -> -1).
void widen_parents(const uint32_t* in, int64_t e0, int64_t e1, int64_t* out) {
  int64_t e = e0;
  auto one = [&](int64_t i) { out[i] = in[i] == kNoLevel ? -1 : (int64_t)in[i]; };
  while (e < e1 && (reinterpret_cast<uintptr_t>(out + e) & 15)) one(e++);
  const __m128i ones = _mm_set1_epi32(-1);
  for (; e + 2 <= e1; e += 2) {
    const __m128i x = _mm_loadl_epi64(reinterpret_cast<const __m128i*>(in + e));
    _mm_stream_si128(reinterpret_cast<__m128i*>(out + e),
                     _mm_unpacklo_epi32(x, _mm_cmpeq_epi32(x, ones)));
  }
  for (; e < e1; ++e) one(e);
}

}  // namespace

// Host threads that widen the landed chunks: created once at engine setup
// and parked on a condition variable between read-outs (no thread creation
// per call); the calling thread takes part as worker size() - 1.
struct ReadPool {
  std::vector<std::thread> th;
  std::mutex mu;
  std::condition_variable go, done;
  std::function<void(int)> job;
  int64_t gen = 0;
  int pending = 0;
  bool stop = false;
  explicit ReadPool(int T, int dev) {
    for (int t = 0; t + 1 < T; ++t)
      th.emplace_back([this, t, dev] {
        cudaSetDevice(dev);
        int64_t seen = 0;
        while (true) {
          std::function<void(int)> j;
          {
            std::unique_lock<std::mutex> lk(mu);
            go.wait(lk, [&] { return stop || gen != seen; });
            if (stop) return;
            seen = gen;
            j = job;
          }
          j(t);
          std::lock_guard<std::mutex> lk(mu);
          if (--pending == 0) done.notify_one();
        }
      });
  }
  ~ReadPool() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    go.notify_all();
    for (auto& t : th) t.join();
  }
  int size() const { return (int)th.size() + 1; }
  template <class F>
  void run(F& f) {
    {
      std::lock_guard<std::mutex> lk(mu);
      job = [&f](int t) { f(t); };
      pending = (int)th.size();
      ++gen;
    }
    go.notify_all();
    f((int)th.size());
    std::unique_lock<std::mutex> lk(mu);
    done.wait(lk, [&] { return pending == 0; });
  }
};

namespace {

int ensure_stage(bfb_ctx* ctx, size_t bytes, int nchunks) {
  HostStage& st = ctx->stage;
  if (st.bytes < bytes) {
    if (st.p) cudaFreeHost(st.p);
    st.p = nullptr;
    st.bytes = 0;
    ++alloc_counter();
    BFB_CUDA(cudaHostAlloc(&st.p, bytes, cudaHostAllocDefault));
    st.bytes = bytes;
  }
  while ((int)st.ev.size() < nchunks) {
    cudaEvent_t e;
    BFB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    st.ev.push_back(e);
  }
  return BFB_OK;
}

// Copies `bytes` from device memory into the stage as a chain of chunks on
// stream s, and runs work(lo, hi) over the landed bytes on the host threads:
// every thread takes its 64-byte-aligned share of each chunk as soon as that
// chunk's event fires, so the widening overlaps the rest of the copy.
template <class Work>
int pipelined_read(bfb_ctx* ctx, const void* src, size_t bytes, cudaStream_t s, Work work) {
  if (bytes == 0) return BFB_OK;
  constexpr size_t kMinChunk = size_t(1) << 20;
  size_t chunk = std::max(kMinChunk, (bytes / 32 + 4095) & ~size_t(4095));
  const int nchunks = (int)((bytes + chunk - 1) / chunk);
  BFB_TRY(ensure_stage(ctx, bytes, nchunks));
  uint8_t* stage = static_cast<uint8_t*>(ctx->stage.p);
  for (int k = 0; k < nchunks; ++k) {
    const size_t lo = (size_t)k * chunk, len = std::min(chunk, bytes - lo);
    BFB_CUDA(cudaMemcpyAsync(stage + lo, static_cast<const uint8_t*>(src) + lo, len,
                             cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaEventRecord(ctx->stage.ev[k], s));
  }
  const int T = bytes < (size_t(8) << 20) || !ctx->pool ? 1 : ctx->pool->size();
  std::atomic<int> bad{0};
  auto run = [&](int t) {
    for (int k = 0; k < nchunks; ++k) {
      if (cudaEventSynchronize(ctx->stage.ev[k]) != cudaSuccess) {
        bad.store(1);
        return;
      }
      const size_t lo = (size_t)k * chunk, len = std::min(chunk, bytes - lo);
      const size_t share = ((len + T - 1) / T + 63) & ~size_t(63);
      const size_t a = lo + std::min(len, share * t), b = lo + std::min(len, share * (t + 1));
      if (a < b) work(a, b);
    }
    _mm_sfence();
  };
  if (T == 1)
    run(0);
  else
    ctx->pool->run(run);
  if (bad.load()) BFB_CUDA(cudaStreamSynchronize(s));
  return BFB_OK;
}

}  // namespace

int readout_setup(bfb_ctx* ctx, int64_t n) {
  if (n <= 0) return BFB_OK;
  // packed levels: 8 bits per vertex at most; stage: a uint32 per vertex
  // (parents, or levels past 255); one event per chunk (<= 32 + 1 chunks)
  const int64_t words = (n + 3) / 4;
  if ((int64_t)ctx->packed.n < words) BFB_TRY(ctx->packed.alloc((size_t)words));
  BFB_TRY(ensure_stage(ctx, (size_t)n * 4, 40));
  if (!ctx->pool) ctx->pool = new ReadPool(host_threads(), ctx->device);
  return BFB_OK;
}

void readout_release(bfb_ctx* ctx) {
  delete ctx->pool;
  ctx->pool = nullptr;
  ctx->packed.release();
  ctx->stage.release();
}

int read_levels(bfb_ctx* ctx, const uint32_t* level, int64_t n, int64_t num_levels,
                uint32_t* out, cudaStream_t s) {
  if (n <= 0) return BFB_OK;
  init_tables();
  const unsigned grid = (unsigned)std::min<int64_t>((n / 8 + 255) / 256 + 1, ctx->num_sms * 8);
  if (num_levels <= 15) {  // values 0..14, 15 = UNREACHED
    const int64_t words = (n + 7) / 8;
    if ((int64_t)ctx->packed.n < words) BFB_TRY(ctx->packed.alloc((size_t)(n + 3) / 4));
    k_pack_levels4<<<grid, 256, 0, s>>>(level, n, ctx->packed.p);
    BFB_CUDA(cudaGetLastError());
    return pipelined_read(ctx, ctx->packed.p, (size_t)((n + 1) / 2), s,
                          [&](size_t lo, size_t hi) {
                            widen_nibbles(static_cast<const uint8_t*>(ctx->stage.p),
                                          (int64_t)lo * 2,
                                          std::min<int64_t>((int64_t)hi * 2, n), out);
                          });
  }
  if (num_levels <= 255) {  // values 0..254, 255 = UNREACHED
    const int64_t words = (n + 3) / 4;
    if ((int64_t)ctx->packed.n < words) BFB_TRY(ctx->packed.alloc((size_t)words));
    k_pack_levels8<<<grid, 256, 0, s>>>(level, n, ctx->packed.p);
    BFB_CUDA(cudaGetLastError());
    return pipelined_read(ctx, ctx->packed.p, (size_t)n, s, [&](size_t lo, size_t hi) {
      widen_bytes(static_cast<const uint8_t*>(ctx->stage.p), (int64_t)lo, (int64_t)hi, out);
    });
  }
  return pipelined_read(ctx, level, (size_t)n * 4, s, [&](size_t lo, size_t hi) {
    std::memcpy(reinterpret_cast<uint8_t*>(out) + lo,
                static_cast<const uint8_t*>(ctx->stage.p) + lo, hi - lo);
  });
}

int read_parents(bfb_ctx* ctx, const uint32_t* parent, int64_t n, int64_t* out, cudaStream_t s) {
  if (n <= 0) return BFB_OK;
  return pipelined_read(ctx, parent, (size_t)n * 4, s, [&](size_t lo, size_t hi) {
    widen_parents(static_cast<const uint32_t*>(ctx->stage.p), (int64_t)(lo / 4),
                  (int64_t)(hi / 4), out);
  });
}

}  // namespace bfb
