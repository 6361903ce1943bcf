// Degree-ordered relabel of the resident graph for the engine (built once per
// partition at engine setup; results are mapped back to the caller's ids).
//
// Phase 1 probes one visited bit per traversed edge, and at scale 29 the
// probes are bound by the L1TEX tag rate: a warp-wide probe touches up to 32
// distinct 128-byte lines.  On Kronecker graphs the edge targets are
// dominated by a small set of hubs, but the generator scatters the hubs over
// the whole id space.  Relabelling each part's vertices by degree class
// (floor(log2 degree), descending; isolated last; ascending old id inside a
// class) packs the hubs into a few lines of the bitmap, so the probes of a
// warp share lines; the rows, re-sorted by new id, list their hub neighbours
// first (the bottom-up scan and the parent pass hit earlier).
//
// The map stays inside each part's range [b[g], b[g+1]), so ownership,
// partition boundaries and every per-node count (frontier sizes, snapshot
// sizes, traversed edges) are unchanged; the BFS levels of vertex v are
// those of perm[v] in the relabelled graph.
#include <algorithm>
#include <cstdlib>

#include "bfb_device.cuh"
#include "bfb_internal.cuh"

namespace bfb {
namespace {

constexpr int kKeyBins = 64;  // degree classes 0..32, isolated = 63
constexpr int kRelabelBlock = 1024;

__device__ __forceinline__ int degree_class(int64_t d) {
  return d <= 0 ? kKeyBins - 1 : 32 - (63 - __clzll((unsigned long long)d));
}

// Per 1024-vertex tile of one part: histogram of degree classes, written
// class-major (hist[key * ntiles + tile]) so one exclusive scan gives every
// (class, tile)'s first new id.
__global__ void __launch_bounds__(kRelabelBlock) k_class_hist(const int64_t* __restrict__ off,
                                                              int64_t lo, int64_t hi,
                                                              int64_t ntiles, uint32_t* hist) {
  __shared__ uint32_t h[kKeyBins];
  if (threadIdx.x < kKeyBins) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t v = lo + (int64_t)blockIdx.x * kRelabelBlock + threadIdx.x;
  if (v < hi) atomicAdd(&h[degree_class(__ldg(off + v + 1) - __ldg(off + v))], 1u);
  __syncthreads();
  if (threadIdx.x < kKeyBins) hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// perm[v] = lo + (class, tile) prefix + stable rank of v among its tile's
// vertices of the same class; inv is its inverse.
__global__ void __launch_bounds__(kRelabelBlock) k_class_scatter(const int64_t* __restrict__ off,
                                                                 int64_t lo, int64_t hi,
                                                                 int64_t ntiles,
                                                                 const int64_t* __restrict__ pos,
                                                                 uint32_t* perm, uint32_t* inv) {
  __shared__ uint32_t wcnt[kRelabelBlock / 32][kKeyBins];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (kRelabelBlock / 32) * kKeyBins; i += kRelabelBlock)
    (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t v = lo + (int64_t)blockIdx.x * kRelabelBlock + threadIdx.x;
  const bool in = v < hi;
  const int key = in ? degree_class(__ldg(off + v + 1) - __ldg(off + v)) : kKeyBins;  // kKeyBins: none
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const unsigned lt = (1u << lane) - 1u;
  const int rank_w = __popc(peers & lt);
  if (in && rank_w == 0) wcnt[warp][key] = __popc(peers);
  __syncthreads();
  if (in) {
    int rank = rank_w;
    for (int w = 0; w < warp; ++w) rank += wcnt[w][key];
    const uint32_t nv = (uint32_t)(lo + pos[(int64_t)key * ntiles + blockIdx.x] + rank);
    perm[v] = nv;
    inv[nv] = (uint32_t)v;
  }
}

__global__ void k_rel_offsets(const int64_t* __restrict__ noff, int64_t lo, int64_t cnt,
                              int64_t* rel) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    rel[i] = noff[lo + i] - noff[lo];
}

__global__ void k_new_degrees(const int64_t* __restrict__ off, const uint32_t* __restrict__ inv,
                              int64_t n, uint32_t* deg) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = inv[r];
    deg[r] = (uint32_t)(__ldg(off + v + 1) - __ldg(off + v));
  }
}

// Row r of the relabelled graph = old row inv[r] with every neighbour mapped
// through perm (unsorted; sort_rows orders it).  Warp per row from a counter,
// so the hub rows (new ids first) start first; 8 loads in flight per lane.
__global__ void __launch_bounds__(256) k_gather_rows(const int64_t* __restrict__ off,
                                                     const uint32_t* __restrict__ adj,
                                                     const int64_t* __restrict__ noff,
                                                     const uint32_t* __restrict__ perm,
                                                     const uint32_t* __restrict__ inv, int64_t r_lo,
                                                     int64_t r_hi, unsigned long long* next,
                                                     uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const int64_t obase = noff[r_lo];
  while (true) {
    unsigned long long k = 0;
    if (lane == 0) k = atomicAdd(next, 1ull);
    const int64_t r = r_lo + (int64_t)__shfl_sync(0xffffffffu, k, 0);
    if (r >= r_hi) return;
    const uint32_t v = __ldg(inv + r);
    const int64_t b = __ldg(off + v), d = __ldg(off + v + 1) - b;
    const int64_t o = __ldg(noff + r) - obase;
    for (int64_t j0 = 0; j0 < d; j0 += 32 * 8) {
      uint32_t u[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t j = j0 + k * 32 + lane;
        u[k] = j < d ? __ldg(adj + b + j) : 0u;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t j = j0 + k * 32 + lane;
        if (j < d) out[o + j] = __ldg(perm + u[k]);
      }
    }
  }
}

unsigned grid_of(int64_t work, int block, int sms) {
  int64_t g = (work + block - 1) / block;
  g = std::min<int64_t>(g, (int64_t)sms * 16);
  return (unsigned)std::max<int64_t>(1, g);
}

}  // namespace

bool relabel_wanted(const bfb_ctx* ctx) {
  const char* e = std::getenv("BFB_RELABEL");
  if (e && e[0] == '0') return false;
  return ctx->g.m > 0;
}

int relabel_build(bfb_ctx* ctx, const std::vector<int64_t>& bounds) {
  if (ctx->relabeled && ctx->relabel_bounds == bounds) return BFB_OK;
  ctx->relabeled = false;
  ctx->eg = DevGraph();
  const int64_t n = ctx->g.n, m = ctx->g.m;
  cudaStream_t s = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t* off = ctx->g.offsets.p;
  BFB_TRY(ctx->perm.alloc(n + 1));
  BFB_TRY(ctx->inv.alloc(n + 1));
  // 1. the permutation, part by part
  for (size_t g = 0; g + 1 < bounds.size(); ++g) {
    const int64_t lo = bounds[g], hi = bounds[g + 1];
    if (hi <= lo) continue;
    const int64_t ntiles = (hi - lo + kRelabelBlock - 1) / kRelabelBlock;
    DevBuf<uint32_t> hist;
    DevBuf<int64_t> pos, tmp;
    BFB_TRY(hist.alloc((size_t)kKeyBins * ntiles));
    BFB_TRY(pos.alloc((size_t)kKeyBins * ntiles + 1));
    BFB_TRY(tmp.alloc(scan_tmp_words((int64_t)kKeyBins * ntiles) + 1));
    k_class_hist<<<(unsigned)ntiles, kRelabelBlock, 0, s>>>(off, lo, hi, ntiles, hist.p);
    BFB_TRY(scan_u32_to_i64(hist.p, (int64_t)kKeyBins * ntiles, pos.p, tmp.p, s));
    k_class_scatter<<<(unsigned)ntiles, kRelabelBlock, 0, s>>>(off, lo, hi, ntiles, pos.p,
                                                                ctx->perm.p, ctx->inv.p);
    BFB_CUDA(cudaStreamSynchronize(s));  // hist / pos are freed at scope end
  }
  // 2. the relabelled CSR: degrees by new id, offsets, mapped rows, sorted
  DevGraph eg;
  eg.n = n;
  eg.m = m;
  eg.max_degree = ctx->g.max_degree;
  {
    DevBuf<uint32_t> deg;
    DevBuf<int64_t> tmp;
    BFB_TRY(deg.alloc(n + 1));
    BFB_TRY(tmp.alloc(scan_tmp_words(n) + 1));
    BFB_TRY(eg.offsets.alloc(n + 1));
    k_new_degrees<<<grid_of(n, 256, sms), 256, 0, s>>>(off, ctx->inv.p, n, deg.p);
    BFB_TRY(scan_u32_to_i64(deg.p, n, eg.offsets.p, tmp.p, s));
    BFB_CUDA(cudaStreamSynchronize(s));
  }
  {
    // the rows this context holds (all of them, or one rank's part: the
    // relabel maps each part onto itself, so the part's rows stay its own)
    const int64_t lo = ctx->g.row_lo, hi = ctx->g.row_hi;
    eg.row_lo = lo;
    eg.row_hi = hi;
    eg.adj_lo = ctx->g.adj_lo;
    int64_t ms = 0;
    BFB_CUDA(cudaMemcpy(&ms, eg.offsets.p + hi, sizeof(int64_t), cudaMemcpyDeviceToHost));
    ms -= eg.adj_lo;
    DevBuf<uint32_t> rows;
    DevBuf<int64_t> rel;
    DevBuf<unsigned long long> next;
    BFB_TRY(rows.alloc(ms + 1));
    BFB_TRY(rel.alloc(hi - lo + 1));
    BFB_TRY(next.alloc(1));
    BFB_CUDA(cudaMemsetAsync(next.p, 0, sizeof(unsigned long long), s));
    k_gather_rows<<<(unsigned)sms * 8, 256, 0, s>>>(off, ctx->g.adj_index(), eg.offsets.p,
                                                    ctx->perm.p, ctx->inv.p, lo, hi, next.p, rows.p);
    k_rel_offsets<<<grid_of(hi - lo + 1, 256, sms), 256, 0, s>>>(eg.offsets.p, lo, hi - lo, rel.p);
    BFB_TRY(eg.adj.alloc(ms + 1));
    BFB_TRY(sort_rows(ctx, rel.p, hi - lo, ms, rows.p, eg.adj.p, n));
    BFB_CUDA(cudaStreamSynchronize(s));
  }
  BFB_CUDA(cudaGetLastError());
  eg.valid = true;
  ctx->eg = std::move(eg);
  ctx->relabel_bounds = bounds;
  ctx->relabeled = true;
  return BFB_OK;
}

void relabel_release(bfb_ctx* ctx) {
  ctx->relabeled = false;
  ctx->relabel_bounds.clear();
  ctx->eg = DevGraph();
  ctx->perm.release();
  ctx->inv.release();
}

}  // namespace bfb
