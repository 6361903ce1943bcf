// Device graph build: RMAT/Kronecker generator (graphs.py:254-285),
// symmetrize (graphs.py:218-230), build_csr (graphs.py:233-251),
// partition_1d (graphs.py:288-305), and root selection helpers.
//
// Build pipeline (all on device, edge-parallel, no 64-bit global sort):
//   count   : degree histogram of the (mirrored, self-loop-free) edges
//   scan    : row starts (int64)
//   scatter : each edge appended to its row (atomic row cursor)
//   sort    : per-row sort (segsort.cu: warp bitonic, block radix for long rows)
//   flag    : first-of-row or differs-from-predecessor, packed 32 per word
//   scan    : popcount prefix -> deduplicated offsets; compact.
// The RMAT source is regenerated for the count and scatter passes instead of
// being stored (2 x 17 GB saved at scale 29); PCG64 jump-ahead makes any draw
// index addressable.

#include <algorithm>

#include "bfb_device.cuh"
#include "bfb_internal.cuh"

namespace bfb {
namespace {

constexpr int kGenEPT = 16;       // edges per lane in the generator
constexpr int kGenBlock = 256;
constexpr int kEdgesPerWarp = 32 * kGenEPT;

enum GenMode { kModeEdges = 0, kModeCount = 1, kModeScatter = 2 };

struct RmatParams {
  Affine step;    // one PCG64 step
  Affine jump32;  // 32 steps: next item of this lane within a draw row
  Affine jump_m;  // m steps: same edge, next draw row
  U128 s0;        // initial state of default_rng(seed)
  int scale;
  int64_t m;
  uint64_t t_bottom, t_right_top, t_right_bottom;  // ceil(p * 2^53)
};

struct BuildSink {
  uint2* edges;            // kModeEdges
  uint32_t* deg;           // kModeCount
  const int64_t* rowstart; // kModeScatter: rows [row_lo, row_hi) only, indexed from row_lo
  uint32_t* fill;
  uint32_t* rows;
  int64_t row_lo, row_hi;
};

__device__ __forceinline__ void sink_row(const BuildSink& k, uint32_t s, uint32_t d) {
  if ((int64_t)s < k.row_lo || (int64_t)s >= k.row_hi) return;
  const int64_t r = (int64_t)s - k.row_lo;
  const uint32_t p = atomicAdd(&k.fill[r], 1u);
  k.rows[k.rowstart[r] + p] = d;
}

__device__ __forceinline__ void sink_edge(int mode, const BuildSink& k, int64_t e, uint32_t s,
                                          uint32_t d) {
  if (mode == kModeEdges) {
    k.edges[e] = make_uint2(s, d);
  } else if (s != d) {  // symmetrize drops self-loops (graphs.py:223-224)
    if (mode == kModeCount) {
      atomicAdd(&k.deg[s], 1u);
      atomicAdd(&k.deg[d], 1u);
    } else {
      sink_row(k, s, d);
      sink_row(k, d, s);
    }
  }
}

// Lane l of warp w owns edges e = w*512 + l + 32*i, i < 16.  Draw index of
// (bit iteration kb from the MSB, j = 0 src / 1 dst, edge e) is (2kb+j)*m + e;
// draw k is the XSL-RR output of the state after k+1 steps.
template <int MODE>
__global__ void __launch_bounds__(kGenBlock) k_rmat(RmatParams P, BuildSink sink) {
  const int64_t warp = ((int64_t)blockIdx.x * kGenBlock + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t base = warp * kEdgesPerWarp + lane;
  if (warp * kEdgesPerWarp >= P.m) return;
  U128 row = apply(affine_pow(P.step, (uint64_t)base + 1), P.s0);
  uint32_t src[kGenEPT], dst[kGenEPT];
#pragma unroll
  for (int i = 0; i < kGenEPT; ++i) src[i] = dst[i] = 0;
  for (int kb = 0; kb < P.scale; ++kb) {
    const int bit = P.scale - 1 - kb;
    uint32_t sbits = 0;
    U128 x = row;
#pragma unroll
    for (int i = 0; i < kGenEPT; ++i) {
      if (i) x = apply(P.jump32, x);
      uint64_t k = xsl_rr(x) >> 11;
      sbits |= (k < P.t_bottom ? 1u : 0u) << i;
    }
    row = apply(P.jump_m, row);
    x = row;
#pragma unroll
    for (int i = 0; i < kGenEPT; ++i) {
      if (i) x = apply(P.jump32, x);
      uint64_t k = xsl_rr(x) >> 11;
      uint32_t sb = (sbits >> i) & 1u;
      uint64_t thr = sb ? P.t_right_bottom : P.t_right_top;
      src[i] |= sb << bit;
      dst[i] |= (k < thr ? 1u : 0u) << bit;
    }
    row = apply(P.jump_m, row);
  }
#pragma unroll
  for (int i = 0; i < kGenEPT; ++i) {
    int64_t e = base + 32 * (int64_t)i;
    if (e < P.m) sink_edge(MODE, sink, e, src[i], dst[i]);
  }
}

// Edge-array source.  mirror: symmetrize semantics (drop self-loops, both
// directions); else build_csr semantics (src rows only, self-edge -> error).
template <int MODE>
__global__ void k_edges(const uint2* __restrict__ edges, int64_t m, int64_t n, int mirror,
                        BuildSink sink, unsigned* err) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint2 p = edges[e];
    if ((int64_t)p.x >= n || (int64_t)p.y >= n) {
      atomicOr(err, 8u);
      continue;
    }
    if (mirror) {
      sink_edge(MODE, sink, e, p.x, p.y);
    } else {
      if (p.x == p.y) atomicOr(err, 1u);
      if (MODE == kModeCount) {
        atomicAdd(&sink.deg[p.x], 1u);
      } else {
        sink_row(sink, p.x, p.y);
      }
    }
  }
}

// Mark the first slot of every non-empty row in a bitmap over element slots.
__global__ void k_mark_rowstarts(const int64_t* __restrict__ rowstart, int64_t n,
                                 uint32_t* rs_bits) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = rowstart[v];
    if (rowstart[v + 1] > p) atomicOr(&rs_bits[p >> 5], 1u << (p & 31));
  }
}

// keep(i) = first of its row or differs from its predecessor; duplicates
// (a kept == false slot) flag error bit 2 when validating.
__global__ void k_flag_unique(const uint32_t* __restrict__ a, int64_t total,
                              const uint32_t* __restrict__ rs_bits, uint32_t* keep_words,
                              unsigned* err) {
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31LL; i0 < total;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = i0 + lane;
    bool keep = false;
    if (i < total) {
      bool rs = (rs_bits[i >> 5] >> (i & 31)) & 1u;
      keep = rs || a[i] != a[i - 1];
    }
    unsigned b = __ballot_sync(0xffffffffu, keep);
    bool dup = (i < total) && !keep;
    if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr(err, 2u);
    if (lane == 0) keep_words[i0 >> 5] = b;
  }
}

__global__ void k_new_offsets(const int64_t* __restrict__ rowstart, int64_t n,
                              const uint32_t* __restrict__ keep_words,
                              const int64_t* __restrict__ word_pre, int64_t* newoff,
                              unsigned long long* maxdeg) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = rowstart[v];
    uint32_t lowmask = (1u << (p & 31)) - 1u;
    int64_t q = word_pre[p >> 5] + ((p & 31) ? __popc(keep_words[p >> 5] & lowmask) : 0);
    newoff[v] = q;
  }
}

__global__ void k_max_degree(const int64_t* __restrict__ off, int64_t n,
                             unsigned long long* maxdeg) {
  unsigned long long best = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long d = (unsigned long long)(off[v + 1] - off[v]);
    best = d > best ? d : best;
  }
  for (int s = 16; s; s >>= 1) {
    unsigned long long o = __shfl_xor_sync(0xffffffffu, best, s);
    best = o > best ? o : best;
  }
  if ((threadIdx.x & 31) == 0 && best) atomicMax(maxdeg, best);
}

__global__ void k_compact(const uint32_t* __restrict__ a, int64_t total,
                          const uint32_t* __restrict__ keep_words,
                          const int64_t* __restrict__ word_pre, uint32_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w = keep_words[i >> 5];
    uint32_t bit = 1u << (i & 31);
    if (w & bit) out[word_pre[i >> 5] + __popc(w & (bit - 1u))] = a[i];
  }
}

// build_csr validation: every (u, v) needs (v, u) (graphs.py:245-247).
__global__ void k_check_reverse(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                int64_t n, unsigned* err) {
  const int lane = threadIdx.x & 31;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int64_t b = off[u], e = off[u + 1];
    bool bad = false;
    for (int64_t j = b + lane; j < e; j += 32) {
      uint32_t v = adj[j];
      int64_t lo = off[v], hi = off[v + 1];
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (adj[mid] < (uint32_t)u) lo = mid + 1; else hi = mid;
      }
      if (lo >= off[v + 1] || adj[lo] != (uint32_t)u) bad = true;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 4u);
  }
}

// Largest v in [lo, hi] with a[v] <= key (a non-decreasing).

__global__ void k_expand_edges(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                               int64_t n, uint2* out) {
  const int lane = threadIdx.x & 31;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    for (int64_t j = off[u] + lane; j < off[u + 1]; j += 32) out[j] = make_uint2((uint32_t)u, adj[j]);
  }
}

// partition_1d: boundary k = searchsorted(offsets, round_half_up(|E| k / P), 'left').
__global__ void k_partition(const int64_t* __restrict__ off, int64_t n, int64_t m, int parts,
                            int64_t* out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > parts) return;
  if (k == 0) { out[0] = 0; return; }
  if (k == parts) { out[parts] = n; return; }
  int64_t target = (2 * m * (int64_t)k + parts) / (2 * (int64_t)parts);
  int64_t lo = 0, hi = n + 1;  // first i in [0, n+1) with off[i] >= target
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (off[mid] < target) lo = mid + 1; else hi = mid;
  }
  out[k] = lo;
}

constexpr int64_t kNzTile = 4096;

__global__ void k_nz_tile_counts(const int64_t* __restrict__ off, int64_t n, uint32_t* counts) {
  int64_t t = blockIdx.x;
  int64_t b = t * kNzTile;
  uint32_t c = 0;
  for (int64_t v = b + threadIdx.x; v < min(n, b + kNzTile); v += blockDim.x)
    c += off[v + 1] > off[v] ? 1u : 0u;
  for (int s = 16; s; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
  __shared__ uint32_t red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    counts[t] = s;
  }
}

__global__ void k_nz_select(const int64_t* __restrict__ off, int64_t n,
                            const int64_t* __restrict__ tile_pre, int64_t ntiles,
                            const int64_t* __restrict__ ranks, int64_t k, int64_t* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  int64_t r = ranks[i];
  if (r < 0 || r >= tile_pre[ntiles]) { out[i] = -1; return; }
  int64_t lo = 0, hi = ntiles - 1;  // last tile with tile_pre[t] <= r
  while (lo < hi) {
    int64_t mid = lo + (hi - lo + 1) / 2;
    if (tile_pre[mid] <= r) lo = mid; else hi = mid - 1;
  }
  int64_t left = r - tile_pre[lo];
  for (int64_t v = lo * kNzTile; v < n; ++v) {
    if (off[v + 1] > off[v]) {
      if (left == 0) { out[i] = v; return; }
      --left;
    }
  }
  out[i] = -1;
}

unsigned grid_for(int64_t work, int block, int num_sms) {
  int64_t g = (work + block - 1) / block;
  int64_t cap = (int64_t)num_sms * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

RmatParams make_params(int scale, int64_t ef, U128 state, U128 inc, const uint64_t thr[3]) {
  RmatParams P;
  P.step.a = U128{kPcgMultHi, kPcgMultLo};
  P.step.c = inc;
  P.jump32 = affine_pow(P.step, 32);
  P.m = ef << scale;
  P.jump_m = affine_pow(P.step, (uint64_t)P.m);
  P.s0 = state;
  P.scale = scale;
  P.t_bottom = thr[0];
  P.t_right_top = thr[1];
  P.t_right_bottom = thr[2];
  return P;
}

int check_rmat_args(int scale, int64_t ef) {
  if (scale < 1 || ef < 1) return fail(BFB_ERR_INVALID, "scale and edge_factor must be >= 1");
  if (scale > 32) return fail(BFB_ERR_INVALID, "scale " + std::to_string(scale) +
                                                   " overflows the vertex-id range");
  if (ef > (int64_t(1) << 40) >> scale) return fail(BFB_ERR_INVALID, "edge count too large");
  return BFB_OK;
}

template <int MODE>
int launch_rmat(const RmatParams& P, const BuildSink& sink, cudaStream_t s) {
  int64_t warps = (P.m + kEdgesPerWarp - 1) / kEdgesPerWarp;
  int64_t blocks = (warps * 32 + kGenBlock - 1) / kGenBlock;
  k_rmat<MODE><<<(unsigned)blocks, kGenBlock, 0, s>>>(P, sink);
  BFB_CUDA(cudaGetLastError());
  return BFB_OK;
}


}  // namespace

namespace {

// Shared tail of both build paths: rows are scattered, now sort, flag, dedup
// (or validate), and install as the resident CSR.
template <class ScatterFn>
int finish_build(bfb_ctx* ctx, int64_t n, DevBuf<uint32_t>& deg, ScatterFn scatter, bool dedup,
                 bool validate) {
  cudaStream_t s = ctx->stream;
  const int sms = ctx->num_sms;
  DevBuf<int64_t> rowstart, scan_tmp;
  BFB_TRY(rowstart.alloc(n + 1));
  BFB_TRY(scan_tmp.alloc(scan_tmp_words(n) + 1));
  BFB_TRY(scan_u32_to_i64(deg.p, n, rowstart.p, scan_tmp.p, s));
  int64_t total = 0;
  BFB_CUDA(cudaMemcpyAsync(&total, rowstart.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  DevBuf<uint32_t> rows;
  BFB_TRY(rows.alloc(total));
  BFB_CUDA(cudaMemsetAsync(deg.p, 0, n * sizeof(uint32_t), s));  // reuse as row cursor
  BuildSink sink{};
  sink.rowstart = rowstart.p;
  sink.fill = deg.p;
  sink.rows = rows.p;
  sink.row_lo = 0;
  sink.row_hi = n;
  BFB_TRY(scatter(sink));
  deg.release();
  DevBuf<uint32_t> sorted;
  BFB_TRY(sorted.alloc(total));
  BFB_TRY(sort_rows(ctx, rowstart.p, n, total, rows.p, sorted.p, n));
  DevBuf<unsigned> err;
  BFB_TRY(err.alloc(1));
  BFB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(unsigned), s));
  int64_t nwords = (total + 31) / 32;
  DevBuf<uint32_t> rs_bits, keep;
  BFB_TRY(rs_bits.alloc(nwords + 1));
  BFB_TRY(keep.alloc(nwords + 1));
  BFB_CUDA(cudaMemsetAsync(rs_bits.p, 0, (nwords + 1) * sizeof(uint32_t), s));
  BFB_CUDA(cudaMemsetAsync(keep.p, 0, (nwords + 1) * sizeof(uint32_t), s));
  k_mark_rowstarts<<<grid_for(n, 256, sms), 256, 0, s>>>(rowstart.p, n, rs_bits.p);
  k_flag_unique<<<grid_for(nwords * 32, 256, sms), 256, 0, s>>>(sorted.p, total, rs_bits.p, keep.p,
                                                               err.p);
  rs_bits.release();
  DevBuf<unsigned long long> maxdeg;
  BFB_TRY(maxdeg.alloc(1));
  BFB_CUDA(cudaMemsetAsync(maxdeg.p, 0, sizeof(unsigned long long), s));
  DevBuf<int64_t> offsets;
  DevBuf<uint32_t> adj;
  int64_t m_final = total;
  if (dedup) {
    DevBuf<int64_t> word_pre;
    BFB_TRY(word_pre.alloc(nwords + 1));
    DevBuf<int64_t> tmp2;
    BFB_TRY(tmp2.alloc(scan_tmp_words(nwords) + 1));
    BFB_TRY(scan_popc_to_i64(keep.p, nwords, word_pre.p, tmp2.p, s));
    BFB_TRY(offsets.alloc(n + 1));
    k_new_offsets<<<grid_for(n + 1, 256, sms), 256, 0, s>>>(rowstart.p, n, keep.p, word_pre.p,
                                                             offsets.p, maxdeg.p);
    BFB_CUDA(cudaMemcpyAsync(&m_final, offsets.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    // compact into the (now free) scatter buffer
    k_compact<<<grid_for(total, 256, sms), 256, 0, s>>>(sorted.p, total, keep.p, word_pre.p,
                                                        rows.p);
    BFB_CUDA(cudaStreamSynchronize(s));
    adj = std::move(rows);
  } else {
    offsets = std::move(rowstart);
    adj = std::move(sorted);
  }
  k_max_degree<<<grid_for(n, 256, sms), 256, 0, s>>>(offsets.p, n, maxdeg.p);
  if (validate) {
    unsigned h = 0;
    BFB_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaStreamSynchronize(s));
    if (h & 8u) return fail(BFB_ERR_RANGE, "edge endpoint exceeds num_vertices");
    if (h & 1u) return fail(BFB_ERR_SELF_EDGE, "input is not symmetrized: self-edge present");
    if (h & 2u) return fail(BFB_ERR_DUPLICATE, "input is not symmetrized: duplicate edge present");
    k_check_reverse<<<grid_for(n * 32, 256, sms), 256, 0, s>>>(offsets.p, adj.p, n, err.p);
    BFB_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaStreamSynchronize(s));
    if (h & 4u) return fail(BFB_ERR_NO_REVERSE, "input is not symmetrized: missing reverse edge");
  } else {
    unsigned h = 0;
    BFB_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaStreamSynchronize(s));
    if (h & 8u) return fail(BFB_ERR_RANGE, "edge endpoint exceeds num_vertices");
  }
  unsigned long long md = 0;
  BFB_CUDA(cudaMemcpyAsync(&md, maxdeg.p, sizeof(md), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  BFB_CUDA(cudaGetLastError());
  engine_release(ctx);
  relabel_release(ctx);
  ctx->g.offsets = std::move(offsets);
  ctx->g.adj = std::move(adj);
  ctx->g.n = n;
  ctx->g.m = m_final;
  ctx->g.max_degree = (int64_t)md;
  ctx->g.row_lo = 0;
  ctx->g.row_hi = n;
  ctx->g.adj_lo = 0;
  ctx->g.valid = true;
  return BFB_OK;
}

}  // namespace

namespace {

__global__ void k_row_degrees(const int64_t* __restrict__ rel_off, int64_t cnt, uint32_t* deg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    deg[i] = (uint32_t)(rel_off[i + 1] - rel_off[i]);
}

// Rows [a, b) of the symmetrized, deduplicated RMAT graph, from the raw
// degrees (count pass): scatter of the edges with an endpoint in [a, b),
// per-row sort, duplicate flags.  Writes the rows' deduplicated degrees to
// ddeg[a..b) and, when adj_out is given, their adjacency (compacted).
int rmat_slice(bfb_ctx* ctx, const RmatParams& P, const uint32_t* deg, int64_t a, int64_t b,
               uint32_t* ddeg, DevBuf<uint32_t>* adj_out) {
  cudaStream_t s = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t ns = b - a;
  if (ns <= 0) return BFB_OK;
  DevBuf<int64_t> rowstart, tmp;
  BFB_TRY(rowstart.alloc(ns + 1));
  BFB_TRY(tmp.alloc(scan_tmp_words(ns) + 1));
  BFB_TRY(scan_u32_to_i64(deg + a, ns, rowstart.p, tmp.p, s));
  int64_t total = 0;
  BFB_CUDA(cudaMemcpyAsync(&total, rowstart.p + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  DevBuf<uint32_t> rows, fill, sorted;
  BFB_TRY(rows.alloc(total + 1));
  BFB_TRY(fill.alloc(ns));
  BFB_CUDA(cudaMemsetAsync(fill.p, 0, ns * sizeof(uint32_t), s));
  BuildSink sink{};
  sink.rowstart = rowstart.p;
  sink.fill = fill.p;
  sink.rows = rows.p;
  sink.row_lo = a;
  sink.row_hi = b;
  BFB_TRY(launch_rmat<kModeScatter>(P, sink, s));
  fill.release();
  BFB_TRY(sorted.alloc(total + 1));
  BFB_TRY(sort_rows(ctx, rowstart.p, ns, total, rows.p, sorted.p, int64_t(1) << P.scale));
  const int64_t nwords = (total + 31) / 32;
  DevBuf<uint32_t> rs_bits, keep;
  DevBuf<unsigned> err;
  BFB_TRY(err.alloc(1));
  BFB_TRY(rs_bits.alloc(nwords + 1));
  BFB_TRY(keep.alloc(nwords + 1));
  BFB_CUDA(cudaMemsetAsync(rs_bits.p, 0, (nwords + 1) * sizeof(uint32_t), s));
  BFB_CUDA(cudaMemsetAsync(keep.p, 0, (nwords + 1) * sizeof(uint32_t), s));
  k_mark_rowstarts<<<grid_for(ns, 256, sms), 256, 0, s>>>(rowstart.p, ns, rs_bits.p);
  k_flag_unique<<<grid_for(nwords * 32, 256, sms), 256, 0, s>>>(sorted.p, total, rs_bits.p, keep.p,
                                                               err.p);
  rs_bits.release();
  DevBuf<int64_t> word_pre, tmp2, rel_off;
  DevBuf<unsigned long long> unused;
  BFB_TRY(word_pre.alloc(nwords + 1));
  BFB_TRY(tmp2.alloc(scan_tmp_words(nwords) + 1));
  BFB_TRY(scan_popc_to_i64(keep.p, nwords, word_pre.p, tmp2.p, s));
  BFB_TRY(rel_off.alloc(ns + 1));
  BFB_TRY(unused.alloc(1));
  k_new_offsets<<<grid_for(ns + 1, 256, sms), 256, 0, s>>>(rowstart.p, ns, keep.p, word_pre.p,
                                                            rel_off.p, unused.p);
  k_row_degrees<<<grid_for(ns, 256, sms), 256, 0, s>>>(rel_off.p, ns, ddeg + a);
  if (adj_out) {
    int64_t ms = 0;
    BFB_CUDA(cudaMemcpyAsync(&ms, rel_off.p + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaStreamSynchronize(s));
    BFB_TRY(adj_out->alloc(ms + 1));
    k_compact<<<grid_for(total, 256, sms), 256, 0, s>>>(sorted.p, total, keep.p, word_pre.p,
                                                        adj_out->p);
  }
  BFB_CUDA(cudaStreamSynchronize(s));
  BFB_CUDA(cudaGetLastError());
  return BFB_OK;
}

}  // namespace

// One rank's share (SURVEY §8 e: GPU g owns offsets[b[g]..b[g+1]] and that
// adjacency slice).  partition_1d needs every vertex's deduplicated degree,
// so the rows are first built slice by slice under a bounded edge budget
// (degrees kept, adjacency dropped), then the offsets and the partition are
// computed, and the owned rows are built once more and kept.  The generator
// re-runs per slice instead of storing the edge list (PCG64 jump-ahead).
int build_from_rmat_part(bfb_ctx* ctx, int scale, int64_t ef, U128 state, U128 inc,
                         const uint64_t thr[3], int parts, int rank, int64_t* bounds_out) {
  BFB_TRY(check_rmat_args(scale, ef));
  if (parts < 1 || rank < 0 || rank >= parts) return fail(BFB_ERR_INVALID, "bad parts / rank");
  RmatParams P = make_params(scale, ef, state, inc, thr);
  const int64_t n = int64_t(1) << scale;
  if (parts > n) return fail(BFB_ERR_INVALID, "num_parts exceeds the number of vertices");
  engine_release(ctx);
  relabel_release(ctx);
  ctx->g = DevGraph();
  cudaStream_t s = ctx->stream;
  const int sms = ctx->num_sms;
  DevBuf<uint32_t> deg, ddeg;
  BFB_TRY(deg.alloc(n));
  BFB_TRY(ddeg.alloc(n));
  BFB_CUDA(cudaMemsetAsync(deg.p, 0, n * sizeof(uint32_t), s));
  BuildSink sink{};
  sink.deg = deg.p;
  BFB_TRY(launch_rmat<kModeCount>(P, sink, s));
  // degree pass: slices of <= kBudget raw (pre-dedup) entries
  const int64_t kBudget = int64_t(1) << 31;
  int64_t raw_total = 0;
  std::vector<int64_t> cuts;
  {
    DevBuf<int64_t> rs, tmp, b;
    BFB_TRY(rs.alloc(n + 1));
    BFB_TRY(tmp.alloc(scan_tmp_words(n) + 1));
    BFB_TRY(scan_u32_to_i64(deg.p, n, rs.p, tmp.p, s));
    BFB_CUDA(cudaMemcpyAsync(&raw_total, rs.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaStreamSynchronize(s));
    const int ns = (int)std::max<int64_t>(1, (raw_total + kBudget - 1) / kBudget);
    BFB_TRY(b.alloc(ns + 1));
    k_partition<<<(ns + 1 + 127) / 128, 128, 0, s>>>(rs.p, n, raw_total, ns, b.p);
    cuts.resize(ns + 1);
    BFB_CUDA(cudaMemcpyAsync(cuts.data(), b.p, (ns + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaStreamSynchronize(s));
  }
  for (size_t k = 0; k + 1 < cuts.size(); ++k)
    BFB_TRY(rmat_slice(ctx, P, deg.p, cuts[k], cuts[k + 1], ddeg.p, nullptr));
  // offsets of the whole graph, max degree, the partition
  DevGraph G;
  G.n = n;
  BFB_TRY(G.offsets.alloc(n + 1));
  {
    DevBuf<int64_t> tmp;
    BFB_TRY(tmp.alloc(scan_tmp_words(n) + 1));
    BFB_TRY(scan_u32_to_i64(ddeg.p, n, G.offsets.p, tmp.p, s));
  }
  DevBuf<unsigned long long> maxdeg;
  BFB_TRY(maxdeg.alloc(1));
  BFB_CUDA(cudaMemsetAsync(maxdeg.p, 0, sizeof(unsigned long long), s));
  k_max_degree<<<grid_for(n, 256, sms), 256, 0, s>>>(G.offsets.p, n, maxdeg.p);
  unsigned long long md = 0;
  BFB_CUDA(cudaMemcpyAsync(&G.m, G.offsets.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaMemcpyAsync(&md, maxdeg.p, sizeof(md), cudaMemcpyDeviceToHost, s));
  std::vector<int64_t> b(parts + 1);
  {
    DevBuf<int64_t> bd;
    BFB_TRY(bd.alloc(parts + 1));
    BFB_CUDA(cudaStreamSynchronize(s));
    k_partition<<<(parts + 1 + 127) / 128, 128, 0, s>>>(G.offsets.p, n, G.m, parts, bd.p);
    BFB_CUDA(cudaMemcpyAsync(b.data(), bd.p, (parts + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaStreamSynchronize(s));
  }
  G.max_degree = (int64_t)md;
  // the owned rows, kept
  G.row_lo = b[rank];
  G.row_hi = b[rank + 1];
  BFB_CUDA(cudaMemcpy(&G.adj_lo, G.offsets.p + G.row_lo, sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (G.row_hi > G.row_lo) {
    BFB_TRY(rmat_slice(ctx, P, deg.p, G.row_lo, G.row_hi, ddeg.p, &G.adj));
  } else {
    BFB_TRY(G.adj.alloc(1));
  }
  G.valid = true;
  ctx->g = std::move(G);
  if (bounds_out) std::copy(b.begin(), b.end(), bounds_out);
  return BFB_OK;
}

int rmat_to_host(bfb_ctx* ctx, int scale, int64_t ef, U128 state, U128 inc, const uint64_t thr[3],
                 uint32_t* out) {
  BFB_TRY(check_rmat_args(scale, ef));
  RmatParams P = make_params(scale, ef, state, inc, thr);
  // chunk the device buffer to bound memory: generate all, copy in pieces
  DevBuf<uint2> edges;
  BFB_TRY(edges.alloc(P.m));
  BuildSink sink{};
  sink.edges = edges.p;
  BFB_TRY(launch_rmat<kModeEdges>(P, sink, ctx->stream));
  BFB_CUDA(cudaMemcpyAsync(out, edges.p, P.m * sizeof(uint2), cudaMemcpyDeviceToHost, ctx->stream));
  BFB_CUDA(cudaStreamSynchronize(ctx->stream));
  return BFB_OK;
}

int build_from_rmat(bfb_ctx* ctx, int scale, int64_t ef, U128 state, U128 inc,
                    const uint64_t thr[3]) {
  BFB_TRY(check_rmat_args(scale, ef));
  RmatParams P = make_params(scale, ef, state, inc, thr);
  int64_t n = int64_t(1) << scale;
  engine_release(ctx);
  relabel_release(ctx);
  ctx->g = DevGraph();  // free the previous graph before the big allocations
  DevBuf<uint32_t> deg;
  BFB_TRY(deg.alloc(n));
  BFB_CUDA(cudaMemsetAsync(deg.p, 0, n * sizeof(uint32_t), ctx->stream));
  BuildSink sink{};
  sink.deg = deg.p;
  BFB_TRY(launch_rmat<kModeCount>(P, sink, ctx->stream));
  cudaStream_t s = ctx->stream;
  return finish_build(
      ctx, n, deg, [&](const BuildSink& k) { return launch_rmat<kModeScatter>(P, k, s); }, true,
      false);
}

int build_from_edges(bfb_ctx* ctx, int64_t n, const uint32_t* host_edges, int64_t m,
                     bool symmetrize) {
  if (n < 0 || m < 0) return fail(BFB_ERR_INVALID, "negative size");
  if (n > (int64_t(1) << 32)) return fail(BFB_ERR_INVALID, "num_vertices exceeds the VID range");
  engine_release(ctx);
  relabel_release(ctx);
  ctx->g = DevGraph();
  DevBuf<uint2> edges;
  BFB_TRY(edges.alloc(m));
  if (m)
    BFB_CUDA(cudaMemcpyAsync(edges.p, host_edges, m * sizeof(uint2), cudaMemcpyHostToDevice,
                             ctx->stream));
  return build_from_device_edges(ctx, n, edges, m, symmetrize);
}

// symmetrize (optional) + build_csr from an edge array already in HBM.
int build_from_device_edges(bfb_ctx* ctx, int64_t n, DevBuf<uint2>& edges, int64_t m,
                            bool symmetrize) {
  if (n < 0 || m < 0) return fail(BFB_ERR_INVALID, "negative size");
  if (n > (int64_t(1) << 32)) return fail(BFB_ERR_INVALID, "num_vertices exceeds the VID range");
  engine_release(ctx);
  relabel_release(ctx);
  ctx->g = DevGraph();
  cudaStream_t s = ctx->stream;
  DevBuf<uint32_t> deg;
  BFB_TRY(deg.alloc(n));
  BFB_CUDA(cudaMemsetAsync(deg.p, 0, n * sizeof(uint32_t), s));
  DevBuf<unsigned> err;
  BFB_TRY(err.alloc(1));
  BFB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(unsigned), s));
  BuildSink sink{};
  sink.deg = deg.p;
  unsigned grid = grid_for(m, 256, ctx->num_sms);
  int mirror = symmetrize ? 1 : 0;
  if (m) k_edges<kModeCount><<<grid, 256, 0, s>>>(edges.p, m, n, mirror, sink, err.p);
  unsigned h = 0;
  BFB_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  if (h & 8u) return fail(BFB_ERR_RANGE, "edge endpoint exceeds num_vertices");
  if (!symmetrize && (h & 1u))
    return fail(BFB_ERR_SELF_EDGE, "input is not symmetrized: self-edge present");
  return finish_build(
      ctx, n, deg,
      [&](const BuildSink& k) {
        if (m) k_edges<kModeScatter><<<grid, 256, 0, s>>>(edges.p, m, n, mirror, k, err.p);
        BFB_CUDA(cudaGetLastError());
        return BFB_OK;
      },
      symmetrize, !symmetrize);
}

int load_csr(bfb_ctx* ctx, int64_t n, int64_t m, const int64_t* offsets, const uint32_t* adj) {
  if (n < 0 || m < 0) return fail(BFB_ERR_INVALID, "negative size");
  engine_release(ctx);
  relabel_release(ctx);
  ctx->g = DevGraph();
  DevBuf<int64_t> off;
  DevBuf<uint32_t> a;
  BFB_TRY(off.alloc(n + 1));
  BFB_TRY(a.alloc(m));
  cudaStream_t s = ctx->stream;
  BFB_CUDA(cudaMemcpyAsync(off.p, offsets, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  if (m) BFB_CUDA(cudaMemcpyAsync(a.p, adj, m * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  DevBuf<unsigned long long> maxdeg;
  BFB_TRY(maxdeg.alloc(1));
  BFB_CUDA(cudaMemsetAsync(maxdeg.p, 0, sizeof(unsigned long long), s));
  k_max_degree<<<grid_for(n, 256, ctx->num_sms), 256, 0, s>>>(off.p, n, maxdeg.p);
  unsigned long long md = 0;
  BFB_CUDA(cudaMemcpyAsync(&md, maxdeg.p, sizeof(md), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  ctx->g.offsets = std::move(off);
  ctx->g.adj = std::move(a);
  ctx->g.n = n;
  ctx->g.m = m;
  ctx->g.max_degree = (int64_t)md;
  ctx->g.row_lo = 0;
  ctx->g.row_hi = n;
  ctx->g.adj_lo = 0;
  ctx->g.valid = true;
  return BFB_OK;
}

int copy_edges(bfb_ctx* ctx, uint32_t* out) {
  cudaStream_t s = ctx->stream;
  DevBuf<uint2> e;
  BFB_TRY(e.alloc(ctx->g.m));
  k_expand_edges<<<grid_for(ctx->g.n * 32, 256, ctx->num_sms), 256, 0, s>>>(
      ctx->g.offsets.p, ctx->g.adj.p, ctx->g.n, e.p);
  if (ctx->g.m)
    BFB_CUDA(cudaMemcpyAsync(out, e.p, ctx->g.m * sizeof(uint2), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  return BFB_OK;
}

int partition_1d(bfb_ctx* ctx, int parts, int64_t* out) {
  if (parts < 1) return fail(BFB_ERR_INVALID, "num_parts must be >= 1");
  if (ctx->g.n && parts > ctx->g.n)
    return fail(BFB_ERR_INVALID, "num_parts exceeds the number of vertices");
  DevBuf<int64_t> b;
  BFB_TRY(b.alloc(parts + 1));
  k_partition<<<(parts + 1 + 127) / 128, 128, 0, ctx->stream>>>(ctx->g.offsets.p, ctx->g.n,
                                                                 ctx->g.m, parts, b.p);
  BFB_CUDA(cudaMemcpyAsync(out, b.p, (parts + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                           ctx->stream));
  BFB_CUDA(cudaStreamSynchronize(ctx->stream));
  return BFB_OK;
}

static int nz_prefix(bfb_ctx* ctx, DevBuf<int64_t>& pre, int64_t* ntiles_out) {
  int64_t n = ctx->g.n;
  int64_t ntiles = (n + kNzTile - 1) / kNzTile;
  if (ntiles == 0) ntiles = 1;
  DevBuf<uint32_t> counts;
  BFB_TRY(counts.alloc(ntiles));
  BFB_CUDA(cudaMemsetAsync(counts.p, 0, ntiles * sizeof(uint32_t), ctx->stream));
  if (n) k_nz_tile_counts<<<(unsigned)ntiles, 256, 0, ctx->stream>>>(ctx->g.offsets.p, n, counts.p);
  BFB_TRY(pre.alloc(ntiles + 1));
  DevBuf<int64_t> tmp;
  BFB_TRY(tmp.alloc(scan_tmp_words(ntiles) + 1));
  BFB_TRY(scan_u32_to_i64(counts.p, ntiles, pre.p, tmp.p, ctx->stream));
  BFB_CUDA(cudaStreamSynchronize(ctx->stream));
  *ntiles_out = ntiles;
  return BFB_OK;
}

int count_nonisolated(bfb_ctx* ctx, int64_t* out) {
  DevBuf<int64_t> pre;
  int64_t ntiles = 0;
  BFB_TRY(nz_prefix(ctx, pre, &ntiles));
  BFB_CUDA(cudaMemcpy(out, pre.p + ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost));
  return BFB_OK;
}

int select_nonisolated(bfb_ctx* ctx, const int64_t* ranks, int64_t k, int64_t* out) {
  if (k <= 0) return BFB_OK;
  DevBuf<int64_t> pre;
  int64_t ntiles = 0;
  BFB_TRY(nz_prefix(ctx, pre, &ntiles));
  DevBuf<int64_t> r, o;
  BFB_TRY(r.alloc(k));
  BFB_TRY(o.alloc(k));
  BFB_CUDA(cudaMemcpyAsync(r.p, ranks, k * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  k_nz_select<<<(unsigned)((k + 127) / 128), 128, 0, ctx->stream>>>(ctx->g.offsets.p, ctx->g.n,
                                                                      pre.p, ntiles, r.p, k, o.p);
  BFB_CUDA(cudaMemcpyAsync(out, o.p, k * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  BFB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int64_t i = 0; i < k; ++i)
    if (out[i] < 0) return fail(BFB_ERR_INVALID, "rank out of range");
  return BFB_OK;
}

}  // namespace bfb
