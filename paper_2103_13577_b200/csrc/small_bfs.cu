// Single-CTA ButterFly BFS for small graphs (Alg. 2), the
// whole run in ONE kernel launch.
//
// The level-synchronous engine (bfs_engine.cu) pays a fixed cost per level:
// a host round trip for the frontier count and, per node and per butterfly
// round, a handful of launches.  On small, deep graphs that cost is all there
// is -- a path of 10,000 vertices has up to 10,000 levels of
// one or two vertices, and the paper's Webbase-2001 has "a large tail ... one
// at each level" where "the synchronizations dominate the execution time"
// (PAPER.md:667).  Here one 1024-thread CTA runs every level of every node:
// a level boundary, a butterfly round and the termination test are CTA
// barriers, not launches or host syncs.
//
// State per node g: its visited bitmap (shared memory when
// P x n/8 fits, else global), q_global_next as an explicit vertex list
// (check-and-set appends, SPEC.md:301,310 -- no duplicates), q_local as the
// list of its owned vertices of the current level.  Per level L:
//   phase 1  every node expands its q_local (warp per frontier vertex, lanes
//            over the row): clear bit -> atomicOr claim -> append to its list;
//            the claimant writes u's parent (any claimant is a valid parent:
//            after phase 2 of level L-1 every node knows levels <= L);
//   phase 2  per round of the schedule: snapshot sizes, RunStats
//            accounting (empty sources skipped), then every
//            (dst, src) pair's snapshot merged with the same check-and-set,
//            work flattened over all pairs of the round;
//   commit   node 0's list -> d_local level L+1 and the frontier size; each
//            node's owned vertices of its own list -> its next q_local and the
//            traversed-edge count; termination when node 0's list is empty
//            (SPEC.md:319,349).
// Checks mode (acceptance 8): after phase 2 every node's list must hold the
// same set as node 0's (same size, every member in node 0's bitmap).
//
// Results land where the level-synchronous engine leaves them (node 0's
// d_local and the output parents, in the caller's ids) so read-out,
// validation and RunStats are shared.  Exchange bytes count 4 B per listed
// vertex (the payload of a list snapshot).
#include <algorithm>
#include <cstdlib>

#include "bfb_device.cuh"
#include "bfb_internal.cuh"

namespace bfb {

constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxParts = 64;
constexpr int64_t kSmallMaxN = 1 << 15;        // vertices
constexpr int64_t kSmallMaxM = 1 << 21;        // directed edges
constexpr int kSmallMaxPairs = 8192;           // (dst, src) transfers over all rounds
constexpr size_t kSmallSmemCap = 200 * 1024;   // dynamic shared memory budget
constexpr uint32_t kSmallNone = 0xFFFFFFFFu;

struct SmallStats {
  int64_t levels, remote_messages, remote_vertices, exchange_bytes, traversed_edges, reached,
      disagree;
};

struct SmallEngine {
  int nrounds = 0, max_pairs = 0, total_pairs = 0;
  int64_t nwp = 0;  // words per node bitmap
  bool smem_vis = false;
  size_t smem = 0;
  std::vector<int32_t> round_first;  // host copy, nrounds + 1
  DevBuf<int64_t> bounds;
  DevBuf<uint8_t> pairs;    // total_pairs dst bytes, then total_pairs src bytes
  DevBuf<int32_t> rfirst;   // nrounds + 1
  DevBuf<uint32_t> vis;     // P x nwp (when the bitmaps do not fit in shared memory)
  DevBuf<uint32_t> qnext;   // P x n
  DevBuf<uint32_t> qloc;    // n: node g's q_local at [b[g], b[g] + qn[g])
  DevBuf<int64_t> sizes;    // n + 1 frontier sizes
  DevBuf<SmallStats> stats;
};

namespace {

struct SmallArgs {
  const int64_t* off;
  const uint32_t* adj;
  int64_t n, nwp;
  int P, nrounds;
  const int64_t* bounds;
  const int32_t* rfirst;
  const uint8_t* pdst;
  const uint8_t* psrc;
  int total_pairs, max_pairs;
  uint32_t* gvis;
  uint32_t* qnext;
  uint32_t* qloc;
  uint32_t* level;   // node 0's d_local (caller's ids)
  uint32_t* parent;  // output parents or nullptr
  int64_t* sizes;
  SmallStats* stats;
  int64_t* high_water;  // per node
  int64_t root;
  int checks;
};

// visited probe: shared memory, or global memory read at L2 (the claims are
// L2 atomics; a stale L1 line would only cost an extra atomic, but keep the
// probe where the claims land)
template <bool kSmem>
__device__ __forceinline__ uint32_t vis_load(const uint32_t* p) {
  if (kSmem) return *p;
  return __ldcg(p);
}

// Block-wide exclusive scan of ints (1024 threads); *total = sum.
__device__ __forceinline__ int block_excl_int(int v, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += t;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int w = wsum[lane];
    int wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += t;
    }
    wsum[lane] = wi - w;
    if (lane == 31) wsum[32] = wi;
  }
  __syncthreads();
  const int r = wsum[warp] + inc - v;
  *total = wsum[32];
  __syncthreads();
  return r;
}

// Last index i in [0, cnt) with pre[i] <= t (pre ascending, pre[0] = 0 <= t).
__device__ __forceinline__ int upper_index(const int* pre, int cnt, int t) {
  int lo = 0, hi = cnt - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <bool kSmem>
__global__ void __launch_bounds__(kSmallThreads, 1) k_small_bfs(SmallArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ int64_t b[kSmallMaxParts + 1];
  __shared__ int qn[kSmallMaxParts], nn[kSmallMaxParts], snap[kSmallMaxParts];
  __shared__ int qpre[kSmallMaxParts + 1], lpre[kSmallMaxParts + 1], in_s[kSmallMaxParts];
  __shared__ int64_t hw[kSmallMaxParts];
  __shared__ int wsum[33];
  __shared__ unsigned long long msgs_s, rv_s, trav_s, dis_s;
  __shared__ int64_t reached_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = kSmallThreads / 32;
  const int P = a.P;
  const int64_t n = a.n;
  // dynamic shared memory: pair bytes (dst, src), the per-round pair prefix,
  // then (kSmem) the P bitmaps
  uint8_t* pdst = dyn;
  uint8_t* psrc = dyn + a.total_pairs;
  int* ppre = reinterpret_cast<int*>(dyn + ((2 * (size_t)a.total_pairs + 15) & ~(size_t)15));
  uint32_t* vis = kSmem ? reinterpret_cast<uint32_t*>(ppre + ((a.max_pairs + 4) & ~3)) : a.gvis;
  for (int i = tid; i < a.total_pairs; i += kSmallThreads) {
    pdst[i] = a.pdst[i];
    psrc[i] = a.psrc[i];
  }
  for (int g = tid; g <= P; g += kSmallThreads) b[g] = a.bounds[g];
  for (int64_t i = tid; i < (int64_t)P * a.nwp; i += kSmallThreads) vis[i] = 0;
  for (int64_t i = tid; i < n; i += kSmallThreads) {
    a.level[i] = kSmallNone;
    if (a.parent) a.parent[i] = kSmallNone;
  }
  if (tid < P) {
    hw[tid] = 0;
    in_s[tid] = 0;
  }
  if (tid == 0) {
    msgs_s = rv_s = trav_s = dis_s = 0;
    reached_s = 1;
  }
  __syncthreads();
  const uint32_t root = (uint32_t)a.root;
  if (tid < P) {
    vis[(int64_t)tid * a.nwp + (root >> 5)] = 1u << (root & 31);
    const bool own = (int64_t)root >= b[tid] && (int64_t)root < b[tid + 1];
    qn[tid] = own ? 1 : 0;
    if (own) a.qloc[b[tid]] = root;
  }
  if (tid == 0) {
    a.level[root] = 0;
    if (a.parent) a.parent[root] = root;
    a.sizes[0] = 1;
    trav_s = (unsigned long long)(a.off[root + 1] - a.off[root]);
  }
  __syncthreads();
  uint32_t L = 0;
  while (true) {
    // ---- phase 1
    if (tid < P) nn[tid] = 0;
    if (tid == 0) {
      int s = 0;
      for (int g = 0; g < P; ++g) {
        qpre[g] = s;
        s += qn[g];
      }
      qpre[P] = s;
    }
    __syncthreads();
    const int F = qpre[P];
    for (int k = warp; k < F; k += nwarps) {
      const int g = upper_index(qpre, P, k);
      const uint32_t v = a.qloc[b[g] + (k - qpre[g])];
      uint32_t* vg = vis + (int64_t)g * a.nwp;
      uint32_t* lg = a.qnext + (int64_t)g * n;
      const int64_t e1 = a.off[v + 1];
      for (int64_t e = a.off[v] + lane; e < e1; e += 32) {
        const uint32_t u = a.adj[e];
        const uint32_t bit = 1u << (u & 31);
        if (vis_load<kSmem>(vg + (u >> 5)) & bit) continue;
        if (atomicOr(vg + (u >> 5), bit) & bit) continue;
        lg[atomicAdd(&nn[g], 1)] = u;
        if (a.parent) a.parent[u] = v;
      }
    }
    __syncthreads();
    // ---- phase 2, rounds of the schedule
    for (int r = 0; r < a.nrounds; ++r) {
      const int p0 = a.rfirst[r], np = a.rfirst[r + 1] - p0;
      if (tid < P) snap[tid] = nn[tid];  // round-start snapshot
      __syncthreads();
      int carry = 0;
      for (int base = 0; base < np; base += kSmallThreads) {
        const int i = base + tid;
        int k = 0;
        if (i < np) {
          k = snap[psrc[p0 + i]];
          if (k > 0) {  // empty-source suppression
            atomicAdd(&in_s[pdst[p0 + i]], k);
            atomicAdd(&msgs_s, 1ull);
          }
        }
        int tot;
        const int ex = block_excl_int(k, wsum, &tot);
        if (i < np) ppre[i] = carry + ex;
        carry += tot;
      }
      if (tid < P) {
        const int x = in_s[tid];
        if (x > hw[tid]) hw[tid] = x;
        if (x) atomicAdd(&rv_s, (unsigned long long)x);
        in_s[tid] = 0;
      }
      __syncthreads();
      const int W = carry;
      for (int t = tid; t < W; t += kSmallThreads) {
        const int i = upper_index(ppre, np, t);
        const int src = psrc[p0 + i], dst = pdst[p0 + i];
        const uint32_t u = a.qnext[(int64_t)src * n + (t - ppre[i])];
        const uint32_t bit = 1u << (u & 31);
        uint32_t* vd = vis + (int64_t)dst * a.nwp;
        if (vis_load<kSmem>(vd + (u >> 5)) & bit) continue;
        if (atomicOr(vd + (u >> 5), bit) & bit) continue;
        a.qnext[(int64_t)dst * n + atomicAdd(&nn[dst], 1)] = u;
      }
      __syncthreads();
    }
    // ---- checks mode: every node holds node 0's synchronized frontier
    if (a.checks && P > 1) {
      if (tid > 0 && tid < P && nn[tid] != nn[0]) atomicAdd(&dis_s, 1ull);
      for (int g = 1; g < P; ++g)
        for (int j = tid; j < nn[g]; j += kSmallThreads) {
          const uint32_t u = a.qnext[(int64_t)g * n + j];
          if (!(vis_load<kSmem>(vis + (u >> 5)) & (1u << (u & 31)))) atomicAdd(&dis_s, 1ull);
        }
    }
    // ---- commit: d_local, next q_local, frontier size, traversed edges
    const int F0 = nn[0];  // (nn is next written after the commit's barrier)
    if (tid == 0) {
      int s = 0;
      for (int g = 0; g < P; ++g) {
        lpre[g] = s;
        s += nn[g];
      }
      lpre[P] = s;
    }
    if (tid < P) qn[tid] = 0;  // q_local of level L is no longer read
    __syncthreads();
    const int T = lpre[P];
    unsigned long long trav = 0;
    for (int t = tid; t < T; t += kSmallThreads) {
      const int g = upper_index(lpre, P, t);
      const uint32_t u = a.qnext[(int64_t)g * n + (t - lpre[g])];
      if (g == 0) a.level[u] = L + 1;
      if ((int64_t)u >= b[g] && (int64_t)u < b[g + 1]) {
        a.qloc[b[g] + atomicAdd(&qn[g], 1)] = u;
        trav += (unsigned long long)(a.off[u + 1] - a.off[u]);
      }
    }
    if (trav) atomicAdd(&trav_s, trav);
    __syncthreads();
    if (F0 == 0) break;
    ++L;
    if (tid == 0) {
      a.sizes[L] = F0;
      reached_s += F0;
    }
  }
  if (tid < P) a.high_water[tid] = hw[tid];
  if (tid == 0) {
    SmallStats s;
    s.levels = (int64_t)L + 1;
    s.remote_messages = (int64_t)msgs_s;
    s.remote_vertices = (int64_t)rv_s;
    s.exchange_bytes = 4 * (int64_t)rv_s;
    s.traversed_edges = (int64_t)trav_s;
    s.reached = reached_s;
    s.disagree = (int64_t)dis_s;
    *a.stats = s;
  }
}

}  // namespace

bool small_eligible(const bfb_ctx* ctx, int parts, int total_pairs) {
  const char* e = std::getenv("BFB_SMALL");
  if (e && e[0] == '0') return false;
  return ctx->g.full() && ctx->g.n <= kSmallMaxN && ctx->g.m <= kSmallMaxM &&
         parts <= kSmallMaxParts && total_pairs <= kSmallMaxPairs;
}

void small_release(bfb_ctx* ctx) {
  delete ctx->small;
  ctx->small = nullptr;
}

int small_setup(bfb_ctx* ctx) {
  small_release(ctx);
  const int P = ctx->num_parts;
  std::vector<uint8_t> dst, src;
  std::vector<int32_t> first;
  int max_pairs = 0;
  for (auto& rnd : ctx->schedule) {
    first.push_back((int32_t)dst.size());
    int np = 0;
    for (int g = 0; g < P; ++g)
      for (int s : rnd[g]) {
        dst.push_back((uint8_t)g);
        src.push_back((uint8_t)s);
        ++np;
      }
    max_pairs = std::max(max_pairs, np);
  }
  first.push_back((int32_t)dst.size());
  const int total = (int)dst.size();
  if (!small_eligible(ctx, P, total)) return BFB_OK;
  auto* S = new SmallEngine();
  ctx->small = S;
  const int64_t n = ctx->g.n;
  S->nrounds = (int)ctx->schedule.size();
  S->max_pairs = max_pairs;
  S->total_pairs = total;
  S->nwp = ((n + 31) / 32 + 3) & ~(int64_t)3;
  S->round_first = first;
  const size_t head = ((2 * (size_t)total + 15) & ~(size_t)15) + 4 * (size_t)((max_pairs + 4) & ~3);
  const size_t vis_bytes = (size_t)P * S->nwp * 4;
  S->smem_vis = head + vis_bytes <= kSmallSmemCap;
  S->smem = head + (S->smem_vis ? vis_bytes : 0);
  BFB_TRY(S->bounds.alloc(P + 1));
  BFB_TRY(S->pairs.alloc(2 * (size_t)total + 1));
  BFB_TRY(S->rfirst.alloc(first.size()));
  if (!S->smem_vis) BFB_TRY(S->vis.alloc((size_t)P * S->nwp));
  BFB_TRY(S->qnext.alloc((size_t)P * n));
  BFB_TRY(S->qloc.alloc(n + 1));
  BFB_TRY(S->sizes.alloc(n + 2));
  BFB_TRY(S->stats.alloc(1));
  BFB_CUDA(cudaMemcpy(S->bounds.p, ctx->bounds.data(), (P + 1) * sizeof(int64_t),
                      cudaMemcpyHostToDevice));
  if (total) {
    BFB_CUDA(cudaMemcpy(S->pairs.p, dst.data(), total, cudaMemcpyHostToDevice));
    BFB_CUDA(cudaMemcpy(S->pairs.p + total, src.data(), total, cudaMemcpyHostToDevice));
  }
  BFB_CUDA(cudaMemcpy(S->rfirst.p, first.data(), first.size() * sizeof(int32_t),
                      cudaMemcpyHostToDevice));
  auto kern = S->smem_vis ? k_small_bfs<true> : k_small_bfs<false>;
  BFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->smem));
  return BFB_OK;
}

int small_bfs(bfb_ctx* ctx, int64_t root, uint32_t* level, uint32_t* parent, int64_t* high_water,
              int checks, cudaEvent_t ev0, cudaEvent_t ev1, SmallResult* res) {
  SmallEngine* S = ctx->small;
  cudaStream_t s = ctx->stream;
  SmallArgs a;
  a.off = ctx->g.offsets.p;
  a.adj = ctx->g.adj.p;
  a.n = ctx->g.n;
  a.nwp = S->nwp;
  a.P = ctx->num_parts;
  a.nrounds = S->nrounds;
  a.bounds = S->bounds.p;
  a.rfirst = S->rfirst.p;
  a.pdst = S->pairs.p;
  a.psrc = S->pairs.p + S->total_pairs;
  a.total_pairs = S->total_pairs;
  a.max_pairs = S->max_pairs;
  a.gvis = S->vis.p;
  a.qnext = S->qnext.p;
  a.qloc = S->qloc.p;
  a.level = level;
  a.parent = parent;
  a.sizes = S->sizes.p;
  a.stats = S->stats.p;
  a.high_water = high_water;
  a.root = root;
  a.checks = checks;
  BFB_CUDA(cudaEventRecord(ev0, s));
  if (S->smem_vis)
    k_small_bfs<true><<<1, kSmallThreads, S->smem, s>>>(a);
  else
    k_small_bfs<false><<<1, kSmallThreads, S->smem, s>>>(a);
  BFB_CUDA(cudaGetLastError());
  BFB_CUDA(cudaEventRecord(ev1, s));
  SmallStats st;
  BFB_CUDA(cudaMemcpyAsync(&st, S->stats.p, sizeof(st), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  res->sizes.resize(st.levels);
  BFB_CUDA(cudaMemcpy(res->sizes.data(), S->sizes.p, st.levels * sizeof(int64_t),
                      cudaMemcpyDeviceToHost));
  res->remote_messages = st.remote_messages;
  res->remote_vertices = st.remote_vertices;
  res->exchange_bytes = st.exchange_bytes;
  res->traversed_edges = st.traversed_edges;
  res->reached = st.reached;
  res->disagree = st.disagree;
  return BFB_OK;
}

}  // namespace bfb
