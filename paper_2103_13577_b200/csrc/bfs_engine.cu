// ButterFly BFS engine on device: Alg. 2.
//
// Per level and per node g (a "part": one per GPU in production -- one
// process per GPU, rank_bfs -- or several in one context for testing):
//   phase 1  k_expand_w      warp-centric top-down expansion of q_local[g]
//                            over 256-edge subtiles of 2048-edge tiles
//                            (visited probe + red.or claim; parent store)
//            k_bottom_up     bottom-up phase 1 (direction-optimizing levels)
//   phase 2  per round i of the butterfly schedule:
//            one context:    k_publish (snapshot q_global_next[g] as the
//                            bitmap visited & ~start), k_account
//                            (RunStats), k_merge (OR each scheduled source's
//                            snapshot into g's visited bitmap)
//            one process per node: k_publish_q, k_signal / k_wait (NVLink
//                            mailbox barrier), k_account_mail, k_merge_queue
//                            / k_merge_mail (sources read in peer HBM)
//   commit   k_commit_count -> k_unit_scan_* -> k_commit_write over g's owned
//                            words: new = visited & ~start, levels, start :=
//                            visited, and the next q_local (ascending) with
//                            its degree prefix and tile starts; frontier count
//            k_commit_rest   the level/start update for the other words
//            k_commit_light[_count]  queue-less variants for bottom-up levels
// The synchronized frontier is the bitmap difference; the queue form of
// q_global is never materialised, so no queue-append atomics exist.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "bfb_device.cuh"
#include "bfb_internal.cuh"

namespace bfb {
namespace {

constexpr int kExpandBlock = 256;
// Parent pass (k_commit_count<true>) once this many vertices are reached:
// n >> BFB_PASS_SHIFT (s29 sweeps: first pass build 4 224.4, 6 226.4, 8
// 226.9, 10 226.4, always 221.1 GTEP/s; with the batched, counter-scheduled
// pass and expand 8 243.6, 10 245.4, 12 245.0, 16 244.0).
// With a floor of BFB_PASS_MIN vertices: on s22-s26 graphs the level after a
// small frontier ran the pass with few hubs in `start`, and its row scans
// cost more than phase-1 stores (16 roots, TD GTEP/s, floor none / 2^14 /
// 2^16 / 2^18: s22 ef16 93 / 101 / 106 / 107, s24 ef16 224 / 236 / 242 / 246,
// s26 269 / - / 276 / 277, s29 315 / 315 / 315 / 313).
#ifndef BFB_PASS_SHIFT
#define BFB_PASS_SHIFT 12
#endif
#ifndef BFB_PASS_MIN
#define BFB_PASS_MIN (1 << 16)
#endif
// (the floor is at most n / 64, so small graphs still run the pass)
constexpr int64_t pass_min_reached(int64_t n) {
  const int64_t floor = (int64_t)BFB_PASS_MIN < (n >> 6) ? (int64_t)BFB_PASS_MIN : (n >> 6);
  return (n >> BFB_PASS_SHIFT) > floor ? (n >> BFB_PASS_SHIFT) : floor;
}
#ifndef BFB_EXPAND_ITEMS
#define BFB_EXPAND_ITEMS 12
#endif
// edges per lane per subtile (s29 TD, 16 roots, with the L1/L2 probe policies:
// 10 294.7, 12 297.8, 14 294.4, 16 288.9 GTEP/s; before them 8 was best)
constexpr int kExpandItems = BFB_EXPAND_ITEMS;
constexpr int64_t kSub = 32 * kExpandItems;     // edges per subtile (one warp pass)
#ifndef BFB_SUB_PER_TILE
#define BFB_SUB_PER_TILE 8
#endif
constexpr int kSubPerTile = BFB_SUB_PER_TILE;
constexpr int64_t kTile = kSub * kSubPerTile;   // edges per tile (tile_vstart granularity)
constexpr int kScanItems = 16;                 // commit unit scan: units per thread
constexpr int64_t kScanTile = 256 * kScanItems;
constexpr int64_t kWordPad = 1024;  // bitmap allocation padding (words)
constexpr uint32_t kNone = 0xFFFFFFFFu;
// rank mode: int64 slots per writer in a node's mailbox (see k_signal)
constexpr int kMail = 5;
#ifndef BFB_HOT_LIMIT
#define BFB_HOT_LIMIT (1u << 20)
#endif
constexpr uint32_t kHotLimit = BFB_HOT_LIMIT;  // see probe_vertex
// d_local is materialised once at termination from per-level new-vertex
// bitmaps (one dense 4-byte word per 32 vertices per level, instead of a
// scattered 4-byte store per discovered vertex); levels from kLevelBits on
// (high-diameter graphs) are written directly.
constexpr int kLevelBits = 32;

struct PartView {
  int64_t lo, hi, wlo, whi, nwords;
  uint32_t* visited;
  uint32_t* start;
  uint32_t* level;
  uint32_t* parent;
  uint32_t* pub;
  uint32_t* front;  // level-L frontier bitmap, written at commit when direction != 0
  uint32_t* lvbits; // commit: this level's new-vertex bitmap (levels materialised at the end),
                    // nullptr = write d_local directly (levels >= kLevelBits)
  uint32_t* q_v;
  int64_t* q_pre;
  int64_t* q_base;  // offsets[v] - q_pre: adjacency index = q_base + edge prefix
  uint32_t* tile_vstart;
  int64_t abase, nunits;  // commit units: words [abase, abase + 32 * nunits)
  uint32_t* ucnt;
  int64_t *udeg, *upos, *uepre, *tcnt, *tdeg;
  bool rebuild;  // commit passes: new vertices = the frontier bitmap (queue rebuild)
  PartCounters* ctr;
  const int64_t* off;  // CSR offsets (rows of q_v)
  const uint32_t* nonisol;  // degree > 0 bitmap
  const uint16_t* deg16;    // min(degree, 65535)
  const uint32_t* nbr0;      // lowest-id neighbour per vertex (kNone if absent)
  const uint32_t* nbr1;      // second-lowest (split arrays: the parent pass mostly needs nbr0)
  const uint32_t* nbr0c;     // nbr0 in the caller's ids (the parent stored on a hit, loaded beside
                             // nbr0: no dependent translation before the store)
  const uint32_t* adj;       // CSR adjacency (the commit's parent pass)
  const uint32_t* inv;       // relabelled engine graph: engine id -> caller's id (parents are
                             // stored in the caller's ids), nullptr = identity
  uint32_t hot_limit;        // phase-1 probes of ids below it cache in L1 (probe_vertex)
  const uint32_t* hot_mask;  // several parts: 1 bit per 2^16 ids, the parts' hub blocks (or nullptr)
  uint32_t* sparse_q;        // sparse level: phase 1 appends its claims here (else nullptr)
  bool rest_degrees;         // k_commit_rest also sums the degrees of its new vertices
  bool wide;           // max degree >= 2^26: 32-vertex degree sums need 64 bits
};

// The graph the engine traverses: the degree-ordered relabel when built
// (relabel.cu), else the resident graph itself.
DevGraph& EG(bfb_ctx* ctx) { return ctx->relabeled ? ctx->eg : ctx->g; }
const uint32_t* perm_of(bfb_ctx* ctx) { return ctx->relabeled ? ctx->perm.p : nullptr; }

PartView view_of(bfb_ctx* ctx, Part& p) {
  PartView v;
  v.lo = p.lo;
  v.hi = p.hi;
  v.wlo = p.wlo;
  v.whi = p.whi;
  v.nwords = (ctx->g.n + 31) / 32;
  v.visited = p.visited.p;
  v.start = p.start.p;
  v.level = p.level.p;
  v.parent = p.parent.p;
  v.pub = p.pub.p;
  v.front = ctx->direction ? p.front.p : nullptr;
  v.lvbits = nullptr;
  v.q_v = p.q_v.p;
  v.q_pre = p.q_pre.p;
  v.q_base = p.q_base.p;
  v.tile_vstart = p.tile_vstart.p;
  v.abase = p.wlo & ~(int64_t)31;
  v.nunits = p.whi > p.wlo ? (p.whi - v.abase + 31) / 32 : 0;
  const int64_t nu = v.nunits + 1, nt = (v.nunits + kScanTile - 1) / kScanTile + 1;
  v.ucnt = p.unit_u32.p;
  v.udeg = p.unit_i64.p;
  v.upos = v.udeg + nu;
  v.uepre = v.upos + nu;
  v.tcnt = v.uepre + nu;
  v.tdeg = v.tcnt + nt;
  v.rebuild = false;
  v.ctr = p.ctr.p;
  DevGraph& G = EG(ctx);
  v.off = G.offsets.p;
  v.nonisol = G.nonisol.p;
  v.deg16 = G.deg16.p;
  v.nbr0 = G.first_nbr.p;
  v.nbr1 = G.first_nbr.p + G.first_nbr.n / 3;
  v.nbr0c = G.first_nbr.p + 2 * (G.first_nbr.n / 3);
  v.adj = G.adj_index();
  v.inv = ctx->relabeled ? ctx->inv.p : nullptr;
  v.rest_degrees = false;
  v.hot_limit = ctx->hot_limit;
  v.hot_mask = ctx->hot_mask.n ? ctx->hot_mask.p : nullptr;
  v.sparse_q = nullptr;
  v.wide = ctx->g.max_degree >= ((int64_t)1 << 26);
  return v;
}

// PartView for the commit of level next_level: new-vertex bitmap slot of
// that level (nullptr past kLevelBits: direct d_local writes).
PartView commit_view_of(bfb_ctx* ctx, Part& p, uint32_t next_level) {
  PartView v = view_of(ctx, p);
  const int64_t pad = (int64_t)(p.lvbits.n / kLevelBits);
  v.lvbits = next_level < (uint32_t)kLevelBits ? p.lvbits.p + (int64_t)next_level * pad : nullptr;
  return v;
}

// A vertex id as the caller sees it (parents are stored in the caller's ids,
// so the output needs no id translation of its values).
__device__ __forceinline__ uint32_t caller_id(const PartView& v, uint32_t x) {
  return v.inv ? __ldg(v.inv + x) : x;
}

// ----------------------------------------------------------------- init ---
// root: the caller's id; perm (relabelled engine graph) maps it to the
// engine's id on device, so no host round trip precedes the launch.
__global__ void k_seed(PartView v, const int64_t* __restrict__ off, int64_t root_in,
                       const uint32_t* __restrict__ perm, int owner, RunCounters* run) {
  const int64_t root = perm ? (int64_t)perm[root_in] : root_in;
  const int64_t w = root >> 5;
  const uint32_t b = 1u << (root & 31);
  if (threadIdx.x == 0) {
    v.visited[w] = b;
    v.start[w] = b;
    if (v.front) v.front[w] = b;
    v.level[root] = 0;
    if (v.parent) v.parent[root] = (uint32_t)root_in;  // parents hold the caller's ids
    PartCounters c{};
    if (owner) {
      int64_t d = off[root + 1] - off[root];
      v.q_v[0] = (uint32_t)root;
      v.q_pre[0] = 0;
      v.q_base[0] = off[root];
      c.q_count = 1;
      c.q_edges = d;
      atomicAdd((unsigned long long*)&run->traversed_edges, (unsigned long long)d);
    }
    *v.ctr = c;
  }
  if (owner) {
    int64_t d = off[root + 1] - off[root];
    int64_t nt = (d + kTile - 1) / kTile;
    for (int64_t t = threadIdx.x; t < nt; t += blockDim.x) v.tile_vstart[t] = 0;
  }
}

// ------------------------------------------------------------ phase 1 ----
// Phase 1: top-down expansion of q_local, warp-centric.
// The frontier's edges (degree prefix q_pre over q_local) are cut into
// 2048-edge tiles; tile_vstart[t] is the row holding tile t's first edge
// (written by the commit).  A warp works through a tile in 256-edge
// subtiles, 8 edges per lane, lane-interleaved so the adjacency loads
// coalesce, and resolves each edge's row in registers -- no shared memory, no
// block barriers:
//   lane j loads row rb+j's degree prefix and adjacency base (q_pre, q_base);
//   the starts of rows rb+1..rb+30 inside the subtile become eight 32-bit
//   masks (one warp OR-reduction per 32 positions); an edge's row is rb + the
//   number of row starts at or before it (popc), its base comes from that
//   row's lane by shuffle.  A subtile spanning more than 31 rows (average
//   degree < 8) takes further batches of 31 rows.  Every reached vertex other
//   than an isolated root has degree >= 1, so row starts are distinct.
// Dense levels: one warp per tile, subtiles in order, the row cursor carried.
// Sparse levels (fewer tiles than warps): one warp per subtile, its first
// row found by a 32-ary warp search of q_pre inside the tile's rows, so a
// small frontier still spreads over many warps.
// Per edge: the adjacency word (no L1 allocation, L2 evict-first), a probe
// of the visited bitmap (default caching: its L1 hits matter)
// and, if the probe saw the bit clear, a fire-and-forget red.or claim
// (check-and-set).  The commit finds the new bits as
// visited & ~start, so no claim needs the atomic's old value.
// Parents: every claimant whose probe saw the bit clear stores its row vertex
// as u's parent (plain store, last writer wins).  Each such writer is a
// level-L vertex adjacent to u, and u is discovered at level L+1 (bits set
// before the launch are never seen clear), so any store that lands is a valid
// BFS parent -- no atomic with return on the critical path.
#ifndef BFB_EXPAND_MINB
#define BFB_EXPAND_MINB 4
#endif
// Adjacency words are read once per BFS: no L1 allocation, evict-first in
// L2 (createpolicy), so the streamed adjacency does not push the visited
// bitmap out of either cache.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t adj_word(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ uint32_t probe_word(const uint32_t* p) {
#ifdef BFB_PROBE_NC
  return __ldg(p);
#else
  return *p;
#endif
}

// Probe of vertex u's visited word.  In the relabelled single-node engine
// the hubs are the lowest ids: probes of ids below hot_limit (2^20 vertices,
// a 128 KB slice of the bitmap, sized to stay in L1 next to the expand's
// other loads) cache in L1 as usual, the rest bypass L1 allocation
// (ld.global.L1::no_allocate) so the random cold probes do not evict the hub
// lines, with an L2 evict_last hint so they keep the bitmap resident in L2
// against the streamed adjacency (+1.9%, 16 roots).  s29 TD, 12 roots: no split 275.4, split at 2^18 258.6, 2^19 272.5,
// 2^20 282.5, 2^21 278.4, 2^22 271.7 GTEP/s; hub probes evict_last /
// cold evict_first variants were slower; 1.25 x 2^20, hub probes evict_last
// and the q_local row loads without L1 allocation are within the +-3%
// run-to-run drift of one gpurun call (16 roots, interleaved A/B).  hot_limit = kNone: every probe
// default-cached (several parts: each part's hubs sit at its own start).
template <bool kMask>
__device__ __forceinline__ uint32_t probe_vertex(const uint32_t* visited, uint32_t u,
                                                 uint32_t hot_limit, const uint32_t* hot_mask) {
  const bool hot = kMask ? ((__ldg(hot_mask + (u >> 21)) >> ((u >> 16) & 31)) & 1u) != 0
                         : u < hot_limit;
  if (hot) return probe_word(visited + (u >> 5));
  uint32_t v;
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v) : "l"(visited + (u >> 5)), "l"(pol));
  return v;
}

// Check-and-set of u's visited bit after a probe saw it clear.
// Dense levels: a fire-and-forget red.or (the commit finds the new bits as
// visited & ~start) and every claimant may store a parent.  Sparse levels
// (v.sparse_q): atomicOr with the old value, the winner appends u to the
// claim queue the sparse commit works from, and only it stores the parent.
// Append u to a claim queue: one atomic per warp (the lanes appending right
// now, found by __activemask), so a sparse level with many claims does not
// serialise on the counter.
__device__ __forceinline__ void append_claim(uint32_t* sq, unsigned long long* counter,
                                             uint32_t u) {
  const unsigned m = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
  base = __shfl_sync(m, base, leader);
  sq[base + __popc(m & ((1u << lane) - 1u))] = u;
}

template <bool kSparse>
__device__ __forceinline__ bool claim(const PartView& v, uint32_t* visited, uint32_t u,
                                      uint32_t bit) {
  if (!kSparse) {
    atomicOr(&visited[u >> 5], bit);
    return true;
  }
  if (atomicOr(&visited[u >> 5], bit) & bit) return false;
  append_claim(v.sparse_q, &v.ctr->sq_claims, u);
  return true;
}

// One subtile: edges [r0, r0 + span) of the frontier, rows vs0.. of q_local
// with rb the row holding edge r0 and ve the last row that can matter.
// Returns the row holding edge r0 + kSub (the next subtile's cursor).
template <bool kParents, bool kSparse, bool kMask>
__device__ __forceinline__ uint32_t expand_subtile(const PartView& v,
                                                   const uint32_t* __restrict__ adj, int64_t r0,
                                                   int span, uint32_t rb, uint32_t ve,
                                                   unsigned le_mask, uint64_t pol) {
  const int lane = threadIdx.x & 31;
  const uint32_t vs = rb;
  uint32_t u[kExpandItems];
  uint32_t rows[kExpandItems / 2];  // parents: row - vs, 16 bits per item
  unsigned done = 0;                // items whose row is resolved
  int lo = 0;                       // first position this batch covers
  uint32_t next = rb;
  while (true) {
    const uint32_t row = rb + lane;
    const bool valid = row <= ve;
    const int64_t pre = valid ? __ldg(v.q_pre + row) : INT64_MAX;
    const int64_t base = valid ? __ldg(v.q_base + row) : 0;
    const int64_t relw = pre - r0;
    const int rel = relw > kSub ? (int)kSub + 1 : (int)relw;  // row start, subtile-relative
    const int hi = __shfl_sync(0xffffffffu, rel, 31);        // rows rb..rb+30 end here
    const int cover_hi = min(hi, span);
    const bool mine = lane >= 1 && lane <= 30 && rel > lo && rel < (int)kSub;
    unsigned before = 0;
#pragma unroll
    for (int it = 0; it < kExpandItems; ++it) {
      const unsigned M =
          __reduce_or_sync(0xffffffffu, (mine && (rel >> 5) == it) ? (1u << (rel & 31)) : 0u);
      const int r = it * 32 + lane;
      const int idx = (int)before + __popc(M & le_mask);
      before += __popc(M);
      const int64_t b = __shfl_sync(0xffffffffu, base, idx);
      if (r >= lo && r < cover_hi) {
        u[it] = adj_word(adj + b + r0 + r, pol);
        done |= 1u << it;
        if (kParents) {
          const uint32_t ro = rb + idx - vs;
          rows[it >> 1] = (it & 1) ? ((rows[it >> 1] & 0xFFFFu) | (ro << 16))
                                   : ((rows[it >> 1] & 0xFFFF0000u) | ro);
        }
      }
    }
    if (hi >= span) {
      // the next subtile starts in the row holding position kSub
      const unsigned last = __ballot_sync(0xffffffffu, rel <= (int)kSub && rel > lo);
      next = rb + (31 - __clz((int)(last | 1u)));
      break;
    }
    rb += 31;
    lo = hi;
  }
  uint32_t* __restrict__ visited = v.visited;
  uint32_t wv[kExpandItems];
#pragma unroll
  for (int it = 0; it < kExpandItems; ++it)
    wv[it] = ((done >> it) & 1u) ? probe_vertex<kMask>(visited, u[it], v.hot_limit, v.hot_mask) : 0xFFFFFFFFu;
#pragma unroll
  for (int it = 0; it < kExpandItems; ++it) {
    const uint32_t bit = 1u << (u[it] & 31);
    if (!(wv[it] & bit) && claim<kSparse>(v, visited, u[it], bit)) {
      if (kParents) {
        const uint32_t ro = (rows[it >> 1] >> ((it & 1) * 16)) & 0xFFFFu;
        v.parent[u[it]] = caller_id(v, __ldg(v.q_v + vs + ro));
      }
    }
  }
  return next;
}

// A tile lying inside one row (hub rows: most of the edges of the hub-heavy
// early levels): no row resolution, no per-batch q loads, and each lane keeps
// kRunItems probes in flight.
#ifndef BFB_RUN_ITEMS
#define BFB_RUN_ITEMS 16
#endif
constexpr int kRunItems = BFB_RUN_ITEMS;  // s29 TD, tiles from a counter: 8 241.2, 12 241.3, 16 243.5, 20 242.6, 24 241.0 GTEP/s

template <bool kParents, bool kSparse, bool kMask>
__device__ __forceinline__ void expand_row_run(const PartView& v, const uint32_t* __restrict__ adj,
                                               int64_t e0, int span, uint32_t row, uint64_t pol) {
  const int lane = threadIdx.x & 31;
  const int64_t base = __ldg(v.q_base + row) + e0;
  const uint32_t src = kParents ? caller_id(v, __ldg(v.q_v + row)) : 0u;
  uint32_t* __restrict__ visited = v.visited;
  for (int k = 0; k < span; k += 32 * kRunItems) {
    uint32_t u[kRunItems], wv[kRunItems];
#pragma unroll
    for (int it = 0; it < kRunItems; ++it) {
      const int r = k + it * 32 + lane;
      u[it] = r < span ? adj_word(adj + base + r, pol) : 0u;
    }
#pragma unroll
    for (int it = 0; it < kRunItems; ++it) {
      const int r = k + it * 32 + lane;
      wv[it] = r < span ? probe_vertex<kMask>(visited, u[it], v.hot_limit, v.hot_mask) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int it = 0; it < kRunItems; ++it) {
      const uint32_t bit = 1u << (u[it] & 31);
      if (!(wv[it] & bit) && claim<kSparse>(v, visited, u[it], bit)) {
        if (kParents) v.parent[u[it]] = src;
      }
    }
  }
}

// Row of q_local rows [lo, hi] holding edge position `pos` (the last row whose
// degree prefix is <= pos): 32-ary warp search, 3 steps for a 2048-edge tile.
__device__ __forceinline__ uint32_t find_row(const int64_t* __restrict__ q_pre, uint32_t lo,
                                             uint32_t hi, int64_t pos) {
  const int lane = threadIdx.x & 31;
  while (hi > lo) {
    const uint32_t span = hi - lo;  // answer in [lo, hi]
    const uint32_t step = span / 32 + 1;  // 32 probes cover the span + 1 rows
    const uint32_t cand = lo + (uint32_t)lane * step;
    const bool le = cand <= hi && (lane == 0 || __ldg(q_pre + cand) <= pos);
    const unsigned m = __ballot_sync(0xffffffffu, le);
    const int k = 31 - __clz((int)m);  // last probe at or before pos (lane 0 always)
    const uint32_t nlo = lo + (uint32_t)k * step;
    const uint32_t nhi = min(hi, nlo + step - 1);
    lo = nlo;
    hi = step == 1 ? nlo : nhi;
  }
  return lo;
}

template <bool kParents, bool kSparse, bool kMask>
__global__ void __launch_bounds__(kExpandBlock, BFB_EXPAND_MINB)
    k_expand_w(PartView v, const uint32_t* __restrict__ adj) {
  const int64_t T = v.ctr->q_edges;
  if (T == 0) return;
  const uint32_t qlast = (uint32_t)(v.ctr->q_count - 1);
  const int64_t ntiles = (T + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31;
  const unsigned le_mask = lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u);  // bits [0, lane]
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t pol = l2_evict_first_policy();
  if (ntiles >= nwarps) {
    // tiles handed out from a counter (zeroed by k_commit_prep): hub tiles
    // (run path) and row-resolving tiles differ in cost, and with a static
    // stride the warps that drew the slow ones set the level's tail
    // (s29: expand 30.6 -> 29.3 ms)
    auto grab = [&]() -> int64_t {
      unsigned long long g = 0;
      if (lane == 0) g = atomicAdd((unsigned long long*)&v.ctr->ex_next, 1ull);
      return (int64_t)__shfl_sync(0xffffffffu, g, 0);
    };
    for (int64_t t = grab(); t < ntiles; t = grab()) {
      const int64_t e0 = t * kTile;
      const int span = (int)min(kTile, T - e0);
      const uint32_t ve = (t + 1 < ntiles) ? v.tile_vstart[t + 1] : qlast;
      uint32_t cur = v.tile_vstart[t];
      if (cur == ve) {  // the whole tile inside one row
        expand_row_run<kParents, kSparse, kMask>(v, adj, e0, span, cur, pol);
        continue;
      }
      for (int k = 0; k * kSub < span; ++k)
        cur = expand_subtile<kParents, kSparse, kMask>(v, adj, e0 + k * kSub, min((int)kSub, span - k * (int)kSub),
                                       cur, ve, le_mask, pol);
    }
  } else {
    const int64_t nsub = (T + kSub - 1) / kSub;
    for (int64_t st = gw; st < nsub; st += nwarps) {
      const int64_t t = st / kSubPerTile;
      const int64_t r0 = st * kSub;
      const uint32_t vs = v.tile_vstart[t];
      const uint32_t ve = (t + 1 < ntiles) ? v.tile_vstart[t + 1] : qlast;
      const uint32_t cur = (st % kSubPerTile) ? find_row(v.q_pre, vs, ve, r0) : vs;
      expand_subtile<kParents, kSparse, kMask>(v, adj, r0, (int)min(kSub, T - r0), cur, ve, le_mask, pol);
    }
  }
}

// Launch phase 1 (top-down) for one part on stream s.
// The sparse-level build (claims queued) is a separate instantiation, so the
// dense levels' kernel carries none of its code (registers).
template <bool kParents, bool kMask>
void launch_expand_m(int grid, const PartView& v, const uint32_t* adj, cudaStream_t s) {
  if (v.sparse_q)
    k_expand_w<kParents, true, kMask><<<grid, kExpandBlock, 0, s>>>(v, adj);
  else
    k_expand_w<kParents, false, kMask><<<grid, kExpandBlock, 0, s>>>(v, adj);
}
// (the hub-block mask of several parts is a separate build too: a runtime
// choice in the probe cost the one-node kernel 35% more instructions)
template <bool kParents>
void launch_expand(int grid, const PartView& v, const uint32_t* adj, cudaStream_t s) {
  if (v.hot_mask)
    launch_expand_m<kParents, true>(grid, v, adj, s);
  else
    launch_expand_m<kParents, false>(grid, v, adj, s);
}

template <bool kParents>
int expand_occupancy(int* occ) {
  BFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k_expand_w<kParents, false, false>, kExpandBlock, 0));
  return BFB_OK;
}

// ------------------------------------------------------------ phase 2 ----
// The phase-2 and commit sweeps over whole bitmaps (k_publish, k_merge,
// k_publish_q, k_merge_mail, k_commit_rest) move 4 words per lane per step
// (16-byte loads and stores): one word per lane left them latency-bound at
// ~2 TB/s.  Bitmaps are allocated with kWordPad padding words, zero beyond
// n, so the last chunk may run past nwords.
__device__ __forceinline__ uint4 ld4(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ void st4(uint32_t* p, uint4 x) { *reinterpret_cast<uint4*>(p) = x; }
__device__ __forceinline__ uint4 andnot4(uint4 a, uint4 b) {
  return make_uint4(a.x & ~b.x, a.y & ~b.y, a.z & ~b.z, a.w & ~b.w);
}
__device__ __forceinline__ int popc4(uint4 a) {
  return __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w);
}
__device__ __forceinline__ uint32_t word4(uint4 a, int k) {
  return k == 0 ? a.x : (k == 1 ? a.y : (k == 2 ? a.z : a.w));
}

__global__ void k_publish(PartView v, int parity) {
  int64_t cnt = 0;
  const int64_t nq = (v.nwords + 3) >> 2;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint4 p = andnot4(ld4(v.visited + 4 * q), ld4(v.start + 4 * q));
    st4(v.pub + 4 * q, p);
    cnt += popc4(p);
  }
  __shared__ int64_t red[32];
  cnt = block_sum_i64(cnt, red);
  if (threadIdx.x == 0 && cnt)
    atomicAdd((unsigned long long*)&v.ctr->pub_count[parity], (unsigned long long)cnt);
}

struct RoundDesc {
  const int32_t* pair_dst;   // per pair: receiving node
  const int32_t* pair_src;   // per pair: source node
  const int32_t* node_first; // per node: first pair index (CN+1 entries)
  int npairs;
  int num_nodes;
};

// One block.  Snapshot sizes live in pub_count[round parity] so a round can
// zero the other parity for the next one.
// bytes_per_transfer < 0: queue-form snapshots (sparse levels), 4 B per vertex
__global__ void k_account(RoundDesc rd, PartCounters** ctrs, RunCounters* run, int64_t* high_water,
                          int parity, int64_t bytes_per_transfer) {
  for (int g = threadIdx.x; g < rd.num_nodes; g += blockDim.x) {
    int64_t in = 0, msgs = 0;
    for (int p = rd.node_first[g]; p < rd.node_first[g + 1]; ++p) {
      PartCounters* c = ctrs[rd.pair_src[p]];
      int64_t k = c->pub_count[parity];
      if (k > 0) {  // empty-buffer suppression
        ++msgs;
        in += k;
      }
    }
    if (msgs) {
      atomicAdd((unsigned long long*)&run->remote_messages, (unsigned long long)msgs);
      atomicAdd((unsigned long long*)&run->remote_vertices, (unsigned long long)in);
      atomicAdd((unsigned long long*)&run->exchange_bytes,
                (unsigned long long)(bytes_per_transfer < 0 ? 4 * in : msgs * bytes_per_transfer));
    }
    if (in > high_water[g]) high_water[g] = in;
  }
}

__global__ void k_zero_parity(PartCounters** ctrs, int num_nodes, int parity) {
  for (int g = threadIdx.x; g < num_nodes; g += blockDim.x) {
    ctrs[g]->pub_count[parity] = 0;
  }
}

__global__ void k_merge(RoundDesc rd, uint32_t* const* pubs, uint32_t* const* visiteds,
                        PartCounters** ctrs, int parity, int64_t nwords) {
  const int p = blockIdx.y;
  const int src = rd.pair_src[p];
  const PartCounters* c = ctrs[src];
  if (c->pub_count[parity] == 0) return;
  const uint32_t* __restrict__ pub = pubs[src];
  uint32_t* vis = visiteds[rd.pair_dst[p]];
  const int64_t nq = (nwords + 3) >> 2;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint4 s4 = ld4(pub + 4 * q);
    if (!(s4.x | s4.y | s4.z | s4.w)) continue;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t sw = word4(s4, k);
      if (sw) {
        const uint32_t nb = sw & ~vis[4 * q + k];
        if (nb) atomicOr(&vis[4 * q + k], nb);
      }
    }
  }
}

// Sparse levels, one context: a round's snapshot of node g is its claim
// queue's length at the round start; k_merge_sparse pulls the
// sources' snapshot prefixes and appends what it sets to the receiver's queue
// (appends land past every snapshot prefix, so a node may be read and
// written in the same round).
__global__ void k_snap_sparse(PartCounters** ctrs, int num_nodes, int parity) {
  for (int g = threadIdx.x; g < num_nodes; g += blockDim.x)
    ctrs[g]->pub_count[parity] = (int64_t)ctrs[g]->sq_claims;
}

__global__ void k_merge_sparse(RoundDesc rd, uint32_t* const* sqs, uint32_t* const* visiteds,
                               PartCounters** ctrs, int parity) {
  const int p = blockIdx.y;
  const int src = rd.pair_src[p], dst = rd.pair_dst[p];
  const int64_t k = ctrs[src]->pub_count[parity];
  const uint32_t* __restrict__ q = sqs[src];
  uint32_t* vis = visiteds[dst];
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = q[j];
    const uint32_t bit = 1u << (u & 31);
    if (vis[u >> 5] & bit) continue;
    if (!(atomicOr(&vis[u >> 5], bit) & bit)) append_claim(sqs[dst], &ctrs[dst]->sq_claims, u);
  }
}

// Checks mode (SPEC.md acceptance 8, frontier agreement): after phase 2 every
// node's visited bitmap -- levels <= L plus the synchronized frontier -- must
// equal node 0's; counts the words that differ.
__global__ void k_agree(uint32_t* const* visiteds, int num_nodes, int64_t nwords,
                        RunCounters* run) {
  unsigned long long bad = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t a = visiteds[0][w];
    for (int g = 1; g < num_nodes; ++g) bad += visiteds[g][w] != a;
  }
  if (bad) atomicAdd((unsigned long long*)&run->disagree, bad);
}

// ------------------------------------------------------------- commit ----
__global__ void k_commit_prep(PartCounters** ctrs, int num_nodes) {
  for (int g = threadIdx.x; g < num_nodes; g += blockDim.x) {
    ctrs[g]->frontier = 0;
    ctrs[g]->q_count = 0;
    ctrs[g]->q_edges = 0;
    ctrs[g]->work_next = 0;  // the count pass's unit counter (parent pass)
    ctrs[g]->bu_next = 0;    // the next level's bottom-up group counter
    ctrs[g]->ex_next = 0;    // the next level's top-down tile counter
    ctrs[g]->rest_edges = 0;
  }
}

__device__ __forceinline__ uint32_t owned_mask(int64_t w, int64_t lo, int64_t hi) {
  const int64_t vb = w << 5;
  uint32_t mask = 0xFFFFFFFFu;
  if (vb < lo) mask = (lo - vb) >= 32 ? 0u : (mask << (lo - vb));
  if (vb + 32 > hi) mask &= (hi - vb) <= 0 ? 0u : ((hi - vb) >= 32 ? 0xFFFFFFFFu : ((1u << (hi - vb)) - 1u));
  return mask;
}

// Commit of the owned words, in warp units of 32 words (1024 vertices):
//   k_commit_count  per unit: owned new vertices and their degree sum (from
//                   the 16-bit degree table), the level's new-vertex bitmap
//   k_unit_scan_*   device-wide exclusive scan of the (count, degree) pairs
//   k_commit_write  per unit, from its prefix: q_v, q_pre, q_base, tile
//                   starts, start snapshot -- q_local in ascending order
// Lane = word for the bitmaps; no block barriers.
__device__ __forceinline__ void unit_word(const PartView& v, int64_t unit, int lane, uint32_t& a,
                                          uint32_t& nb, uint32_t& own) {
  const int64_t w = v.abase + unit * 32 + lane;
  const bool in = w >= v.wlo && w < v.whi;
  a = in ? v.visited[w] : 0u;
  if (v.rebuild)
    nb = in ? v.front[w] : 0u;  // this level's new vertices, already committed
  else
    nb = a & ~(in ? v.start[w] : 0u);
  own = nb & owned_mask(w, v.lo, v.hi);
}

// Degree sum of the vertices whose bits are set in x (word w: vertices
// 32w..32w+31) from the 16-bit degree table: the word's 32 degrees are four
// 16-byte loads (a warp reads its unit's 2 KB contiguously); degrees >= 65535
// come from the offsets.
__device__ __forceinline__ int64_t word_degree_sum16(uint32_t x, int64_t w,
                                                     const uint16_t* __restrict__ deg16,
                                                     const int64_t* __restrict__ off) {
  if (!x) return 0;
  const uint4* p = reinterpret_cast<const uint4*>(deg16 + (w << 5));
  uint32_t q[16];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint4 t = __ldg(p + k);
    q[4 * k] = t.x;
    q[4 * k + 1] = t.y;
    q[4 * k + 2] = t.z;
    q[4 * k + 3] = t.w;
  }
  int64_t d = 0;
  bool esc = false;
#pragma unroll
  for (int b = 0; b < 32; ++b) {
    const uint32_t db = (q[b >> 1] >> ((b & 1) * 16)) & 0xFFFFu;
    if ((x >> b) & 1u) {
      d += db;
      esc |= db == 0xFFFFu;
    }
  }
  if (esc) {  // a hub: recount its exact degree (re-reading deg16 keeps q in registers)
    for (uint32_t y = x; y; y &= y - 1) {
      const int64_t u = (w << 5) + __ffs(y) - 1;
      if (__ldg(deg16 + u) == 0xFFFFu) d += (__ldg(off + u + 1) - __ldg(off + u)) - 0xFFFF;
    }
  }
  return d;
}

// Parent pass (kParents; single node, dense levels): phase 1 ran without
// parent stores, and each owned new vertex u of this level takes as parent
// its lowest-id neighbour in `start` -- the vertices of levels <= L, all of
// which are at level L exactly when u is at L + 1 (one at L - 1 or below
// would have discovered u earlier).  `start` is not written before the write
// pass, so the probes see exactly levels <= L.  The two lowest neighbours come
// from the first_nbr table; the row is scanned only when both miss.  One
// store per reached vertex in ascending order replaces phase 1's random
// store per clear-probe claim, and the parent is deterministic.
// `start` is probed at random while the pass streams GBs of first_nbr and
// degree entries: an L2 evict-last hint keeps the 67 MB bitmap resident
// (commit 6.54 -> 6.42 ms at s29).
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// (start is not written while the pass runs, so the load needs no volatile)
__device__ __forceinline__ bool in_start(const uint32_t* __restrict__ start, uint32_t z,
                                         uint64_t pol) {
  uint32_t w;
  asm("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(w) : "l"(start + (z >> 5)), "l"(pol));
  return (w >> (z & 31)) & 1u;
}

// units per counter grab (s29 commit: 1 -> 6.05, 2 -> 5.56, 4 -> 5.48, 8 -> 5.55, 16 -> 5.68 ms)
#ifndef BFB_UNIT_CHUNK
#define BFB_UNIT_CHUNK 4
#endif
constexpr int64_t kUnitChunk = BFB_UNIT_CHUNK;
__device__ __forceinline__ int64_t grab_units(PartCounters* ctr, int lane) {
  unsigned long long u = 0;
  if (lane == 0) u = atomicAdd((unsigned long long*)&ctr->work_next, (unsigned long long)kUnitChunk);
  return (int64_t)__shfl_sync(0xffffffffu, u, 0);
}

#ifndef BFB_PASS_BATCH
#define BFB_PASS_BATCH 4
#endif
constexpr int kPassBatch = BFB_PASS_BATCH;

#ifdef BFB_COUNT_MINB
#define BFB_COUNT_LB __launch_bounds__(256, BFB_COUNT_MINB)
#else
#define BFB_COUNT_LB __launch_bounds__(256)
#endif
template <bool kParents>
__global__ void BFB_COUNT_LB k_commit_count(PartView v, const int64_t* __restrict__ off) {
  __shared__ uint16_t s_list[kParents ? 256 / 32 : 1][kParents ? 1024 : 1];
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t fr = 0, re = 0;
  // with the parent pass a unit's work varies with its new vertices: units
  // are handed out in chunks from a counter (zeroed by k_commit_prep)
  int64_t unit = kParents ? grab_units(v.ctr, lane) : gw;
  int64_t chunk_end = unit + kUnitChunk;
  while (unit < v.nunits) {
    uint32_t a, nb, own;
    unit_word(v, unit, lane, a, nb, own);
    if (!v.rebuild) fr += __popc(nb);  // a rebuild's frontier was counted by its level's commit
    if (v.lvbits && !v.rebuild) {
      const int64_t w = v.abase + unit * 32 + lane;
      if (w >= v.wlo && w < v.whi) v.lvbits[w] = nb;
    }
    const uint32_t c = __reduce_add_sync(0xffffffffu, (unsigned)__popc(own));
    int64_t d = 0;
    if (c) d = warp_sum_i64(word_degree_sum16(own, v.abase + unit * 32 + lane, v.deg16, off));
    // rank mode, direction-optimizing: the new vertices of the partial
    // boundary words that a neighbouring node owns are in neither this
    // node's q_edges nor k_commit_rest's words -- sum them here so every
    // rank's next-frontier degree sum is the same global number
    if (v.rest_degrees && !v.rebuild && (nb & ~own))
      re += word_degree_sum16(nb & ~own, v.abase + unit * 32 + lane, v.deg16, off);
    if (lane == 0) {
      v.ucnt[unit] = c;
      v.udeg[unit] = d;
    }
    if (kParents && c) {
      uint16_t* list = s_list[threadIdx.x >> 5];
      const int cnt = __popc(own);
      int pos = cnt;
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, pos, k);
        if (lane >= k) pos += t;
      }
      pos -= cnt;
      for (uint32_t x = own; x; x &= x - 1) list[pos++] = (uint16_t)((lane << 5) + __ffs(x) - 1);
      __syncwarp();
      const int64_t ubase = (v.abase + unit * 32) << 5;
      const uint64_t pol = l2_evict_last_policy();
      // kPassBatch vertices per lane in flight: their table loads, then
      // their first probes, then the rare second probes / row scans
      for (int k0 = 0; k0 < (int)c; k0 += 32 * kPassBatch) {
        uint32_t u[kPassBatch], f0[kPassBatch], c0[kPassBatch];
        bool hit[kPassBatch];
#pragma unroll
        for (int b = 0; b < kPassBatch; ++b) {
          const int k = k0 + b * 32 + lane;
          u[b] = k < (int)c ? (uint32_t)(ubase + list[k]) : kNone;
          f0[b] = u[b] != kNone ? __ldg(v.nbr0 + u[b]) : kNone;
          c0[b] = u[b] != kNone ? __ldg(v.nbr0c + u[b]) : kNone;
        }
#pragma unroll
        for (int b = 0; b < kPassBatch; ++b)
          hit[b] = f0[b] != kNone && in_start(v.start, f0[b], pol);
#pragma unroll
        for (int b = 0; b < kPassBatch; ++b) {
          if (u[b] == kNone) continue;
          if (hit[b]) {  // the common case: nbr0's caller id was loaded beside nbr0
            v.parent[u[b]] = c0[b];
            continue;
          }
          uint32_t p = kNone;
          uint32_t f1;
          if ((f1 = __ldg(v.nbr1 + u[b])) != kNone && in_start(v.start, f1, pol)) {
            p = f1;
          } else {
            const int64_t e = __ldg(off + u[b] + 1);
            for (int64_t j = __ldg(off + u[b]) + 2; j < e; ++j) {
              const uint32_t z = __ldg(v.adj + j);
              if (in_start(v.start, z, pol)) {
                p = z;
                break;
              }
            }
          }
          v.parent[u[b]] = p == kNone ? kNone : caller_id(v, p);
        }
      }
      __syncwarp();
    }
    if (kParents) {
      if (++unit >= chunk_end) {
        unit = grab_units(v.ctr, lane);
        chunk_end = unit + kUnitChunk;
      }
    } else {
      unit += nw;
    }
  }
  __shared__ int64_t red[32];
  fr = block_sum_i64(fr, red);
  if (threadIdx.x == 0 && fr) atomicAdd((unsigned long long*)&v.ctr->frontier, (unsigned long long)fr);
  if (v.rest_degrees) {
    re = block_sum_i64(re, red);
    if (threadIdx.x == 0 && re)
      atomicAdd((unsigned long long*)&v.ctr->rest_edges, (unsigned long long)re);
  }
}

__global__ void __launch_bounds__(256) k_unit_scan_reduce(PartView v) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  int64_t c = 0, d = 0;
#pragma unroll 4
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + (int64_t)k * 256 + threadIdx.x;
    if (i < v.nunits) {
      c += v.ucnt[i];
      d += v.udeg[i];
    }
  }
  __shared__ int64_t red[32];
  c = block_sum_i64(c, red);
  d = block_sum_i64(d, red);
  if (threadIdx.x == 0) {
    v.tcnt[blockIdx.x] = c;
    v.tdeg[blockIdx.x] = d;
  }
}

// Single block: exclusive scan of the tile sums; totals -> next q_local size
// and edge count (and RunStats.traversed_edges).
__global__ void __launch_bounds__(1024) k_unit_scan_tiles(PartView v, int64_t ntiles,
                                                          RunCounters* run) {
  __shared__ int64_t wsum[33];
  __shared__ int64_t carry_c, carry_d;
  if (threadIdx.x == 0) carry_c = carry_d = 0;
  __syncthreads();
  for (int64_t base = 0; base < ntiles; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int64_t c = i < ntiles ? v.tcnt[i] : 0;
    const int64_t d = i < ntiles ? v.tdeg[i] : 0;
    int64_t tc, td;
    const int64_t ec = block_exclusive_i64(c, wsum, &tc);
    const int64_t ed = block_exclusive_i64(d, wsum, &td);
    const int64_t cc = carry_c, cd = carry_d;
    if (i < ntiles) {
      v.tcnt[i] = cc + ec;
      v.tdeg[i] = cd + ed;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry_c = cc + tc;
      carry_d = cd + td;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    v.ctr->work_next = 0;  // the write pass's unit counter
    v.ctr->q_count = carry_c;
    v.ctr->q_edges = carry_d;
    if (!v.rebuild) atomicAdd((unsigned long long*)&run->traversed_edges, (unsigned long long)carry_d);
  }
}

__global__ void __launch_bounds__(256) k_unit_scan_apply(PartView v) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t c[kScanItems], d[kScanItems];
  int64_t sc = 0, sd = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    c[k] = i < v.nunits ? (int64_t)v.ucnt[i] : 0;
    d[k] = i < v.nunits ? v.udeg[i] : 0;
    sc += c[k];
    sd += d[k];
  }
  __shared__ int64_t wsum[33];
  int64_t tc, td;
  int64_t ec = block_exclusive_i64(sc, wsum, &tc) + v.tcnt[blockIdx.x];
  int64_t ed = block_exclusive_i64(sd, wsum, &td) + v.tdeg[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    if (i < v.nunits) {
      v.upos[i] = ec;
      v.uepre[i] = ed;
    }
    ec += c[k];
    ed += d[k];
  }
}

// Tile starts of 32 consecutive queue rows (one per lane): tiles whose first
// edge lies in a row's [e, e + d) start in that row.  Rows spanning many
// tiles (hubs: up to max_degree / 256) are written by the whole warp.
__device__ __forceinline__ void write_tile_starts(uint32_t* __restrict__ tile_vstart, bool ok,
                                                  int64_t e, int64_t d, int64_t p) {
  const int lane = threadIdx.x & 31;
  const int64_t t0 = ok ? (e + kTile - 1) / kTile : 0;
  const int64_t t1 = ok ? (e + d + kTile - 1) / kTile : 0;
  const bool wide = t1 - t0 > 32;
  if (!wide)
    for (int64_t t = t0; t < t1; ++t) tile_vstart[t] = (uint32_t)p;
  for (unsigned big = __ballot_sync(0xffffffffu, wide); big; big &= big - 1) {
    const int j = __ffs(big) - 1;
    const int64_t a = __shfl_sync(0xffffffffu, t0, j), b = __shfl_sync(0xffffffffu, t1, j);
    const uint32_t pj = (uint32_t)__shfl_sync(0xffffffffu, p, j);
    for (int64_t t = a + lane; t < b; t += 32) tile_vstart[t] = pj;
  }
}

// Write pass, per 32-word unit (1024 vertices) and warp:
//   1. levels >= kLevelBits only (shallower ones come from the level
//      bitmaps at termination): lane = bit, one coalesced store per word;
//   2. the owned new vertices compacted into a per-warp shared list in
//      ascending order (lane = word: position = prefix of the words' counts);
//   3. the list, 32 vertices at a time, lane = vertex: offsets pair, a warp
//      scan of the degrees continuing the unit's edge prefix, and coalesced
//      q_v / q_pre / q_base stores; tile starts for the tiles whose first edge
//      falls in the vertex's row.
// A 32-vertex degree sum fits 32 bits when max degree < 2^26 (kWide = false).
//
// Two builds are launched back to back and the level's new-vertex count
// (ctr->q_count, from the scan) picks the one that runs: kPrefetch (dense
// levels, >= pf_min new vertices) loads the next batch's offsets before the
// current batch's scan and stores, two batches of gathers in flight per warp
// at 44 registers; the plain build keeps 38 registers and one more CTA per SM
// for the sparse levels, which are bound by the per-unit bitmap loads.
#ifdef BFB_WRITE_MINB
#define BFB_WRITE_LB __launch_bounds__(256, BFB_WRITE_MINB)
#else
#define BFB_WRITE_LB __launch_bounds__(256)
#endif
template <bool kWide, bool kPrefetch>
__global__ void BFB_WRITE_LB k_commit_write(PartView v, const int64_t* __restrict__ off,
                                                      uint32_t next_level, int64_t pf_min) {
  if ((v.ctr->q_count >= pf_min) != kPrefetch) return;
  __shared__ uint16_t s_list[256 / 32][1024];  // unit-local vertex index (word * 32 + bit)
  const int lane = threadIdx.x & 31;
  uint16_t* list = s_list[threadIdx.x >> 5];
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // dense levels: units handed out in chunks from a counter (their work
  // varies 0..1024 vertices; a static stride left warps idle at the tail)
  int64_t unit = kPrefetch ? grab_units(v.ctr, lane) : gw;
  int64_t chunk_end = unit + kUnitChunk;
  while (unit < v.nunits) {
    do {
    uint32_t a, nb, own;
    unit_word(v, unit, lane, a, nb, own);
    unsigned m = __ballot_sync(0xffffffffu, nb != 0);
    if (!m) continue;
    const int64_t w0 = v.abase + unit * 32;
    while (m && !v.rebuild && !v.lvbits) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t x = __shfl_sync(0xffffffffu, nb, j);
      if ((x >> lane) & 1u) v.level[((w0 + j) << 5) + lane] = next_level;
    }
    const int cnt = __popc(own);
    int pos = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, pos, d);
      if (lane >= d) pos += t;
    }
    const int total = __shfl_sync(0xffffffffu, pos, 31);
    pos -= cnt;
    for (uint32_t x = own; x; x &= x - 1) list[pos++] = (uint16_t)((lane << 5) + __ffs(x) - 1);
    __syncwarp();
    const int64_t p0 = v.upos[unit];
    int64_t ecarry = v.uepre[unit];
    uint32_t un = 0;
    int64_t o0n = 0, o1n = 0;
    if (kPrefetch) {
      un = lane < total ? (uint32_t)((w0 << 5) + list[lane]) : 0u;
      o0n = lane < total ? __ldg(off + un) : 0;
      o1n = lane < total ? __ldg(off + un + 1) : 0;
    }
    for (int i = 0; i < total; i += 32) {
      const int k = i + lane;
      const bool ok = k < total;
      uint32_t u;
      int64_t o0, d;
      if (kPrefetch) {
        u = un;
        o0 = o0n;
        d = o1n - o0n;
        if (i + 32 < total) {
          const bool okn = k + 32 < total;
          un = okn ? (uint32_t)((w0 << 5) + list[k + 32]) : 0u;
          o0n = okn ? __ldg(off + un) : 0;
          o1n = okn ? __ldg(off + un + 1) : 0;
        }
      } else {
        u = ok ? (uint32_t)((w0 << 5) + list[k]) : 0u;
        o0 = ok ? __ldg(off + u) : 0;
        d = ok ? __ldg(off + u + 1) - o0 : 0;
      }
      int64_t inc;
      if (kWide) {
        inc = warp_inclusive_i64(d);
      } else {
        int x = (int)d;
#pragma unroll
        for (int s2 = 1; s2 < 32; s2 <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, x, s2);
          if (lane >= s2) x += t;
        }
        inc = x;
      }
      const int64_t e = ecarry + inc - d;
      const int64_t p = p0 + k;
      if (ok) {
        v.q_v[p] = u;
        v.q_pre[p] = e;
        v.q_base[p] = o0 - e;
      }
      write_tile_starts(v.tile_vstart, ok, e, d, p);
      ecarry += __shfl_sync(0xffffffffu, inc, 31);
    }
    __syncwarp();
    if (nb && !v.rebuild) {
      v.start[w0 + lane] = a;
      if (v.front) v.front[w0 + lane] = nb;
    }
    } while (0);
    if (kPrefetch) {
      if (++unit >= chunk_end) {
        unit = grab_units(v.ctr, lane);
        chunk_end = unit + kUnitChunk;
      }
    } else {
      unit += nw;
    }
  }
}

// Commit of a sparse level (one node, top-down): the phase-1 claims (one
// per new vertex, atomicOr winners) replace the count / scan / write sweeps
// over the whole bitmap.  Per claimed vertex u: d_local written directly
// (this level's lvbits slice stays unwritten; the materialisation skips it),
// u's start bit set, and a q_local row.  Rows and their degree prefix come
// from one block-aggregated 64-bit atomic on (row count << 40) + edge count,
// so q_pre is ascending in row order without a device-wide scan; tile starts
// for the tiles whose first edge falls in the row.  k_sparse_finalize turns
// the packed totals into the next frontier's counters.
constexpr int kPackShift = 40;
#ifndef BFB_SPARSE_SHIFT
#define BFB_SPARSE_SHIFT 5  // sparse levels: at most n >> this many frontier edges
#endif
#ifndef BFB_SPARSE_CAP
#define BFB_SPARSE_CAP (1 << 23)  // ... and at most this many (the packed row count is 24 bits)
#endif
__global__ void __launch_bounds__(256) k_sparse_commit(PartView v, const int64_t* __restrict__ off,
                                                       uint32_t next_level) {
  __shared__ int64_t wsum[33];
  __shared__ unsigned long long base;
  const int64_t nq = (int64_t)v.ctr->sq_claims;
  for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < nq; b0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    const bool ok = i < nq;
    uint32_t u = 0;
    int64_t o = 0, d = 0;
    bool own = false;
    if (ok) {
      u = v.sparse_q[i];
      v.level[u] = next_level;
      atomicOr(&v.start[u >> 5], 1u << (u & 31));
      if (v.front) atomicOr(&v.front[u >> 5], 1u << (u & 31));  // the next bottom-up level's frontier
      own = (int64_t)u >= v.lo && (int64_t)u < v.hi;
      if (own) {
        o = __ldg(off + u);
        d = __ldg(off + u + 1) - o;
      } else if (v.rest_degrees) {
        // rank mode, direction-optimizing: the next frontier's non-owned edges
        atomicAdd((unsigned long long*)&v.ctr->rest_edges,
                  (unsigned long long)(__ldg(off + u + 1) - __ldg(off + u)));
      }
    }
    // q_local rows: the owned new vertices only (one node: all of them)
    int64_t tot_d;
    const int64_t ed = block_exclusive_i64(d, wsum, &tot_d);
    int64_t tot_c;
    const int64_t ec = block_exclusive_i64(own ? 1 : 0, wsum, &tot_c);
    if (threadIdx.x == 0)
      base = atomicAdd(&v.ctr->sq_packed,
                       ((unsigned long long)tot_c << kPackShift) + (unsigned long long)tot_d);
    __syncthreads();
    const unsigned long long bb = base;
    __syncthreads();
    if (own) {
      const int64_t row = (int64_t)(bb >> kPackShift) + ec;
      const int64_t e = (int64_t)(bb & ((1ull << kPackShift) - 1)) + ed;
      v.q_v[row] = u;
      v.q_pre[row] = e;
      v.q_base[row] = o - e;
      for (int64_t t = (e + kTile - 1) / kTile; t < (e + d + kTile - 1) / kTile; ++t)
        v.tile_vstart[t] = (uint32_t)row;
    }
  }
}

__global__ void k_sparse_finalize(PartCounters* ctr, RunCounters* run) {
  const unsigned long long pk = ctr->sq_packed;
  const int64_t cnt = (int64_t)(pk >> kPackShift), edges = (int64_t)(pk & ((1ull << kPackShift) - 1));
  ctr->q_count = cnt;
  ctr->q_edges = edges;
  ctr->frontier = (int64_t)ctr->sq_claims;  // every new vertex, owned or not
  ctr->sq_claims = 0;
  ctr->sq_packed = 0;
  run->traversed_edges += edges;
}

// Thin levels (one node, top-down): consecutive levels whose frontier has at
// most kTailEdges (2^13) edges run inside ONE single-CTA launch -- expand (warp per
// frontier vertex, lanes over its row, atomicOr winners appended to the
// claim queue, parents by the winners), then the commit of the claimed
// vertices (d_local directly, start bit, q_local rows with their degree
// prefix by a block scan, tile starts) -- with CTA barriers between the
// steps instead of launches and a host round trip per level.  Long thin tails
// (the paper's Webbase-2001, "one at each level"; deep paths)
// cost ~microseconds per level instead of ~20.  The launch stops after
// kTailMax levels, on an empty frontier, or when the frontier outgrows
// kTailEdges; the state it leaves (q_local, counters) is the one the
// level-synchronous passes continue from.
// one SM expands a thin level; past ~8K edges the grid-wide passes win
// (s29 TD, 16 roots: 2^15 309.6, 2^13 314.4, 2^12 313.3, 2^10 314.5 GTEP/s)
#ifndef BFB_TAIL_EDGES
#define BFB_TAIL_EDGES (1 << 13)
#endif
constexpr int64_t kTailEdges = BFB_TAIL_EDGES;
constexpr int kTailMax = 4096;
constexpr int kTailThreads = 1024;
constexpr int kTailBig = (int)(kTailEdges / 33) + 1;  // rows of > 32 edges a thin level can hold
struct TailOut {
  int64_t levels;  // levels committed (the last may be empty: the BFS ended)
};

template <bool kParents>
__global__ void __launch_bounds__(kTailThreads, 1) k_tail(PartView v, const int64_t* __restrict__ off,
                                                          const uint32_t* __restrict__ adj,
                                                          uint32_t level0, RunCounters* run,
                                                          int64_t* sizes, TailOut* out) {
  __shared__ unsigned long long cnt_s;
  __shared__ int64_t wsum[33];
  __shared__ int64_t carry_e, carry_r;
  __shared__ unsigned nbig_s;
  __shared__ uint32_t big_s[kTailBig];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = kTailThreads / 32;
  uint32_t L = level0;
  int done = 0;
  while (done < kTailMax) {
    const int64_t qn = ((volatile PartCounters*)v.ctr)->q_count;
    const int64_t qe = ((volatile PartCounters*)v.ctr)->q_edges;
    if (qn == 0 || qe > kTailEdges) break;
    if (tid == 0) cnt_s = 0;
    __syncthreads();
    // phase 1 over q_local (rows in q_v): a thread per frontier vertex of
    // degree <= 32 (a thin level's frontier can still hold thousands of
    // low-degree vertices), the longer rows queued for a warp each
    if (tid == 0) nbig_s = 0;
    __syncthreads();
    for (int64_t k = tid; k < qn; k += kTailThreads) {
      const uint32_t x = v.q_v[k];
      const int64_t e0 = off[x], e1 = off[x + 1];
      if (e1 - e0 > 32) {
        const unsigned slot = atomicAdd(&nbig_s, 1u);
        if (slot < kTailBig) big_s[slot] = x;
        continue;
      }
      for (int64_t j = e0; j < e1; ++j) {
        const uint32_t z = adj[j];
        const uint32_t bit = 1u << (z & 31);
        if (__ldcg(v.visited + (z >> 5)) & bit) continue;
        if (atomicOr(v.visited + (z >> 5), bit) & bit) continue;
        v.sparse_q[atomicAdd(&cnt_s, 1ull)] = z;
        if (kParents) v.parent[z] = caller_id(v, x);
      }
    }
    __syncthreads();
    // rows longer than 32: a warp each (kTailEdges bounds them to kTailBig)
    for (unsigned k = warp; k < min(nbig_s, (unsigned)kTailBig); k += nwarps) {
      const uint32_t x = big_s[k];
      const int64_t e1 = off[x + 1];
      for (int64_t j = off[x] + lane; j < e1; j += 32) {
        const uint32_t z = adj[j];
        const uint32_t bit = 1u << (z & 31);
        if (__ldcg(v.visited + (z >> 5)) & bit) continue;
        if (atomicOr(v.visited + (z >> 5), bit) & bit) continue;
        v.sparse_q[atomicAdd(&cnt_s, 1ull)] = z;
        if (kParents) v.parent[z] = caller_id(v, x);
      }
    }
    __syncthreads();
    const int64_t nc = (int64_t)cnt_s;
    if (tid == 0) carry_e = carry_r = 0;
    __syncthreads();
    // commit of the claimed vertices, rows in claim order
    for (int64_t b0 = 0; b0 < nc; b0 += kTailThreads) {
      const int64_t i = b0 + tid;
      uint32_t u = 0;
      int64_t o = 0, d = 0;
      if (i < nc) {
        u = v.sparse_q[i];
        o = off[u];
        d = off[u + 1] - o;
        v.level[u] = L + 1;
        atomicOr(v.start + (u >> 5), 1u << (u & 31));
      }
      int64_t tot;
      const int64_t ex = block_exclusive_i64(d, wsum, &tot);
      if (i < nc) {
        const int64_t e = carry_e + ex;
        v.q_v[i] = u;
        v.q_pre[i] = e;
        v.q_base[i] = o - e;
        for (int64_t t = (e + kTile - 1) / kTile; t < (e + d + kTile - 1) / kTile; ++t)
          v.tile_vstart[t] = (uint32_t)i;
      }
      __syncthreads();
      if (tid == 0) carry_e += tot;
      __syncthreads();
    }
    if (tid == 0) {
      v.ctr->q_count = nc;
      v.ctr->q_edges = carry_e;
      v.ctr->frontier = nc;
      run->traversed_edges += carry_e;
      sizes[done] = nc;
    }
    __threadfence_block();
    __syncthreads();
    ++done;
    ++L;
    if (nc == 0) break;
  }
  if (tid == 0) out->levels = done;
}

// Queue-less commit of a bottom-up level in one pass (the next phase 1 is
// bottom-up again, which reads only bitmaps): per 32-word unit, levels of the
// new vertices (lane = bit, coalesced), start := visited, the frontier
// bitmap, and the totals -- frontier, owned new vertices and their degree sum
// (q_count / q_edges for the direction heuristic, RunStats traversed edges).
// If the heuristic then switches to top-down, the queue is rebuilt from the
// frontier bitmap by the regular count -> scan -> write passes (PartView
// rebuild).
__global__ void __launch_bounds__(256) k_commit_light_count(PartView v, const int64_t* __restrict__ off,
                                                            uint32_t next_level, RunCounters* run) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t fr = 0, qc = 0, qe = 0, re = 0;
  for (int64_t unit = gw; unit < v.nunits; unit += nw) {
    uint32_t a, nb, own;
    unit_word(v, unit, lane, a, nb, own);
    const int64_t w0 = v.abase + unit * 32;
    if (v.lvbits && w0 + lane >= v.wlo && w0 + lane < v.whi) v.lvbits[w0 + lane] = nb;
    unsigned m = __ballot_sync(0xffffffffu, nb != 0);
    if (!m) continue;
    while (m && !v.lvbits) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t x = __shfl_sync(0xffffffffu, nb, j);
      if ((x >> lane) & 1u) v.level[((w0 + j) << 5) + lane] = next_level;
    }
    if (nb) {
      v.start[w0 + lane] = a;
      if (v.front) v.front[w0 + lane] = nb;
      fr += __popc(nb);
    }
    if (own) {
      qc += __popc(own);
      qe += word_degree_sum16(own, w0 + lane, v.deg16, off);
    }
    if (v.rest_degrees && (nb & ~own)) re += word_degree_sum16(nb & ~own, w0 + lane, v.deg16, off);
  }
  __shared__ int64_t red[32];
  fr = block_sum_i64(fr, red);
  qc = block_sum_i64(qc, red);
  qe = block_sum_i64(qe, red);
  if (v.rest_degrees) {
    re = block_sum_i64(re, red);
    if (threadIdx.x == 0 && re)
      atomicAdd((unsigned long long*)&v.ctr->rest_edges, (unsigned long long)re);
  }
  if (threadIdx.x == 0) {
    if (fr) atomicAdd((unsigned long long*)&v.ctr->frontier, (unsigned long long)fr);
    if (qc) atomicAdd((unsigned long long*)&v.ctr->q_count, (unsigned long long)qc);
    if (qe) {
      atomicAdd((unsigned long long*)&v.ctr->q_edges, (unsigned long long)qe);
      atomicAdd((unsigned long long*)&run->traversed_edges, (unsigned long long)qe);
    }
  }
}

// Commit without the queue: levels (coalesced, lane = bit), start := visited
// and the frontier bitmap for the owned words.
__global__ void __launch_bounds__(256) k_commit_light(PartView v, uint32_t next_level) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t unit = gw; unit < v.nunits; unit += nw) {
    uint32_t a, nb, own;
    unit_word(v, unit, lane, a, nb, own);
    unsigned m = __ballot_sync(0xffffffffu, nb != 0);
    if (!m) continue;
    const int64_t w0 = v.abase + unit * 32;
    while (m && !v.lvbits) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t x = __shfl_sync(0xffffffffu, nb, j);
      if ((x >> lane) & 1u) v.level[((w0 + j) << 5) + lane] = next_level;
    }
    if (nb) {
      v.start[w0 + lane] = a;
      if (v.front) v.front[w0 + lane] = nb;
    }
  }
}

// Commit of the words outside this node's owned range (its replicated
// d_local): the level's new-vertex bitmap (or, past kLevelBits,
// the levels themselves), start := visited, the frontier bitmap and the
// frontier count.  Warp = 32 consecutive words (lane = word for the bitmaps,
// lane = bit for coalesced level stores).
__global__ void __launch_bounds__(256) k_commit_rest(PartView v, uint32_t next_level) {
  const int lane = threadIdx.x & 31;
  // 4-word chunks of [0, wlo) and [whi, nwords): chunk indices [0, ca) and
  // [cb, cn), words of the owned range [wlo, whi) masked out
  const int64_t ca = (v.wlo + 3) >> 2, cb = max(v.whi >> 2, ca), cn = (v.nwords + 3) >> 2;
  const int64_t nch = ca + (cn > cb ? cn - cb : 0);
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t fr = 0, re = 0;
  for (int64_t base = gw * 32; base < nch; base += nw * 32) {
    const int64_t i = base + lane;
    const bool in = i < nch;
    const int64_t c = i < ca ? i : cb + (i - ca);
    const int64_t w0 = 4 * c;
    uint4 a = make_uint4(0, 0, 0, 0), nb4 = a;
    if (in) {
      a = ld4(v.visited + w0);
      nb4 = andnot4(a, ld4(v.start + w0));
    }
    uint32_t nbk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t w = w0 + k;
      const bool mine = in && (w < v.wlo || w >= v.whi) && w < v.nwords;
      nbk[k] = mine ? word4(nb4, k) : 0u;
      if (v.lvbits && mine) v.lvbits[w] = nbk[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      unsigned m = __ballot_sync(0xffffffffu, nbk[k] != 0);
      while (m && !v.lvbits) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t x = __shfl_sync(0xffffffffu, nbk[k], j);
        const int64_t wj = __shfl_sync(0xffffffffu, w0 + k, j);
        if ((x >> lane) & 1u) v.level[(wj << 5) + lane] = next_level;
      }
      if (nbk[k]) {
        const int64_t w = w0 + k;
        fr += __popc(nbk[k]);
        v.start[w] = word4(a, k);
        if (v.front) v.front[w] = nbk[k];
        if (v.rest_degrees) re += word_degree_sum16(nbk[k], w, v.deg16, v.off);
      }
    }
  }
  __shared__ int64_t red[32];
  fr = block_sum_i64(fr, red);
  if (threadIdx.x == 0 && fr) atomicAdd((unsigned long long*)&v.ctr->frontier, (unsigned long long)fr);
  if (v.rest_degrees) {
    re = block_sum_i64(re, red);
    if (threadIdx.x == 0 && re)
      atomicAdd((unsigned long long*)&v.ctr->rest_edges, (unsigned long long)re);
  }
}

// ------------------------------------------------------- bottom-up phase 1 --
// Direction-optimizing phase 1 (Beamer et al.): every owned
// unvisited vertex scans its row (ascending ids, so hubs first) for a
// neighbour in the level-L frontier bitmap and claims itself on the first hit.
// Discoveries are owned vertices only; phase 2 and the commit are unchanged,
// so levels, frontier sizes and traversed edges are identical to
// top-down.  A warp takes 32 bitmap words at a time (one coalesced load of
// their visited / non-isolated bits), then walks the words that have
// candidates with lane = vertex: first the vertex's lowest-id neighbour from
// a per-vertex table, then the rest of its row, kBuBatch neighbours per
// round trip.
constexpr int kBuBatch = 2;  // measured: 1 -> 607, 2 -> 611, 4 -> 554, 8 -> 455 GTEP/s (s29 DO)

#ifdef BFB_BU_MINB
#define BFB_BU_LB __launch_bounds__(256, BFB_BU_MINB)
#else
#define BFB_BU_LB __launch_bounds__(256)
#endif
template <bool kParents>
__global__ void BFB_BU_LB k_bottom_up(PartView v, const uint32_t* __restrict__ adj,
                                                   unsigned long long* examined) {
  const int lane = threadIdx.x & 31;
  const uint32_t* __restrict__ front = v.front;
  unsigned long long ex = 0;
  // 32 words per step: lane k reads word k's visited / non-isolated bits
  // (one coalesced load each), then the warp walks the words with candidates
  // Groups are handed out from a counter (zeroed by k_commit_prep): the
  // candidates' row scans vary widely, and a static stride left most warps
  // idle behind the slowest (s29 DO 892 -> 954 GTEP/s).
  auto grab = [&]() -> int64_t {
    unsigned long long g = 0;
    if (lane == 0) g = atomicAdd((unsigned long long*)&v.ctr->bu_next, 1ull);
    return v.wlo + 32 * (int64_t)__shfl_sync(0xffffffffu, g, 0);
  };
  for (int64_t w0 = grab(); w0 < v.whi; w0 = grab()) {
    const int64_t wk = w0 + lane;
    const uint32_t vis_k = wk < v.whi ? v.visited[wk] : 0xFFFFFFFFu;
    const uint32_t cand_k = wk < v.whi ? owned_mask(wk, v.lo, v.hi) & ~vis_k & v.nonisol[wk] : 0u;
    // the next candidate word's nbr0 / degree entries are loaded while the
    // current word is decided (one round trip less per word)
    unsigned todo = __ballot_sync(0xffffffffu, cand_k != 0);
    uint32_t fx_n = 0;
    uint16_t dg_n = 0;
    if (todo) {
      const int jn = __ffs(todo) - 1;
      const uint32_t cn = __shfl_sync(0xffffffffu, cand_k, jn);
      const int64_t un = ((w0 + jn) << 5) + lane;
      if ((cn >> lane) & 1u) {
        fx_n = __ldg(v.nbr0 + un);
        dg_n = __ldg(v.deg16 + un);
      }
    }
    for (; todo; ) {
      const int jw = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t fx = fx_n;
      const uint16_t dg = dg_n;
      if (todo) {
        const int jn = __ffs(todo) - 1;
        const uint32_t cn = __shfl_sync(0xffffffffu, cand_k, jn);
        const int64_t un = ((w0 + jn) << 5) + lane;
        if ((cn >> lane) & 1u) {
          fx_n = __ldg(v.nbr0 + un);
          dg_n = __ldg(v.deg16 + un);
        }
      }
      const int64_t w = w0 + jw;
      const uint32_t vis = __shfl_sync(0xffffffffu, vis_k, jw);
      const uint32_t cand = __shfl_sync(0xffffffffu, cand_k, jw);
      const int64_t u = (w << 5) + lane;
      bool found = false, first = false;  // first: found at nbr0 (its caller id is tabled)
      uint32_t par = 0;
      const bool is_cand = (cand >> lane) & 1u;
      int64_t b = 0, e = 0;
      bool more = false;
      if (is_cand) {
        // the two lowest-id neighbours (hubs, on Kronecker graphs) decide most
        // candidates -- all of those with degree <= 2 -- from a per-vertex
        // table read coalesced across the warp; only the rest load the row
        more = dg > 2;
        ++ex;
        if ((front[fx >> 5] >> (fx & 31)) & 1u) {
          found = true;
          par = fx;
          first = true;
        } else {
          const uint32_t fy = __ldg(v.nbr1 + u);
          if (fy != kNone) {
            ++ex;
            if ((front[fy >> 5] >> (fy & 31)) & 1u) {
              found = true;
              par = fy;
            }
          }
        }
      }
      if (is_cand && !found && more) {
        b = __ldg(v.off + u) + 2;
        e = __ldg(v.off + u + 1);
        for (int64_t j = b; j < e && !found; j += kBuBatch) {
          uint32_t p[kBuBatch];
          bool hit[kBuBatch];
#pragma unroll
          for (int k = 0; k < kBuBatch; ++k) p[k] = j + k < e ? ld_stream_u32(adj + j + k) : 0u;
#pragma unroll
          for (int k = 0; k < kBuBatch; ++k)
            hit[k] = j + k < e && ((front[p[k] >> 5] >> (p[k] & 31)) & 1u);
#pragma unroll
          for (int k = 0; k < kBuBatch; ++k) {
            if (!found && j + k < e) {
              ++ex;
              if (hit[k]) {
                found = true;
                par = p[k];
              }
            }
          }
        }
      }
      const uint32_t nbits = __ballot_sync(0xffffffffu, found);
      if (lane == 0 && nbits) v.visited[w] = vis | nbits;  // this node is the word's only writer
      if (kParents && found) v.parent[u] = first ? __ldg(v.nbr0c + u) : caller_id(v, par);
    }
  }
  ex = (unsigned long long)warp_sum_i64((int64_t)ex);
  if (lane == 0 && ex) atomicAdd(examined, ex);
}

// d_local at termination: vertex u gets the level l in
// [1, nl] whose new-vertex bitmap holds it; otherwise, if visited, the value
// already in d_local (the root's 0, or a level >= kLevelBits written
// directly); otherwise UNREACHED.  Warp = 32 consecutive words: lane k loads
// word k of every level bitmap (coalesced, all in flight at once) and folds
// them into bit slices of the level index, then lanes take 4 vertices each
// (shuffles) and write d_local with 16-byte stores, 512 contiguous bytes per
// warp store.
// Bit slices of one unit (32 words): lane k folds word k of every level
// bitmap into five words holding bit k of the level index for each of the
// word's 32 vertices, plus "in some bitmap" and the visited word.
struct LevelSlices {
  uint32_t s[5], any, vis;
};

__device__ __forceinline__ void load_level_slices(const uint32_t* __restrict__ lvbits, int64_t pad,
                                                  int nl, uint32_t valid,
                                                  const uint32_t* __restrict__ visited,
                                                  int64_t wk, bool in, LevelSlices& L) {
#pragma unroll
  for (int k = 0; k < 5; ++k) L.s[k] = 0u;
  L.any = 0u;
  if (in) {
    // groups of 8 levels: the group's loads issue together, then fold; fully
    // unrolled, so each level's bits are compile-time (one OR per set bit)
#pragma unroll
    for (int g0 = 1; g0 < kLevelBits; g0 += 8) {
      if (g0 > nl) break;
      uint32_t x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int l = g0 + j;
        x[j] = (l < kLevelBits && l <= nl && ((valid >> l) & 1u)) ? __ldg(lvbits + l * pad + wk) : 0u;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int l = g0 + j;
        if (l >= kLevelBits) break;
        L.any |= x[j];
#pragma unroll
        for (int k = 0; k < 5; ++k)
          if ((l >> k) & 1) L.s[k] |= x[j];
      }
    }
  }
  L.vis = in ? __ldg(visited + wk) : 0u;
}

// Bits 0..3 of n to bit 0 of bytes 0..3 (the four copies n << 7i do not
// overlap, so the product has no carries).
__device__ __forceinline__ uint32_t spread4(uint32_t n) { return (n * 0x00204081u) & 0x01010101u; }

// Byte t of x as a uint32, its top bit replicated into bytes 1..3 (prmt sign
// mode): 0xFF -> 0xFFFFFFFF (UNREACHED), levels < 128 zero-extended.
template <int t>
__device__ __forceinline__ uint32_t byte_sext(uint32_t x) {
  uint32_t r;
  constexpr uint32_t sel = t | ((8 | t) << 4) | ((8 | t) << 8) | ((8 | t) << 12);
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(x), "n"(sel));
  return r;
}

// d_local of one unit from its slices: 8 passes of 128 vertices, lane = 4
// consecutive vertices of word q * 4 + lane / 8, one 16-byte store each (a
// warp writes 512 contiguous bytes per pass).
__device__ __forceinline__ void store_unit_levels(const LevelSlices& L, int64_t w0,
                                                  uint32_t* __restrict__ level, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int sub = lane >> 3, b0 = (lane & 7) * 4;
#pragma unroll 2
  for (int q = 0; q < 8; ++q) {
    const int j = q * 4 + sub;
    uint32_t sl[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) sl[k] = __shfl_sync(0xffffffffu, L.s[k], j) >> b0;
    const uint32_t aj = __shfl_sync(0xffffffffu, L.any, j) >> b0;
    const uint32_t vj = __shfl_sync(0xffffffffu, L.vis, j) >> b0;
    const int64_t u0 = ((w0 + j) << 5) + b0;
    if (u0 >= n) continue;
    // byte t = level of vertex u0 + t (bit k from slice k), 0xFF if in no bitmap
    uint32_t bytes = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) bytes |= spread4(sl[k] & 0xFu) << k;
    const uint32_t f = aj & 0xFu;
    bytes |= ~(spread4(f) * 0xFFu);
    const uint32_t lv[4] = {byte_sext<0>(bytes), byte_sext<1>(bytes), byte_sext<2>(bytes),
                            byte_sext<3>(bytes)};
    const bool keep = (vj & ~f & 0xFu) != 0u;  // visited, level in d_local already
    if (u0 + 4 <= n && !keep) {
      *reinterpret_cast<uint4*>(level + u0) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
    } else {
      for (int t = 0; t < 4 && u0 + t < n; ++t)
        if (((aj >> t) & 1u) || !((vj >> t) & 1u)) level[u0 + t] = lv[t];
    }
  }
}

// Byte form (relabelled engine graph, whose d_local is only ever read back
// through the un-permute gather): one byte per vertex -- the level 1..31 from
// the bitmaps, kLv8Keep where d_local holds it (the root's 0, levels >=
// kLevelBits written directly), kLv8None unreached.  A quarter of the bytes of
// the uint32 form, written and then gathered.
constexpr uint32_t kLv8None = 0xFFu, kLv8Keep = 0xFEu;
// Each lane turns its own word's slices into 32 bytes (two 16-byte stores),
// no shuffles: 469 -> 286 us at s29 (ncu), DO +2.5%, against the layout that
// shuffled each word's slices to 8 lanes for 128-byte contiguous warp stores
// (the kernel was issue-bound on the shuffles at 39% occupancy).
__device__ __forceinline__ void store_word_levels8(const LevelSlices& L, int64_t wk, int64_t nwords,
                                                   uint8_t* __restrict__ lv8, int64_t n) {
  if (wk >= nwords) return;
  const int64_t u0 = wk << 5;
  uint32_t out[8];
  // 8x8 bit transposes (rows = level bit-planes 0..4, "in no bitmap",
  // "kept"; one 8x8 block per byte): row r byte c then holds vertex 8c + r.
  // 3 delta-swap stages + 3 byte permutes per output word: 261 -> 217 us at
  // s29 against spreading each nibble of each plane with a multiply.
  uint32_t r[8] = {L.s[0], L.s[1], L.s[2], L.s[3], L.s[4], ~L.any, L.vis & ~L.any, 0u};
#pragma unroll
  for (int d = 4, st = 0; st < 3; d >>= 1, ++st) {
    const uint32_t m = d == 4 ? 0x0F0F0F0Fu : (d == 2 ? 0x33333333u : 0x55555555u);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i & d) continue;
      const uint32_t t = ((r[i] >> d) ^ r[i + d]) & m;
      r[i + d] ^= t;
      r[i] ^= t << d;
    }
  }
  // bit 5 (in no bitmap) -> 0xFF, or 0xFE with bit 6 (kept)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t m5 = ((r[i] >> 5) & 0x01010101u) * 0xFFu;
    const uint32_t m6 = (r[i] >> 6) & 0x01010101u;
    r[i] = (r[i] & ~m5) | (m5 ^ m6);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = q >> 1, r0 = (q & 1) * 4;
    const uint32_t sel = (uint32_t)c | ((uint32_t)(4 + c) << 4);
    const uint32_t lo = __byte_perm(r[r0], r[r0 + 1], sel);
    const uint32_t hi = __byte_perm(r[r0 + 2], r[r0 + 3], sel);
    out[q] = __byte_perm(lo, hi, 0x5410);
  }
  if (u0 + 32 <= n) {
    uint4* d = reinterpret_cast<uint4*>(lv8 + u0);
    d[0] = make_uint4(out[0], out[1], out[2], out[3]);
    d[1] = make_uint4(out[4], out[5], out[6], out[7]);
  } else {
    for (int t = 0; u0 + t < n; ++t) lv8[u0 + t] = (uint8_t)(out[t >> 2] >> (8 * (t & 3)));
  }
}

// Units are taken two at a time so each warp has both units' bitmap loads in
// flight before the stores (uint32 d_local; the byte form is k_levels8_from_bits).
#ifdef BFB_LEVELS_MINB
#define BFB_LEVELS_LB __launch_bounds__(256, BFB_LEVELS_MINB)
#else
#define BFB_LEVELS_LB __launch_bounds__(256)
#endif
__global__ void BFB_LEVELS_LB k_levels_from_bits(const uint32_t* __restrict__ lvbits,
                                                          int64_t pad, int nl, uint32_t valid,
                                                          const uint32_t* __restrict__ visited,
                                                          uint32_t* __restrict__ level, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t nwords = (n + 31) / 32;
  const int64_t nunits = (nwords + 31) / 32;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t unit = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; unit < nunits;
       unit += 2 * nw) {
    const int64_t unit2 = unit + nw;
    LevelSlices A, B;
    load_level_slices(lvbits, pad, nl, valid, visited, unit * 32 + lane, unit * 32 + lane < nwords,
                      A);
    load_level_slices(lvbits, pad, nl, valid, visited, unit2 * 32 + lane,
                      unit2 < nunits && unit2 * 32 + lane < nwords, B);
    store_unit_levels(A, unit * 32, level, n);
    if (unit2 < nunits) store_unit_levels(B, unit2 * 32, level, n);
  }
}

// Byte form: one word per thread, 8 blocks per SM (32 registers): 284 ->
// 261 us at s29 against two units per warp at 40 registers.
__global__ void __launch_bounds__(256, 8) k_levels8_from_bits(const uint32_t* __restrict__ lvbits,
                                                            int64_t pad, int nl, uint32_t valid,
                                                            const uint32_t* __restrict__ visited,
                                                            uint8_t* __restrict__ lv8, int64_t n) {
  const int64_t nwords = (n + 31) / 32;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    LevelSlices A;
    load_level_slices(lvbits, pad, nl, valid, visited, w, true, A);
    store_word_levels8(A, w, nwords, lv8, n);
  }
}

// ------------------------------------------------------------ outputs ----
// Results in the caller's ids (relabelled engine graph): out[v] = engine
// result at perm[v], from the byte form of d_local (lv8; kLv8Keep -> the
// uint32 d_local).  The relabel keeps each degree class in the caller's
// order, so the lanes of a warp (consecutive v) gather from one ascending
// stream most of the time (isolated vertices: one stream of UNREACHED).
// Parents are stored in the caller's ids already; an unreached vertex gets
// none (this also masks a single node's stale entries).  out_level ==
// nullptr: parents only.
// Each block takes 1024 vertices per step (4 per thread, lane-consecutive);
// the next step's perm entries are copied into shared memory by one TMA bulk
// copy while this step gathers, so perm is off the per-vertex dependence
// chain (perm -> byte level -> parent -> store).  s29, ncu: 1.80 -> 1.55 ms,
// DO 1180 -> 1226 GTEP/s (per-thread 16-byte cp.async copies measured the
// same as the bulk copy), against the register-only kernel whose best setting
// was 4 vertices per thread at 8 blocks/SM (prefetching perm in registers
// spilled at 32 registers; 4 consecutive vertices per thread with 16-byte
// stores: 1.66 ms, the warp's gathers spread over 4x the lines).
constexpr int kOutChunk = 1024;  // vertices per block per step (256 threads x 4)
__global__ void __launch_bounds__(256, 8) k_output(const uint32_t* __restrict__ perm,
                                                   const uint8_t* __restrict__ lv8,
                                                   const uint32_t* __restrict__ level,
                                                   const uint32_t* __restrict__ parent,
                                                   uint32_t* __restrict__ out_level,
                                                   uint32_t* __restrict__ out_parent, int64_t n) {
  __shared__ __align__(128) uint32_t sp[2][kOutChunk];
  const int64_t nfull = n / kOutChunk;  // whole chunks; the remainder below
  int64_t c = blockIdx.x;  // uniform per block: the barriers below are safe
  // one bulk copy (TMA engine) of 4 KB per step, issued by thread 0, landing
  // on an mbarrier per buffer (phase parity flips with each use)
  __shared__ __align__(8) unsigned long long bar[2];
  const unsigned bar0 = (unsigned)__cvta_generic_to_shared(&bar[0]);
  auto bulk = [&](int buf, int64_t chunk) {
    const unsigned dst = (unsigned)__cvta_generic_to_shared(&sp[buf][0]);
    const unsigned mb = bar0 + 8u * (unsigned)buf;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                 "r"(kOutChunk * 4) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
        "l"(perm + chunk * kOutChunk), "r"(kOutChunk * 4), "r"(mb) : "memory");
  };
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0 + 8u));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && c < nfull) bulk(0, c);
  for (int b = 0, use = 0; c < nfull; c += gridDim.x, b ^= 1, ++use) {
    const int64_t cn = c + gridDim.x;
    if (threadIdx.x == 0 && cn < nfull) bulk(b ^ 1, cn);
    const unsigned parity = (unsigned)(use >> 1) & 1u;
    asm volatile(
        "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT%=;\n}\n" ::"r"(bar0 + 8u * (unsigned)b),
        "r"(parity) : "memory");
    uint32_t p[4], l[4], q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = sp[b][k * 256 + threadIdx.x];
#pragma unroll
    for (int k = 0; k < 4; ++k) l[k] = __ldg(lv8 + p[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      l[k] = l[k] == kLv8None ? kNone : (l[k] == kLv8Keep ? __ldg(level + p[k]) : l[k]);
    const int64_t v = c * kOutChunk + threadIdx.x;
    if (out_parent) {
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] = l[k] != kNone ? __ldg(parent + p[k]) : kNone;
#pragma unroll
      for (int k = 0; k < 4; ++k) out_parent[v + k * 256] = q[k];
    }
    if (out_level) {
#pragma unroll
      for (int k = 0; k < 4; ++k) out_level[v + k * 256] = l[k];
    }
    __syncthreads();  // buffer b is refilled by the next step's copies
  }
  // remainder (< kOutChunk vertices): block 0, one vertex per thread
  if (blockIdx.x == 0) {
    for (int64_t v = nfull * kOutChunk + threadIdx.x; v < n; v += blockDim.x) {
      const uint32_t pp = perm[v];
      uint32_t lv = lv8[pp];
      lv = lv == kLv8None ? kNone : (lv == kLv8Keep ? level[pp] : lv);
      if (out_level) out_level[v] = lv;
      if (out_parent) out_parent[v] = lv != kNone ? parent[pp] : kNone;
    }
  }
}

__global__ void k_parents_min(uint32_t* const* parents, int num_nodes, int64_t n, uint32_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t best = kNone;
    for (int g = 0; g < num_nodes; ++g) best = min(best, parents[g][i]);
    out[i] = best;
  }
}

// Bitmap of vertices with degree > 0 (lane = vertex, ballot per word).
// Per-vertex tables built once per engine setup (lane = vertex): the bitmap
// of degree > 0 and min(degree, 65535) as 16 bits.
__global__ void k_vertex_tables(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                int64_t n, int64_t row_lo, int64_t row_hi, uint32_t* nonisol,
                                uint16_t* deg16, uint32_t* nbr0, uint32_t* nbr1,
                                uint32_t* nbr0c, const uint32_t* __restrict__ inv,
                                int64_t nwords_pad) {
  const int lane = threadIdx.x & 31;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwords_pad;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t u = (w << 5) + lane;
    const int64_t o = u < n ? __ldg(off + u) : 0;
    const int64_t d = u < n ? __ldg(off + u + 1) - o : 0;
    const unsigned b = __ballot_sync(0xffffffffu, d > 0);
    if (lane == 0) nonisol[w] = b;
    deg16[u] = (uint16_t)min(d, (int64_t)0xFFFF);
    // (a rank's partitioned graph holds only its own rows' adjacency; the
    // tables of the other rows are never read)
    const bool mine = u >= row_lo && u < row_hi;
    const uint32_t f0 = mine && d > 0 ? __ldg(adj + o) : kNone;
    nbr0[u] = f0;
    nbr1[u] = mine && d > 1 ? __ldg(adj + o + 1) : kNone;
    nbr0c[u] = f0 != kNone && inv ? __ldg(inv + f0) : f0;
  }
}


// Single-node runs skip the 2 GB parent reset: every reached vertex but the
// root gets its parent from its own claim, so only unreached vertices hold
// stale values -- cleared here, from d_local, when parents are read out.
__global__ void k_mask_parents(const uint32_t* __restrict__ level, uint32_t* __restrict__ parent,
                               int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (level[i] == kNone) parent[i] = kNone;
}

// Certificate + parent validity, warp per vertex.
__global__ void k_validate(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                           int64_t n, const uint32_t* __restrict__ level,
                           const uint32_t* __restrict__ parent, int64_t root, unsigned* err) {
  const int lane = threadIdx.x & 31;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint32_t lu = level[u];
    unsigned e = 0;
    bool pred = false;
    for (int64_t j = off[u] + lane; j < off[u + 1]; j += 32) {
      const uint32_t lv = level[adj[j]];
      if ((lu == kNone) != (lv == kNone)) e |= 2u;
      else if (lu != kNone) {
        const int64_t dl = (int64_t)lu - (int64_t)lv;
        if (dl > 1 || dl < -1) e |= 4u;
        if (lv + 1 == lu) pred = true;
      }
    }
    e |= __reduce_or_sync(0xffffffffu, e);
    pred = __any_sync(0xffffffffu, pred);
    if (lane == 0) {
      if (u == root) {
        if (lu != 0) e |= 1u;
        if (parent && parent[u] != (uint32_t)root) e |= 16u;
      } else if (lu != kNone) {
        if (!pred) e |= 8u;
        if (parent) {
          const uint32_t p = parent[u];
          if (p == kNone || (int64_t)p >= n || level[p] + 1 != lu) {
            e |= 16u;
          } else {
            int64_t lo = off[p], hi = off[p + 1];
            while (lo < hi) {
              int64_t mid = (lo + hi) >> 1;
              if (adj[mid] < (uint32_t)u) lo = mid + 1; else hi = mid;
            }
            if (lo >= off[p + 1] || adj[lo] != (uint32_t)u) e |= 16u;
          }
        }
      } else if (parent && parent[u] != kNone) {
        e |= 16u;
      }
      if (e) atomicOr(err, e);
    }
  }
}

// Grid of a grid-stride kernel: one full wave of resident CTAs (148 SMs x the
// kernel's occupancy), fewer if the work is smaller.  Occupancy is queried
// once per kernel.
template <class K>
unsigned resident_grid(K kernel, int64_t work, int block, int num_sms, size_t smem = 0) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> occ_of;
  int occ = 1;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = occ_of.find((const void*)kernel);
    if (it == occ_of.end()) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, smem) != cudaSuccess)
        occ = 4;
      occ = std::max(1, occ);
      occ_of[(const void*)kernel] = occ;
    } else {
      occ = it->second;
    }
  }
  int64_t g = (work + block - 1) / block;
  g = std::min<int64_t>(g, (int64_t)num_sms * occ);
  return (unsigned)std::max<int64_t>(1, g);
}

unsigned grid_cap(int64_t work, int block, int num_sms, int per_sm = 8) {
  int64_t g = (work + block - 1) / block;
  int64_t cap = (int64_t)num_sms * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}


// d_local from the level bitmaps at termination (last_level = the deepest
// level committed); returns kernels launched.
int launch_materialise_levels(bfb_ctx* ctx, Part& p, int64_t last_level, cudaStream_t s,
                              uint8_t* lv8 = nullptr) {
  const int64_t pad = (int64_t)(p.lvbits.n / kLevelBits);
  const int nl = (int)std::min<int64_t>(last_level, kLevelBits - 1);
  if (lv8) {
    k_levels8_from_bits<<<resident_grid(k_levels8_from_bits, (ctx->g.n + 31) / 32, 256,
                                        ctx->num_sms),
                          256, 0, s>>>(p.lvbits.p, pad, nl, ctx->lvbits_valid, p.visited.p, lv8,
                                       ctx->g.n);
    return 1;
  }
  k_levels_from_bits<<<resident_grid(k_levels_from_bits, (ctx->g.n + 31) / 32, 256,
                                     ctx->num_sms),
                       256, 0, s>>>(p.lvbits.p, pad, nl, ctx->lvbits_valid, p.visited.p, p.level.p,
                                    ctx->g.n);
  return 1;
}

// Node 0's results in the caller's ids (relabelled engine graph).
int launch_output(bfb_ctx* ctx, Part& p, int64_t last_level, const uint32_t* parent, bool levels,
                  cudaStream_t s) {
  int k = 0;
  // (the byte form of d_local: levels=false reuses the run's, for the mask)
  if (levels) k += launch_materialise_levels(ctx, p, last_level, s, ctx->lv8.p);
  const int64_t n = ctx->g.n;
  k_output<<<grid_cap((n + kOutChunk - 1) / kOutChunk * 256, 256, ctx->num_sms, 8), 256, 0, s>>>(
      ctx->perm.p, ctx->lv8.p, p.level.p, parent, levels ? ctx->out_level.p : nullptr,
      parent ? ctx->out_parent.p : nullptr, n);
  return k + 1;
}

// Multi-process merge: OR the round's source snapshots (peer memory mapped
// over NVLink by CUDA IPC, or local) into this node's visited bitmap.  This
// node is the only writer of its bitmap during the merge, so no atomics.
constexpr int kMaxSrc = 64;
struct SrcList {
  const uint32_t* p[kMaxSrc];
  int n;
};

__global__ void k_merge_peers(SrcList L, uint32_t* __restrict__ vis, int64_t nwords) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t acc = 0;
    for (int i = 0; i < L.n; ++i) acc |= L.p[i][w];
    if (acc) {
      const uint32_t cur = vis[w];
      if (acc & ~cur) vis[w] = cur | acc;
    }
  }
}

// Owned-words commit (count -> pair scan -> write); returns kernels launched.
// First half of the owned-words commit: per-unit counts and degree sums and
// the tile scan (totals -> ctr->q_count / q_edges, RunStats traversed_edges).
int launch_commit_count(const PartView& v, const int64_t* off, RunCounters* run, int sms,
                        cudaStream_t s, bool parent_pass = false) {
  const int64_t ntiles = std::max<int64_t>(1, (v.nunits + kScanTile - 1) / kScanTile);
  if (parent_pass)
    k_commit_count<true><<<resident_grid(k_commit_count<true>, v.nunits * 32, 256, sms), 256, 0,
                           s>>>(v, off);
  else
    k_commit_count<false><<<resident_grid(k_commit_count<false>, v.nunits * 32, 256, sms), 256, 0,
                            s>>>(v, off);
  k_unit_scan_reduce<<<(unsigned)ntiles, 256, 0, s>>>(v);
  k_unit_scan_tiles<<<1, 1024, 0, s>>>(v, ntiles, run);
  return 3;
}

// Second half: with_queue builds the next q_local (unit prefixes + write);
// without it (next phase 1 runs bottom-up, which reads only bitmaps) only
// levels, the start snapshot and the frontier bitmap are written.
int launch_commit_write(const PartView& v, const int64_t* off, uint32_t next_level, bool with_queue,
                        int sms, cudaStream_t s) {
  const int64_t ntiles = std::max<int64_t>(1, (v.nunits + kScanTile - 1) / kScanTile);
  const int64_t work = v.nunits * 32;
  if (!with_queue) {
    k_commit_light<<<resident_grid(k_commit_light, work, 256, sms), 256, 0, s>>>(v, next_level);
    return 1;
  }
  k_unit_scan_apply<<<(unsigned)ntiles, 256, 0, s>>>(v);
  const int64_t pf_min = v.nunits * 16;  // 1/64 of the part's vertices
  if (v.wide) {
    k_commit_write<true, false><<<resident_grid(k_commit_write<true, false>, work, 256, sms), 256,
                                   0, s>>>(v, off, next_level, pf_min);
    k_commit_write<true, true><<<resident_grid(k_commit_write<true, true>, work, 256, sms), 256,
                                  0, s>>>(v, off, next_level, pf_min);
  } else {
    k_commit_write<false, false><<<resident_grid(k_commit_write<false, false>, work, 256, sms),
                                   256, 0, s>>>(v, off, next_level, pf_min);
    k_commit_write<false, true><<<resident_grid(k_commit_write<false, true>, work, 256, sms), 256,
                                  0, s>>>(v, off, next_level, pf_min);
  }
  return 3;
}

// Bottom-up level commit (one pass); rebuild: the queue for a following
// top-down level, from the frontier bitmap, by count -> scan -> write.
int launch_commit_light_count(const PartView& v, const int64_t* off, uint32_t next_level,
                              RunCounters* run, int sms, cudaStream_t s) {
  k_commit_light_count<<<resident_grid(k_commit_light_count, v.nunits * 32, 256, sms), 256, 0, s>>>(
      v, off, next_level, run);
  return 1;
}

int launch_commit_rebuild(PartView v, const int64_t* off, uint32_t next_level, RunCounters* run,
                          int sms, cudaStream_t s) {
  v.rebuild = true;
  return launch_commit_count(v, off, run, sms, s) +
         launch_commit_write(v, off, next_level, true, sms, s);
}

int launch_commit(const PartView& v, const int64_t* off, uint32_t next_level, RunCounters* run,
                  int sms, cudaStream_t s) {
  return launch_commit_count(v, off, run, sms, s) +
         launch_commit_write(v, off, next_level, true, sms, s);
}

}  // namespace

// Device-side tables built at setup (pointer arrays indexed by node, the
// butterfly rounds as (dst, src) pair lists) and the timing events.
struct EngineTables {
  DevBuf<uint32_t*> pubs, visiteds, parents, sqs;  // sqs: every node's claim queue (sparse levels)
  DevBuf<PartCounters*> ctrs;
  std::vector<DevBuf<int32_t>> round_tables;
  std::vector<RoundDesc> rounds;
  DevBuf<uint32_t> parents_final;  // assembled output parents when num_parts > 1
  DevBuf<int64_t> tail_sizes;      // k_tail: frontier sizes of the levels it committed
  DevBuf<TailOut> tail_out;
  std::vector<int64_t> tail_host;  // their host copy (sized at setup)
  cudaEvent_t ev[6] = {};
  std::vector<cudaEvent_t> part_ev;  // timing mode, CN > 1: per-node phase-1 bounds
  // multi-process mode (rank >= 0): this context holds node `rank` only
  int rank = -1;
  std::vector<const uint32_t*> peer_pub[2];  // per node, by round parity
  std::vector<void*> opened;                 // IPC mappings to close
  // device-synchronised rank mode (rank_bfs): this node's mailbox (one
  // {seq, count} slot per writer, written by peers over NVLink), the peers'
  // mailboxes (IPC-mapped), a barrier-timeout flag, and the round counter
  DevBuf<int64_t> mail;
  DevBuf<int64_t*> peer_mail_dev;
  DevBuf<int32_t> err;
  std::vector<int64_t*> peer_mail;
  std::vector<uint32_t*> peer_parent;  // every node's phase-1 parents (IPC-mapped)
  std::vector<const uint32_t*> peer_q; // every node's queue-form snapshots (IPC-mapped)
  int64_t seq = 0;
  int64_t level = 0, reached = 0, launches = 0, levels = 0;
  int64_t remote_messages = 0, remote_vertices = 0, high_water = 0, exchange_bytes = 0;
  ~EngineTables() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : part_ev) cudaEventDestroy(e);
  }
};

bool rank_mode(const bfb_ctx* ctx) { return ctx->tables && ctx->tables->rank >= 0; }

// d_local of node 0 in the caller's ids
static const uint32_t* out_levels(bfb_ctx* ctx) {
  return ctx->relabeled ? ctx->out_level.p : ctx->parts[0].level.p;
}

void engine_release(bfb_ctx* ctx) {
  small_release(ctx);
  ctx->parts.clear();
  ctx->run.release();
  ctx->high_water.release();
  ctx->engine_ready = false;
  ctx->have_run = false;
  if (ctx->pinned) {
    cudaFreeHost(ctx->pinned);
    ctx->pinned = nullptr;
  }
  delete ctx->tables;
  ctx->tables = nullptr;
}

// Several parts over the relabelled graph: each part's hubs are its first
// ids, so the hot probes are those of the first kHotLimit / P ids of every
// part, marked per 2^16-id block (the probe reads one L1-resident word).
// One part (or no relabel): no mask, the single hot range [0, hot_limit).
#ifndef BFB_HOT_MASK
#define BFB_HOT_MASK 1
#endif
static int build_hot_mask(bfb_ctx* ctx, const std::vector<int64_t>& b) {
  ctx->hot_mask.release();
  const int P = (int)b.size() - 1;
  if (!BFB_HOT_MASK || !ctx->relabeled || P <= 1) return BFB_OK;
  const int64_t n = ctx->g.n, nblk = (n + 65535) >> 16;
  std::vector<uint32_t> m((nblk + 31) / 32 + 1, 0u);
  for (int g = 0; g < P; ++g) {
    const int64_t h = std::min<int64_t>(b[g + 1] - b[g], (int64_t)kHotLimit / P);
    if (h <= 0) continue;
    for (int64_t k = b[g] >> 16; k <= (b[g] + h - 1) >> 16; ++k) m[k >> 5] |= 1u << (k & 31);
  }
  BFB_TRY(ctx->hot_mask.alloc(m.size()));
  BFB_CUDA(cudaMemcpy(ctx->hot_mask.p, m.data(), m.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  return BFB_OK;
}

// rb: the partition the engine graph is relabelled within (the engine's own
// partition, or the global one for a rank's single-node engine)
static int engine_setup_rb(bfb_ctx* ctx, int parts, const int64_t* bounds, int fanout,
                           int strategy, int want_parents, const std::vector<int64_t>& rb);

int engine_setup(bfb_ctx* ctx, int parts, const int64_t* bounds, int fanout, int strategy,
                 int want_parents) {
  if (parts < 1) return fail(BFB_ERR_PARTITION, "num_parts must be >= 1");
  if (ctx->g.valid && !ctx->g.full())
    return fail(BFB_ERR_STATE, "this context holds one rank's rows only (use bfb_rank_setup)");
  BFB_TRY(engine_setup_rb(ctx, parts, bounds, fanout, strategy, want_parents,
                          std::vector<int64_t>(bounds, bounds + parts + 1)));
  return small_setup(ctx);  // small graphs: the single-CTA engine's tables too
}

static int engine_setup_rb(bfb_ctx* ctx, int parts, const int64_t* bounds, int fanout,
                           int strategy, int want_parents, const std::vector<int64_t>& rb) {
  if (!ctx->g.valid) return fail(BFB_ERR_STATE, "no graph loaded");

  const int64_t n = ctx->g.n;
  if (parts < 1) return fail(BFB_ERR_PARTITION, "num_parts must be >= 1");
  if (bounds[0] != 0 || bounds[parts] != n)
    return fail(BFB_ERR_PARTITION, "partition does not match graph");
  for (int g = 0; g < parts; ++g)
    if (bounds[g + 1] < bounds[g]) return fail(BFB_ERR_PARTITION, "partition does not match graph");
  if (strategy != BFB_STRATEGY_BUTTERFLY && strategy != BFB_STRATEGY_ALL2ALL)
    return fail(BFB_ERR_INVALID, "unknown strategy");
  if (fanout < 1) return fail(BFB_ERR_FANOUT, "fanout must be >= 1");
  if (fanout > parts) return fail(BFB_ERR_FANOUT, "fanout exceeds num_nodes");
  engine_release(ctx);
  BFB_TRY(make_schedule(parts, fanout, strategy, ctx->schedule));
  ctx->num_parts = parts;
  ctx->fanout = fanout;
  ctx->strategy = strategy;
  ctx->want_parents = want_parents ? 1 : 0;
  ctx->bounds.assign(bounds, bounds + parts + 1);
  ctx->tables = new EngineTables();
  EngineTables* D = ctx->tables;
  const int64_t nwords = (n + 31) / 32;
  const int64_t nwords_pad = (nwords + kWordPad - 1) / kWordPad * kWordPad + kWordPad;
  std::vector<int64_t> off_h(parts + 1);
  {
    // owned edge counts: offsets at the boundaries
    for (int g = 0; g <= parts; ++g)
      BFB_CUDA(cudaMemcpy(&off_h[g], ctx->g.offsets.p + bounds[g], sizeof(int64_t),
                          cudaMemcpyDeviceToHost));
  }
  // the engine's graph: degree-ordered within the parts of rb (relabel.cu)
  if (relabel_wanted(ctx)) {
    BFB_TRY(relabel_build(ctx, rb));
  } else {
    relabel_release(ctx);
  }
  DevGraph& G = EG(ctx);
  BFB_TRY(G.nonisol.alloc(nwords_pad));
  BFB_TRY(G.deg16.alloc((size_t)nwords_pad * 32));
  BFB_TRY(G.first_nbr.alloc((size_t)nwords_pad * 96));  // nbr0 | nbr1 | nbr0 in caller ids
  k_vertex_tables<<<grid_cap(nwords_pad * 32, 256, ctx->num_sms, 8), 256, 0, ctx->stream>>>(
      G.offsets.p, G.adj_index(), n, G.row_lo, G.row_hi, G.nonisol.p, G.deg16.p, G.first_nbr.p,
      G.first_nbr.p + (size_t)nwords_pad * 32, G.first_nbr.p + (size_t)nwords_pad * 64,
      ctx->relabeled ? ctx->inv.p : nullptr,
      nwords_pad);
  if (ctx->relabeled) {
    BFB_TRY(ctx->out_level.alloc(n + 1));
    BFB_TRY(ctx->lv8.alloc(n + 16));
    if (want_parents) BFB_TRY(ctx->out_parent.alloc(n + 1));
  }
  BFB_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->parts.resize(parts);
  std::vector<uint32_t*> pubs(parts), viss(parts), pars(parts);
  std::vector<PartCounters*> ctrs(parts);
  for (int g = 0; g < parts; ++g) {
    Part& p = ctx->parts[g];
    p.lo = bounds[g];
    p.hi = bounds[g + 1];
    p.wlo = p.lo >> 5;
    p.whi = (p.hi + 31) >> 5;
    if (p.hi == p.lo) p.whi = p.wlo;  // empty part owns no words
    p.owned_edges = off_h[g + 1] - off_h[g];
    p.tile_cap = (p.owned_edges + kTile - 1) / kTile + 2;
    const int64_t owned = p.hi - p.lo;
    BFB_TRY(p.visited.alloc(nwords_pad));
    BFB_TRY(p.start.alloc(nwords_pad));
    BFB_TRY(p.level.alloc(n + 1));
    if (want_parents) BFB_TRY(p.parent.alloc(n + 1));
    if (parts > 1) BFB_TRY(p.pub.alloc(nwords_pad));
    {
      // sparse levels' claim queue: frontiers of at most this many edges
      const int64_t cap = std::min<int64_t>(
          std::min<int64_t>(std::max<int64_t>(n >> BFB_SPARSE_SHIFT, 65536), BFB_SPARSE_CAP), n);
      BFB_TRY(p.sparse_q.alloc(cap));
    }
    BFB_TRY(p.q_v.alloc(owned + 1));
    BFB_TRY(p.q_pre.alloc(owned + 1));
    BFB_TRY(p.q_base.alloc(owned + 1));
    BFB_TRY(p.tile_vstart.alloc(p.tile_cap));
    BFB_TRY(p.front.alloc(nwords_pad));
    BFB_TRY(p.lvbits.alloc((size_t)kLevelBits * nwords_pad));
    {
      const int64_t nunits = (p.whi - (p.wlo & ~(int64_t)31) + 31) / 32 + 1;
      const int64_t ntiles = (nunits + kScanTile - 1) / kScanTile + 1;
      BFB_TRY(p.unit_u32.alloc(nunits));
      BFB_TRY(p.unit_i64.alloc(3 * nunits + 2 * ntiles));
    }
    BFB_TRY(p.ctr.alloc(1));
    BFB_CUDA(cudaMemset(p.visited.p, 0, nwords_pad * sizeof(uint32_t)));
    BFB_CUDA(cudaMemset(p.start.p, 0, nwords_pad * sizeof(uint32_t)));
    if (parts > 1) BFB_CUDA(cudaMemset(p.pub.p, 0, nwords_pad * sizeof(uint32_t)));
    BFB_CUDA(cudaMemset(p.ctr.p, 0, sizeof(PartCounters)));
    pubs[g] = p.pub.p;
    viss[g] = p.visited.p;
    pars[g] = p.parent.p;
    ctrs[g] = p.ctr.p;
  }
  BFB_TRY(D->pubs.alloc(parts));
  BFB_TRY(D->sqs.alloc(parts));
  BFB_TRY(D->visiteds.alloc(parts));
  BFB_TRY(D->parents.alloc(parts));
  BFB_TRY(D->ctrs.alloc(parts));
  BFB_CUDA(cudaMemcpy(D->pubs.p, pubs.data(), parts * sizeof(void*), cudaMemcpyHostToDevice));
  {
    std::vector<uint32_t*> sqs(parts);
    for (int g = 0; g < parts; ++g) sqs[g] = ctx->parts[g].sparse_q.p;
    BFB_CUDA(cudaMemcpy(D->sqs.p, sqs.data(), parts * sizeof(void*), cudaMemcpyHostToDevice));
  }
  BFB_CUDA(cudaMemcpy(D->visiteds.p, viss.data(), parts * sizeof(void*), cudaMemcpyHostToDevice));
  BFB_CUDA(cudaMemcpy(D->parents.p, pars.data(), parts * sizeof(void*), cudaMemcpyHostToDevice));
  BFB_CUDA(cudaMemcpy(D->ctrs.p, ctrs.data(), parts * sizeof(void*), cudaMemcpyHostToDevice));
  // round tables
  for (auto& rnd : ctx->schedule) {
    std::vector<int32_t> dst, src, first(parts + 1, 0);
    for (int g = 0; g < parts; ++g) {
      first[g] = (int32_t)dst.size();
      for (int s : rnd[g]) {
        dst.push_back(g);
        src.push_back(s);
      }
    }
    first[parts] = (int32_t)dst.size();
    DevBuf<int32_t> tab;
    const int np = (int)dst.size();
    BFB_TRY(tab.alloc(2 * (size_t)np + parts + 1));
    if (np) {
      BFB_CUDA(cudaMemcpy(tab.p, dst.data(), np * sizeof(int32_t), cudaMemcpyHostToDevice));
      BFB_CUDA(cudaMemcpy(tab.p + np, src.data(), np * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    BFB_CUDA(cudaMemcpy(tab.p + 2 * np, first.data(), (parts + 1) * sizeof(int32_t),
                        cudaMemcpyHostToDevice));
    RoundDesc rd;
    rd.pair_dst = tab.p;
    rd.pair_src = tab.p + np;
    rd.node_first = tab.p + 2 * np;
    rd.npairs = np;
    rd.num_nodes = parts;
    D->rounds.push_back(rd);
    D->round_tables.push_back(std::move(tab));
  }
  if (want_parents && parts > 1) BFB_TRY(D->parents_final.alloc(n + 1));
  if (parts == 1) {  // thin levels run in k_tail
    BFB_TRY(D->tail_sizes.alloc(kTailMax));
    BFB_TRY(D->tail_out.alloc(1));
    D->tail_host.assign(kTailMax + 1, 0);
  }
  BFB_TRY(ctx->run.alloc(1));
  BFB_TRY(ctx->high_water.alloc(parts));
  BFB_CUDA(cudaMallocHost(&ctx->pinned, sizeof(int64_t) * (8 + 8 * (size_t)parts)));
  int occ = 0;
  if (want_parents)
    BFB_TRY(expand_occupancy<true>(&occ));
  else
    BFB_TRY(expand_occupancy<false>(&occ));
  ctx->expand_grid = std::max(1, occ) * ctx->num_sms;
  BFB_TRY(readout_setup(ctx, n));  // read-out buffers: bfb_bfs allocates nothing
  for (auto& ev : D->ev) BFB_CUDA(cudaEventCreate(&ev));
  if (parts > 1) {
    D->part_ev.resize(parts + 1);
    for (auto& ev : D->part_ev) BFB_CUDA(cudaEventCreate(&ev));
  }
  // one node over the relabelled graph: its hubs are the lowest ids (probe_vertex)
  ctx->hot_limit = ctx->relabeled && parts == 1 ? kHotLimit : kNone;
  BFB_TRY(build_hot_mask(ctx, rb));
  ctx->engine_ready = true;
  return BFB_OK;
}

// Small graphs (small_bfs.cu): the whole top-down run in one single-CTA
// launch; results land in the same device buffers as engine_bfs's, so the
// read-out, the parents view and validation are shared.
static int small_run(bfb_ctx* ctx, int64_t root, uint32_t* levels_out, int64_t* parents_out,
                     int64_t* sizes_out, int64_t max_levels, int64_t* hw_out, bfb_run_stats* st) {
  EngineTables* D = ctx->tables;
  cudaStream_t s = ctx->stream;
  const int P = ctx->num_parts;
  const int64_t n = ctx->g.n;
  uint32_t* lv = const_cast<uint32_t*>(out_levels(ctx));
  uint32_t* par = nullptr;
  if (ctx->want_parents)
    par = ctx->relabeled ? ctx->out_parent.p : (P > 1 ? D->parents_final.p : ctx->parts[0].parent.p);
  SmallResult r;
  BFB_TRY(small_bfs(ctx, root, lv, par, ctx->high_water.p, ctx->checks & 1, D->ev[0], D->ev[1], &r));
  const int64_t nsizes = (int64_t)r.sizes.size();
  if (sizes_out)
    for (int64_t i = 0; i < std::min(nsizes, max_levels); ++i) sizes_out[i] = r.sizes[i];
  ctx->last_sizes = r.sizes;
  std::vector<int64_t> hw(P);
  BFB_CUDA(cudaMemcpyAsync(hw.data(), ctx->high_water.p, P * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, s));
  if (levels_out) BFB_TRY(read_levels(ctx, lv, n, nsizes, levels_out, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  float elapsed = 0;
  BFB_CUDA(cudaEventElapsedTime(&elapsed, D->ev[0], D->ev[1]));
  if (parents_out) {
    if (!ctx->want_parents) return fail(BFB_ERR_STATE, "engine set up without parents");
    BFB_TRY(read_parents(ctx, par, n, parents_out, s));
    BFB_CUDA(cudaStreamSynchronize(s));
  }
  if (hw_out) std::memcpy(hw_out, hw.data(), P * sizeof(int64_t));
  ctx->have_run = true;
  ctx->last_root = root;
  ctx->last_levels = nsizes;
  int64_t mx = 0;
  for (auto x : hw) mx = std::max(mx, x);
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->levels = nsizes;
    st->rounds_executed = nsizes * (int64_t)ctx->schedule.size();
    st->remote_messages = r.remote_messages;
    st->remote_vertices = r.remote_vertices;
    st->traversed_edges = r.traversed_edges;
    st->reached = r.reached;
    st->buffer_high_water_max = mx;
    st->exchange_bytes = r.exchange_bytes;
    st->elapsed_ms = elapsed;
    st->kernel_launches = 1;
    st->expand_launches = 1;
  }
  if (r.disagree)
    return fail(BFB_ERR_CAPACITY, "frontier disagreement after phase 2 (" +
                                      std::to_string(r.disagree) + " vertices differ)");
  if (mx > (int64_t)ctx->fanout * n && ctx->strategy == BFB_STRATEGY_BUTTERFLY)
    return fail(BFB_ERR_CAPACITY, "buffer bound violated");
  return BFB_OK;
}

int engine_bfs(bfb_ctx* ctx, int64_t root, uint32_t* levels_out, int64_t* parents_out,
               int64_t* sizes_out, int64_t max_levels, int64_t* hw_out, bfb_run_stats* st) {
  if (!ctx->engine_ready) return fail(BFB_ERR_STATE, "engine not set up");
  const int64_t n = ctx->g.n;
  if (root < 0 || root >= n)
    return fail(BFB_ERR_ROOT, "root " + std::to_string(root) + " out of range [0, " +
                                  std::to_string(n) + ")");
  if (ctx->small && ctx->small_mode && ctx->direction == 0)
    return small_run(ctx, root, levels_out, parents_out, sizes_out, max_levels, hw_out, st);
  EngineTables* D = ctx->tables;
  cudaStream_t s = ctx->stream;
  const int P = ctx->num_parts;
  const int sms = ctx->num_sms;
  const int64_t nwords = (n + 31) / 32;
  const int64_t* off = EG(ctx).offsets.p;
  int64_t launches = 0;
  double t_expand = 0, t_exchange = 0, t_commit = 0, t_expand_max = 0;
  int64_t expand_launches = 0;

  BFB_CUDA(cudaEventRecord(D->ev[0], s));
  // init: every node d_local = UNREACHED, d_local[root] = 0
  BFB_CUDA(cudaMemsetAsync(ctx->run.p, 0, sizeof(RunCounters), s));
  BFB_CUDA(cudaMemsetAsync(ctx->high_water.p, 0, P * sizeof(int64_t), s));
  int owner = 0;
  for (int g = 0; g < P; ++g)
    if (root >= ctx->bounds[g] && root < ctx->bounds[g + 1]) owner = g;
  for (int g = 0; g < P; ++g) {
    Part& p = ctx->parts[g];
    BFB_CUDA(cudaMemsetAsync(p.visited.p, 0, nwords * sizeof(uint32_t), s));
    BFB_CUDA(cudaMemsetAsync(p.start.p, 0, nwords * sizeof(uint32_t), s));
    // (d_local needs no reset: it is materialised at termination)
    // parents: a multi-node run takes the min over nodes, so non-claimed
    // entries must read kNone; a single node masks at read-out instead
    if (ctx->want_parents && P > 1)
      BFB_CUDA(cudaMemsetAsync(p.parent.p, 0xFF, n * sizeof(uint32_t), s));
    if (ctx->direction) BFB_CUDA(cudaMemsetAsync(p.front.p, 0, nwords * sizeof(uint32_t), s));
    k_seed<<<1, 256, 0, s>>>(view_of(ctx, p), off, root, perm_of(ctx), g == owner ? 1 : 0,
                             ctx->run.p);
    ++launches;
  }
  // Direction-optimizing state (Beamer's heuristic): switch to bottom-up when
  // the frontier's edges exceed the unexplored edges / alpha, back to
  // top-down when the frontier shrinks below |V| / beta.
  bool bottom_up = ctx->direction == 2;
  int64_t bu_levels = 0;
  int64_t prev_frontier = 1;
  const int64_t bytes_per_transfer = nwords * (int64_t)sizeof(uint32_t);
  int64_t level = 0;
  int64_t nsizes = 0;
  if (max_levels > 0 && sizes_out) sizes_out[0] = 1;
  nsizes = 1;
  ctx->last_sizes.assign(1, 1);
  int64_t reached = 1;
  int64_t switch_chk = 0;
  const unsigned small_grid = grid_cap(nwords, 256, sms, 4);
  // sparse levels (one node, top-down): the frontier's edge count bounds the
  // claims; below the threshold phase 1 queues its claims and the commit works
  // from the queue (k_sparse_commit) instead of sweeping the bitmaps
  const bool sparse_ok = ctx->sparse_mode && ctx->direction != 2 &&
                         ctx->parts[0].sparse_q.p != nullptr;
  const int64_t sparse_cap = (int64_t)ctx->parts[0].sparse_q.n;
  int64_t cur_edges = ctx->g.max_degree;  // the root's degree, bounded
  int64_t sparse_levels = 0;
  ctx->lvbits_valid = 0xFFFFFFFFu;
  const bool tail_ok = sparse_ok && P == 1 && ctx->direction == 0 && D->tail_sizes.p != nullptr;
  bool finished = false;
  while (true) {
    if (tail_ok && cur_edges <= kTailEdges) {
      // a run of thin levels in one single-CTA launch (k_tail)
      Part& tp = ctx->parts[0];
      PartView tv = view_of(ctx, tp);
      tv.sparse_q = tp.sparse_q.p;
      if (ctx->want_parents)
        k_tail<true><<<1, kTailThreads, 0, s>>>(tv, off, EG(ctx).adj_index(), (uint32_t)level,
                                                 ctx->run.p, D->tail_sizes.p, D->tail_out.p);
      else
        k_tail<false><<<1, kTailThreads, 0, s>>>(tv, off, EG(ctx).adj_index(), (uint32_t)level,
                                                  ctx->run.p, D->tail_sizes.p, D->tail_out.p);
      ++launches;
      ++expand_launches;
      BFB_CUDA(cudaMemcpyAsync(D->tail_host.data() + kTailMax, D->tail_out.p, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
      BFB_CUDA(cudaMemcpyAsync(D->tail_host.data(), D->tail_sizes.p, kTailMax * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
      BFB_CUDA(cudaMemcpyAsync(ctx->pinned + 5, tp.ctr.p, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost,
                               s));
      BFB_CUDA(cudaStreamSynchronize(s));
      BFB_CUDA(cudaGetLastError());
      const int64_t nl = D->tail_host[kTailMax];
      for (int64_t i = 0; i < nl; ++i) {
        const uint32_t committed = (uint32_t)(level + 1);
        if (committed < (uint32_t)kLevelBits) ctx->lvbits_valid &= ~(1u << committed);
        ++sparse_levels;
        const int64_t f = D->tail_host[i];
        if (f == 0) {
          finished = true;
          break;
        }
        prev_frontier = f;
        if (nsizes < max_levels && sizes_out) sizes_out[nsizes] = f;
        ctx->last_sizes.push_back(f);
        ++nsizes;
        reached += f;
        ++level;
      }
      if (finished) break;
      cur_edges = ctx->pinned[6];
      if (level > n) return fail(BFB_ERR_CAPACITY, "level count exceeded |V| (internal error)");
      if (cur_edges <= kTailEdges && ctx->pinned[5] > 0 && nl < kTailMax)
        return fail(BFB_ERR_CUDA, "thin-level kernel stopped early (internal error)");
      continue;
    }
    const bool sparse = sparse_ok && !bottom_up && cur_edges <= sparse_cap;
    if (ctx->timing) BFB_CUDA(cudaEventRecord(D->ev[2], s));
    // Parents of a top-down level with a large frontier come from the
    // commit's parent pass instead of phase-1 stores (k_commit_count): each
    // node's pass covers its owned new vertices, whoever found them, and the
    // output takes the min over nodes.  `start` (levels <= L, = `reached`)
    // must be large for the pass's lowest-neighbour probes to hit without
    // row scans.
    const bool parent_pass = ctx->want_parents && !bottom_up &&
                             prev_frontier >= std::max<int64_t>(1, n >> 12) &&
                             reached >= pass_min_reached(n);
    const bool expand_parents = ctx->want_parents && (!parent_pass || sparse);
    // Phase 1
    const bool part_timing = ctx->timing && P > 1;
    for (int g = 0; g < P; ++g) {
      if (part_timing) BFB_CUDA(cudaEventRecord(D->part_ev[g], s));
      PartView v = view_of(ctx, ctx->parts[g]);
      if (sparse) v.sparse_q = ctx->parts[g].sparse_q.p;
      if (bottom_up) {
        const unsigned bg = grid_cap(std::max<int64_t>(1, v.whi - v.wlo), 256, sms, 8);
        unsigned long long* ex = (unsigned long long*)&ctx->run.p->edges_examined;
        if (ctx->want_parents)
          k_bottom_up<true><<<bg, 256, 0, s>>>(v, EG(ctx).adj_index(), ex);
        else
          k_bottom_up<false><<<bg, 256, 0, s>>>(v, EG(ctx).adj_index(), ex);
      } else if (expand_parents) {
        launch_expand<true>(ctx->expand_grid, v, EG(ctx).adj_index(), s);
      } else {
        launch_expand<false>(ctx->expand_grid, v, EG(ctx).adj_index(), s);
      }
      ++launches;
      ++expand_launches;
    }
    if (bottom_up) ++bu_levels;
    if (part_timing) BFB_CUDA(cudaEventRecord(D->part_ev[P], s));
    if (ctx->timing) BFB_CUDA(cudaEventRecord(D->ev[3], s));
    // Phase 2
    if (!D->rounds.empty()) {
      k_zero_parity<<<1, 256, 0, s>>>(D->ctrs.p, P, 0);
      k_zero_parity<<<1, 256, 0, s>>>(D->ctrs.p, P, 1);
      launches += 2;
    }
    for (size_t r = 0; r < D->rounds.size(); ++r) {
      const int parity = (int)(r & 1);
      const RoundDesc& rd = D->rounds[r];
      if (sparse) {  // snapshot = each node's claim queue as it stands
        k_snap_sparse<<<1, 256, 0, s>>>(D->ctrs.p, P, parity);
        ++launches;
      }
      for (int g = 0; g < P && !sparse; ++g) {
        k_publish<<<small_grid, 256, 0, s>>>(view_of(ctx, ctx->parts[g]), parity);
        ++launches;
      }
      k_account<<<1, 256, 0, s>>>(rd, D->ctrs.p, ctx->run.p, ctx->high_water.p, parity,
                                  sparse ? -1 : bytes_per_transfer);
      k_zero_parity<<<1, 256, 0, s>>>(D->ctrs.p, P, parity ^ 1);
      launches += 2;
      if (rd.npairs && sparse) {
        dim3 grid(grid_cap(sparse_cap, 256, sms, 1), rd.npairs);
        k_merge_sparse<<<grid, 256, 0, s>>>(rd, D->sqs.p, D->visiteds.p, D->ctrs.p, parity);
        ++launches;
      } else if (rd.npairs) {
        dim3 grid(grid_cap(nwords, 256, sms, 2), rd.npairs);
        k_merge<<<grid, 256, 0, s>>>(rd, D->pubs.p, D->visiteds.p, D->ctrs.p, parity, nwords);
        ++launches;
      }
    }
    if (ctx->checks & 1 && P > 1) {
      k_agree<<<grid_cap(nwords, 256, sms, 2), 256, 0, s>>>(D->visiteds.p, P, nwords, ctx->run.p);
      ++launches;
    }
    if (ctx->timing) BFB_CUDA(cudaEventRecord(D->ev[4], s));
    // Commit: levels, start snapshot, next q_local, frontier count.
    k_commit_prep<<<1, 256, 0, s>>>(D->ctrs.p, P);
    ++launches;
    const uint32_t next_level = (uint32_t)(level + 1);
    if (ctx->direction)
      for (int g = 0; g < P; ++g)
        BFB_CUDA(cudaMemsetAsync(ctx->parts[g].front.p, 0, nwords * sizeof(uint32_t), s));
    // Top-down level: count, [decide,] write with or without the queue.
    // Bottom-up level: one queue-less pass; the queue is rebuilt from the
    // frontier bitmap only on the switch back to top-down.
    const bool light = ctx->direction != 0 && bottom_up;
    for (int g = 0; g < P && sparse; ++g) {
      Part& p = ctx->parts[g];
      PartView v = view_of(ctx, p);
      v.sparse_q = p.sparse_q.p;
      k_sparse_commit<<<grid_cap(sparse_cap, 256, sms, 8), 256, 0, s>>>(v, off, next_level);
      k_sparse_finalize<<<1, 1, 0, s>>>(p.ctr.p, ctx->run.p);
      launches += 2;
    }
    if (sparse) {
      if (next_level < (uint32_t)kLevelBits) ctx->lvbits_valid &= ~(1u << next_level);
      ++sparse_levels;
    }
    for (int g = 0; g < P && !sparse; ++g) {
      Part& p = ctx->parts[g];
      PartView v = commit_view_of(ctx, p, next_level);
      if (p.whi > p.wlo) {
        if (light)
          launches += launch_commit_light_count(v, off, next_level, ctx->run.p, sms, s);
        else
          launches += launch_commit_count(v, off, ctx->run.p, sms, s, parent_pass);
      }
      if (nwords - (p.whi - p.wlo) > 0) {
        k_commit_rest<<<resident_grid(k_commit_rest, nwords, 256, sms), 256, 0, s>>>(v, next_level);
        ++launches;
      }
    }
    // Termination: node 0's synchronized frontier.  With
    // direction optimization the next phase-1 direction is chosen here, from
    // every node's next-frontier edge count and the degree sum of everything
    // visited so far, before the commit's write half (which skips the queue
    // when phase 1 will run bottom-up).
    bool next_bu = ctx->direction == 2;
    int64_t frontier = -1;
    if (ctx->direction == 1) {
      BFB_CUDA(cudaMemcpyAsync(ctx->pinned, &ctx->parts[0].ctr.p->frontier, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
      for (int g = 0; g < P; ++g)
        BFB_CUDA(cudaMemcpyAsync(ctx->pinned + 2 + g, &ctx->parts[g].ctr.p->q_edges,
                                 sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      BFB_CUDA(cudaMemcpyAsync(ctx->pinned + 1, &ctx->run.p->traversed_edges, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
      BFB_CUDA(cudaStreamSynchronize(s));
      frontier = ctx->pinned[0];
      int64_t mf = 0;
      for (int g = 0; g < P; ++g) mf += ctx->pinned[2 + g];
      switch_chk += (level + 1) * mf;
      const double mu = (double)(ctx->g.m - ctx->pinned[1]);  // unexplored edges
      next_bu = bottom_up;
      if (!bottom_up && (double)mf > mu / ctx->do_alpha && frontier > prev_frontier)
        next_bu = true;
      else if (bottom_up && (double)frontier < (double)n / ctx->do_beta && frontier < prev_frontier)
        next_bu = false;
    }
    for (int g = 0; g < P && !sparse; ++g) {
      Part& p = ctx->parts[g];
      if (p.whi <= p.wlo) continue;
      if (light) {
        if (!next_bu)
          launches += launch_commit_rebuild(commit_view_of(ctx, p, next_level), off, next_level,
                                            ctx->run.p, sms, s);
      } else {
        launches += launch_commit_write(commit_view_of(ctx, p, next_level), off, next_level,
                                        !next_bu, sms, s);
      }
    }
    if (ctx->timing) BFB_CUDA(cudaEventRecord(D->ev[5], s));
    // node 0's counters: q_count, q_edges (the next frontier's edges, for
    // the sparse decision), frontier; the other nodes' q_edges
    BFB_CUDA(cudaMemcpyAsync(ctx->pinned + 5, ctx->parts[0].ctr.p, 3 * sizeof(int64_t),
                             cudaMemcpyDeviceToHost, s));
    for (int g = 1; g < P && sparse_ok; ++g)
      BFB_CUDA(cudaMemcpyAsync(ctx->pinned + 8 + g, &ctx->parts[g].ctr.p->q_edges,
                               sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaStreamSynchronize(s));
    BFB_CUDA(cudaGetLastError());
    cur_edges = ctx->pinned[6];
    for (int g = 1; g < P && sparse_ok; ++g) cur_edges += ctx->pinned[8 + g];
    if (ctx->timing) {
      float a = 0, b = 0, c = 0;
      BFB_CUDA(cudaEventElapsedTime(&a, D->ev[2], D->ev[3]));
      BFB_CUDA(cudaEventElapsedTime(&b, D->ev[3], D->ev[4]));
      BFB_CUDA(cudaEventElapsedTime(&c, D->ev[4], D->ev[5]));
      t_expand += a;
      t_exchange += b;
      t_commit += c;
      float mx = 0;
      for (int g = 0; part_timing && g < P; ++g) {
        float d = 0;
        BFB_CUDA(cudaEventElapsedTime(&d, D->part_ev[g], D->part_ev[g + 1]));
        mx = std::max(mx, d);
      }
      t_expand_max += part_timing ? mx : a;
    }
    frontier = ctx->pinned[7];
    if (frontier == 0) break;
    bottom_up = next_bu;
    prev_frontier = frontier;
    if (nsizes < max_levels && sizes_out) sizes_out[nsizes] = frontier;
    ctx->last_sizes.push_back(frontier);
    ++nsizes;
    reached += frontier;
    ++level;
    if (level > n) return fail(BFB_ERR_CAPACITY, "level count exceeded |V| (internal error)");
  }
  // d_local at termination (the relabelled engine writes node 0's straight
  // into the caller's ids below)
  if (!ctx->relabeled)
    for (int g = 0; g < P; ++g) launches += launch_materialise_levels(ctx, ctx->parts[g], level + 1, s);
  // Parents of the output view: any node's phase-1 claim is a valid parent.
  const uint32_t* parents_dev = nullptr;
  if (ctx->want_parents) {
    if (P == 1) {
      parents_dev = ctx->parts[0].parent.p;
    } else {
      k_parents_min<<<grid_cap(n, 256, sms, 8), 256, 0, s>>>(D->parents.p, P, n,
                                                             D->parents_final.p);
      parents_dev = D->parents_final.p;
      ++launches;
    }
  }
  // results in the caller's ids (relabelled engine graph), inside the timed
  // region: levels and parents final on device
  if (ctx->relabeled) {
    launches += launch_output(ctx, ctx->parts[0], level + 1, parents_dev, true, s);
    if (parents_dev) parents_dev = ctx->out_parent.p;
  }
  BFB_CUDA(cudaEventRecord(D->ev[1], s));
  // Stats
  RunCounters rc;
  BFB_CUDA(cudaMemcpyAsync(&rc, ctx->run.p, sizeof(rc), cudaMemcpyDeviceToHost, s));
  std::vector<int64_t> hw(P);
  BFB_CUDA(cudaMemcpyAsync(hw.data(), ctx->high_water.p, P * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, s));
  if (levels_out) BFB_TRY(read_levels(ctx, out_levels(ctx), n, nsizes, levels_out, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  float elapsed = 0;
  BFB_CUDA(cudaEventElapsedTime(&elapsed, D->ev[0], D->ev[1]));
  if (parents_out) {
    if (!ctx->want_parents) return fail(BFB_ERR_STATE, "engine set up without parents");
    if (P == 1 && !ctx->relabeled)  // (the un-permute masked them already)
      k_mask_parents<<<grid_cap(n, 256, sms, 8), 256, 0, s>>>(ctx->parts[0].level.p,
                                                              ctx->parts[0].parent.p, n);
    BFB_TRY(read_parents(ctx, parents_dev, n, parents_out, s));
    BFB_CUDA(cudaStreamSynchronize(s));
  }
  if (hw_out) std::memcpy(hw_out, hw.data(), P * sizeof(int64_t));
  ctx->have_run = true;
  ctx->last_root = root;
  ctx->last_levels = nsizes;
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->levels = nsizes;
    st->rounds_executed = nsizes * (int64_t)ctx->schedule.size();
    st->remote_messages = rc.remote_messages;
    st->remote_vertices = rc.remote_vertices;
    st->traversed_edges = rc.traversed_edges;
    st->reached = reached;
    int64_t mx = 0;
    for (auto x : hw) mx = std::max(mx, x);
    st->buffer_high_water_max = mx;
    st->exchange_bytes = rc.exchange_bytes;
    st->elapsed_ms = elapsed;
    st->expand_ms = t_expand;
    st->exchange_ms = t_exchange;
    st->commit_ms = t_commit;
    st->expand_launches = expand_launches;
    st->kernel_launches = launches;
    st->edges_examined = rc.edges_examined;
    st->bottom_up_levels = bu_levels;
    st->expand_max_part_ms = t_expand_max;
    st->switch_checksum = switch_chk;
    st->sparse_levels = sparse_levels;
  }
  if (rc.disagree)
    return fail(BFB_ERR_CAPACITY, "frontier disagreement after phase 2 (" +
                                      std::to_string(rc.disagree) + " bitmap words differ)");
  // buffer-bound check: incoming <= f * |V|
  for (auto x : hw)
    if (x > (int64_t)ctx->fanout * n && ctx->strategy == BFB_STRATEGY_BUTTERFLY)
      return fail(BFB_ERR_CAPACITY, "buffer bound violated");
  return BFB_OK;
}

int engine_copy_levels(bfb_ctx* ctx, uint32_t* out) {
  if (!ctx->have_run) return fail(BFB_ERR_STATE, "no BFS has run");
  BFB_TRY(read_levels(ctx, out_levels(ctx), ctx->g.n, ctx->last_levels, out, ctx->stream));
  BFB_CUDA(cudaStreamSynchronize(ctx->stream));
  return BFB_OK;
}

// Device array of the last run's output parents (kNone where unreached).
static int output_parents(bfb_ctx* ctx, const uint32_t** out) {
  EngineTables* D = ctx->tables;
  if (ctx->relabeled) {  // mapped back (and masked) by the run's un-permute
    *out = ctx->out_parent.p;
    return BFB_OK;
  }
  if (ctx->num_parts > 1) {
    *out = D->parents_final.p;
    return BFB_OK;
  }
  Part& p = ctx->parts[0];
  k_mask_parents<<<grid_cap(ctx->g.n, 256, ctx->num_sms, 8), 256, 0, ctx->stream>>>(
      p.level.p, p.parent.p, ctx->g.n);
  BFB_CUDA(cudaGetLastError());
  *out = p.parent.p;
  return BFB_OK;
}

int engine_copy_parents(bfb_ctx* ctx, int64_t* out) {
  if (!ctx->have_run) return fail(BFB_ERR_STATE, "no BFS has run");
  if (!ctx->want_parents) return fail(BFB_ERR_STATE, "engine set up without parents");
  const uint32_t* src = nullptr;
  BFB_TRY(output_parents(ctx, &src));
  BFB_TRY(read_parents(ctx, src, ctx->g.n, out, ctx->stream));
  BFB_CUDA(cudaStreamSynchronize(ctx->stream));
  return BFB_OK;
}

int engine_validate(bfb_ctx* ctx, int64_t root, int64_t* errs) {
  if (!ctx->have_run) return fail(BFB_ERR_STATE, "no BFS has run");
  if (!ctx->g.full()) return fail(BFB_ERR_STATE, "the certificate needs the whole graph");
  const uint32_t* par = nullptr;
  if (ctx->want_parents) BFB_TRY(output_parents(ctx, &par));
  DevBuf<unsigned> err;
  BFB_TRY(err.alloc(1));
  BFB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(unsigned), ctx->stream));
  // the caller's graph and ids: independent of the engine's relabel
  k_validate<<<grid_cap(ctx->g.n * 32, 256, ctx->num_sms, 16), 256, 0, ctx->stream>>>(
      ctx->g.offsets.p, ctx->g.adj.p, ctx->g.n, out_levels(ctx), par, root, err.p);
  unsigned h = 0;
  BFB_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  BFB_CUDA(cudaStreamSynchronize(ctx->stream));
  *errs = (int64_t)h;
  return BFB_OK;
}

__global__ void k_parents_from_i64(const int64_t* __restrict__ in, uint32_t* __restrict__ out,
                                   int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = in[i];
    out[i] = (p < 0 || p >= (int64_t)kNone) ? kNone : (uint32_t)p;
  }
}

int validate_host(bfb_ctx* ctx, int64_t root, const uint32_t* levels, const int64_t* parents,
                  int64_t* errs) {
  if (!ctx->g.full()) return fail(BFB_ERR_STATE, "the certificate needs the whole graph");
  const int64_t n = ctx->g.n;
  cudaStream_t s = ctx->stream;
  DevBuf<uint32_t> lv, par;
  DevBuf<int64_t> par64;
  DevBuf<unsigned> err;
  BFB_TRY(lv.alloc(n));
  BFB_TRY(err.alloc(1));
  BFB_CUDA(cudaMemcpyAsync(lv.p, levels, n * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  if (parents) {
    BFB_TRY(par64.alloc(n));
    BFB_TRY(par.alloc(n));
    BFB_CUDA(cudaMemcpyAsync(par64.p, parents, n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    k_parents_from_i64<<<grid_cap(n, 256, ctx->num_sms, 8), 256, 0, s>>>(par64.p, par.p, n);
  }
  BFB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(unsigned), s));
  k_validate<<<grid_cap(n * 32, 256, ctx->num_sms, 16), 256, 0, s>>>(
      ctx->g.offsets.p, ctx->g.adj.p, n, lv.p, parents ? par.p : nullptr, root, err.p);
  unsigned h = 0;
  BFB_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  *errs = (int64_t)h;
  return BFB_OK;
}

// ------------------------------------------------------ multi-process mode --
// One process per GPU (torchrun): this context runs node `rank` of CN.  The
// host driver (paper_2103_13577_b200/dist.py) sequences the steps below and
// provides the cross-process barrier + snapshot-size exchange between publish
// and merge; peers' snapshots are read directly from their HBM (CUDA IPC).

int rank_setup(bfb_ctx* ctx, int parts, const int64_t* bounds, int fanout, int strategy,
               int want_parents, int rank) {
  if (rank < 0 || rank >= parts) return fail(BFB_ERR_INVALID, "rank out of range");
  if (parts > kMaxSrc) return fail(BFB_ERR_INVALID, "at most 64 nodes in multi-process mode");
  const int64_t n = ctx->g.n;
  if (bounds[0] != 0 || bounds[parts] != n)
    return fail(BFB_ERR_PARTITION, "partition does not match graph");
  for (int g = 0; g < parts; ++g)
    if (bounds[g + 1] < bounds[g]) return fail(BFB_ERR_PARTITION, "partition does not match graph");
  if (!ctx->g.full() && (ctx->g.row_lo != bounds[rank] || ctx->g.row_hi != bounds[rank + 1]))
    return fail(BFB_ERR_PARTITION, "this context holds the rows of another part");
  // Validate and allocate as a single-node engine over the local part, then
  // re-label it with the global partition.  The engine graph is relabelled
  // within the GLOBAL partition, so every rank holds the same relabel.
  BFB_TRY(engine_setup_rb(ctx, 1, std::vector<int64_t>{0, ctx->g.n}.data(), 1, strategy,
                          want_parents, std::vector<int64_t>(bounds, bounds + parts + 1)));
  if (fanout < 1 || fanout > parts) return fail(BFB_ERR_FANOUT, "fanout exceeds num_nodes");
  BFB_TRY(make_schedule(parts, fanout, strategy, ctx->schedule));
  ctx->num_parts = parts;
  ctx->fanout = fanout;
  ctx->bounds.assign(bounds, bounds + parts + 1);
  // hubs sit at every part's start of the global relabel: probes stay default-cached
  ctx->hot_limit = parts == 1 ? ctx->hot_limit : kNone;
  BFB_TRY(build_hot_mask(ctx, ctx->bounds));
  // host scratch for P nodes (the mailbox copy of rank_bfs)
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  ctx->pinned = nullptr;
  ++alloc_counter();
  BFB_CUDA(cudaMallocHost(&ctx->pinned, sizeof(int64_t) * (8 + 8 * (size_t)parts)));
  EngineTables* D = ctx->tables;
  D->rank = rank;
  Part& p = ctx->parts[0];
  p.lo = bounds[rank];
  p.hi = bounds[rank + 1];
  p.wlo = p.lo >> 5;
  p.whi = p.hi == p.lo ? (p.lo >> 5) : ((p.hi + 31) >> 5);
  int64_t ob[2];
  BFB_CUDA(cudaMemcpy(&ob[0], ctx->g.offsets.p + p.lo, sizeof(int64_t), cudaMemcpyDeviceToHost));
  BFB_CUDA(cudaMemcpy(&ob[1], ctx->g.offsets.p + p.hi, sizeof(int64_t), cudaMemcpyDeviceToHost));
  p.owned_edges = ob[1] - ob[0];
  const int64_t nwords = (n + 31) / 32;
  const int64_t nwords_pad = (nwords + kWordPad - 1) / kWordPad * kWordPad + kWordPad;
  BFB_TRY(p.pub.alloc(nwords_pad));
  BFB_TRY(p.pub_alt.alloc(nwords_pad));
  BFB_CUDA(cudaMemset(p.pub.p, 0, nwords_pad * sizeof(uint32_t)));
  BFB_CUDA(cudaMemset(p.pub_alt.p, 0, nwords_pad * sizeof(uint32_t)));
  for (int par = 0; par < 2; ++par) D->peer_pub[par].assign(parts, nullptr);
  D->peer_pub[0][rank] = p.pub.p;
  D->peer_pub[1][rank] = p.pub_alt.p;
  BFB_TRY(p.pub_q.alloc(2 * (size_t)nwords_pad));
  BFB_TRY(D->mail.alloc(kMail * (size_t)parts));
  BFB_CUDA(cudaMemset(D->mail.p, 0, kMail * (size_t)parts * sizeof(int64_t)));
  BFB_TRY(D->peer_mail_dev.alloc(parts));
  BFB_TRY(D->err.alloc(1));
  BFB_CUDA(cudaMemset(D->err.p, 0, sizeof(int32_t)));
  D->peer_mail.assign(parts, nullptr);
  D->peer_mail[rank] = D->mail.p;
  D->peer_q.assign(parts, nullptr);
  D->peer_q[rank] = p.pub_q.p;
  D->peer_parent.assign(parts, nullptr);
  if (want_parents) {
    D->peer_parent[rank] = p.parent.p;
    BFB_TRY(D->parents_final.alloc(n + 1));
    BFB_TRY(D->parents.alloc(parts));  // peers' parent pointers (rank_parents)
  }
  D->seq = 0;
  if (ctx->direction) BFB_CUDA(cudaMemset(p.front.p, 0, nwords_pad * sizeof(uint32_t)));
  return BFB_OK;
}

int rank_ipc_handles(bfb_ctx* ctx, void* out) {
  if (!ctx->tables || ctx->tables->rank < 0) return fail(BFB_ERR_STATE, "not in rank mode");
  cudaIpcMemHandle_t h[5];
  std::memset(h, 0, sizeof(h));
  BFB_CUDA(cudaIpcGetMemHandle(&h[0], ctx->parts[0].pub.p));
  BFB_CUDA(cudaIpcGetMemHandle(&h[1], ctx->parts[0].pub_alt.p));
  BFB_CUDA(cudaIpcGetMemHandle(&h[2], ctx->tables->mail.p));
  BFB_CUDA(cudaIpcGetMemHandle(&h[3], ctx->parts[0].pub_q.p));
  if (ctx->want_parents) BFB_CUDA(cudaIpcGetMemHandle(&h[4], ctx->parts[0].parent.p));
  std::memcpy(out, h, sizeof(h));
  return BFB_OK;
}

int rank_open_peer(bfb_ctx* ctx, int peer, const void* handles) {
  EngineTables* D = ctx->tables;
  if (!D || D->rank < 0) return fail(BFB_ERR_STATE, "not in rank mode");
  if (peer < 0 || peer >= ctx->num_parts || peer == D->rank)
    return fail(BFB_ERR_INVALID, "bad peer");
  cudaIpcMemHandle_t h[5];
  std::memcpy(h, handles, sizeof(h));
  for (int k = 0; k < (ctx->want_parents ? 5 : 4); ++k) {
    void* ptr = nullptr;
    BFB_CUDA(cudaIpcOpenMemHandle(&ptr, h[k], cudaIpcMemLazyEnablePeerAccess));
    D->opened.push_back(ptr);
    if (k < 2)
      D->peer_pub[k][peer] = static_cast<const uint32_t*>(ptr);
    else if (k == 2)
      D->peer_mail[peer] = static_cast<int64_t*>(ptr);
    else if (k == 3)
      D->peer_q[peer] = static_cast<const uint32_t*>(ptr);
    else
      D->peer_parent[peer] = static_cast<uint32_t*>(ptr);
  }
  return BFB_OK;
}

int rank_begin(bfb_ctx* ctx, int64_t root) {
  EngineTables* D = ctx->tables;
  if (!D || D->rank < 0) return fail(BFB_ERR_STATE, "not in rank mode");
  const int64_t n = ctx->g.n;
  if (root < 0 || root >= n)
    return fail(BFB_ERR_ROOT, "root " + std::to_string(root) + " out of range [0, " +
                                  std::to_string(n) + ")");
  for (int par = 0; par < 2; ++par)
    for (int g = 0; g < ctx->num_parts; ++g)
      if (!D->peer_pub[par][g]) return fail(BFB_ERR_STATE, "peer snapshots not mapped");
  cudaStream_t s = ctx->stream;
  Part& p = ctx->parts[0];
  const int64_t nwords = (n + 31) / 32;
  BFB_CUDA(cudaEventRecord(D->ev[0], s));
  BFB_CUDA(cudaMemsetAsync(ctx->run.p, 0, sizeof(RunCounters), s));
  BFB_CUDA(cudaMemsetAsync(D->err.p, 0, sizeof(int32_t), s));  // a past barrier timeout
  BFB_CUDA(cudaMemsetAsync(p.visited.p, 0, nwords * sizeof(uint32_t), s));
  BFB_CUDA(cudaMemsetAsync(p.start.p, 0, nwords * sizeof(uint32_t), s));
  if (ctx->want_parents) BFB_CUDA(cudaMemsetAsync(p.parent.p, 0xFF, n * sizeof(uint32_t), s));
  if (ctx->direction) BFB_CUDA(cudaMemsetAsync(p.front.p, 0, nwords * sizeof(uint32_t), s));
  const int owner = root >= p.lo && root < p.hi;
  k_seed<<<1, 256, 0, s>>>(view_of(ctx, p), EG(ctx).offsets.p, root, perm_of(ctx), owner,
                           ctx->run.p);
  BFB_CUDA(cudaGetLastError());
  D->level = 0;
  D->levels = 1;
  D->reached = 1;
  ctx->last_sizes.assign(1, 1);
  ctx->lvbits_valid = 0xFFFFFFFFu;
  D->launches = 1;
  D->remote_messages = D->remote_vertices = D->high_water = D->exchange_bytes = 0;
  ctx->last_root = root;
  return BFB_OK;
}

int rank_expand(bfb_ctx* ctx) {
  PartView v = view_of(ctx, ctx->parts[0]);
  if (ctx->want_parents)
    launch_expand<true>(ctx->expand_grid, v, EG(ctx).adj_index(), ctx->stream);
  else
    launch_expand<false>(ctx->expand_grid, v, EG(ctx).adj_index(), ctx->stream);
  ++ctx->tables->launches;
  BFB_CUDA(cudaGetLastError());
  return BFB_OK;
}

int rank_publish(bfb_ctx* ctx, int parity, int64_t* count_out) {
  cudaStream_t s = ctx->stream;
  Part& p = ctx->parts[0];
  PartView v = view_of(ctx, p);
  v.pub = parity ? p.pub_alt.p : p.pub.p;
  const int64_t nwords = (ctx->g.n + 31) / 32;
  BFB_CUDA(cudaMemsetAsync(&p.ctr.p->pub_count[parity], 0, sizeof(int64_t), s));
  k_publish<<<grid_cap(nwords, 256, ctx->num_sms, 4), 256, 0, s>>>(v, parity);
  ++ctx->tables->launches;
  BFB_CUDA(cudaMemcpyAsync(ctx->pinned, &p.ctr.p->pub_count[parity], sizeof(int64_t),
                           cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  *count_out = ctx->pinned[0];
  return BFB_OK;
}

int rank_merge(bfb_ctx* ctx, int parity, const int32_t* srcs, const int64_t* counts, int nsrc) {
  EngineTables* D = ctx->tables;
  SrcList L;
  L.n = 0;
  int64_t incoming = 0;
  for (int i = 0; i < nsrc; ++i) {
    const int g = srcs[i];
    if (g < 0 || g >= ctx->num_parts || g == D->rank) return fail(BFB_ERR_INVALID, "bad source");
    if (counts[i] <= 0) continue;  // empty-buffer suppression
    L.p[L.n++] = D->peer_pub[parity][g];
    incoming += counts[i];
  }
  const int64_t nwords = (ctx->g.n + 31) / 32;
  D->remote_messages += L.n;
  D->remote_vertices += incoming;
  D->exchange_bytes += (int64_t)L.n * nwords * (int64_t)sizeof(uint32_t);
  D->high_water = std::max(D->high_water, incoming);
  if (incoming > (int64_t)ctx->fanout * ctx->g.n && ctx->strategy == BFB_STRATEGY_BUTTERFLY)
    return fail(BFB_ERR_CAPACITY, "buffer bound violated");
  if (L.n == 0) return BFB_OK;
  k_merge_peers<<<grid_cap(nwords, 256, ctx->num_sms, 4), 256, 0, ctx->stream>>>(
      L, ctx->parts[0].visited.p, nwords);
  ++D->launches;
  BFB_CUDA(cudaGetLastError());
  return BFB_OK;
}

int rank_commit(bfb_ctx* ctx, int64_t* frontier_out, int64_t* owned_out) {
  EngineTables* D = ctx->tables;
  cudaStream_t s = ctx->stream;
  Part& p = ctx->parts[0];
  const int64_t nwords = (ctx->g.n + 31) / 32;
  const uint32_t next_level = (uint32_t)(D->level + 1);
  PartView v = commit_view_of(ctx, p, next_level);
  k_commit_prep<<<1, 32, 0, s>>>(D->ctrs.p, 1);
  ++D->launches;
  if (p.whi > p.wlo) {
    D->launches += launch_commit(v, EG(ctx).offsets.p, next_level, ctx->run.p, ctx->num_sms, s);
  }
  if (nwords - (p.whi - p.wlo) > 0) {
    k_commit_rest<<<resident_grid(k_commit_rest, nwords, 256, ctx->num_sms), 256, 0, s>>>(v, next_level);
    ++D->launches;
  }
  BFB_CUDA(cudaMemcpyAsync(ctx->pinned, p.ctr.p, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  BFB_CUDA(cudaGetLastError());
  const int64_t f = ctx->pinned[2];  // PartCounters: q_count, q_edges, frontier
  *frontier_out = f;
  *owned_out = ctx->pinned[0];
  if (f) {
    ++D->level;
    ++D->levels;
    D->reached += f;
    ctx->last_sizes.push_back(f);
  }
  return BFB_OK;
}

int rank_finish(bfb_ctx* ctx, bfb_run_stats* st) {
  EngineTables* D = ctx->tables;
  cudaStream_t s = ctx->stream;
  if (ctx->relabeled)
    D->launches += launch_output(ctx, ctx->parts[0], D->level + 1, nullptr, true, s);
  else
    D->launches += launch_materialise_levels(ctx, ctx->parts[0], D->level + 1, s);
  BFB_CUDA(cudaEventRecord(D->ev[1], s));
  RunCounters rc;
  BFB_CUDA(cudaMemcpyAsync(&rc, ctx->run.p, sizeof(rc), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  float elapsed = 0;
  BFB_CUDA(cudaEventElapsedTime(&elapsed, D->ev[0], D->ev[1]));
  ctx->have_run = true;
  ctx->last_levels = D->levels;
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->levels = D->levels;
    st->rounds_executed = D->levels * (int64_t)ctx->schedule.size();
    st->remote_messages = D->remote_messages;
    st->remote_vertices = D->remote_vertices;
    st->traversed_edges = rc.traversed_edges;  // this node's q_local edges only
    st->reached = D->reached;
    st->buffer_high_water_max = D->high_water;
    st->exchange_bytes = D->exchange_bytes;
    st->elapsed_ms = elapsed;
    st->kernel_launches = D->launches;
  }
  return BFB_OK;
}

// Output parents of the last rank_bfs: element-wise min over every node's
// phase-1 parents, read in place from the peers' HBM (all ranks must have
// finished the BFS -- the caller's barrier).
int rank_parents(bfb_ctx* ctx, int64_t* out) {
  EngineTables* D = ctx->tables;
  if (!D || D->rank < 0) return fail(BFB_ERR_STATE, "not in rank mode");
  if (!ctx->want_parents) return fail(BFB_ERR_STATE, "engine set up without parents");
  const int P = ctx->num_parts;
  for (int g = 0; g < P; ++g)
    if (!D->peer_parent[g]) return fail(BFB_ERR_STATE, "peer parents not mapped");
  BFB_CUDA(cudaMemcpy(D->parents.p, D->peer_parent.data(), P * sizeof(uint32_t*),
                      cudaMemcpyHostToDevice));
  const int64_t n = ctx->g.n;
  k_parents_min<<<grid_cap(n, 256, ctx->num_sms, 8), 256, 0, ctx->stream>>>(
      D->parents.p, P, n, D->parents_final.p);
  const uint32_t* src = D->parents_final.p;
  if (ctx->relabeled) {
    launch_output(ctx, ctx->parts[0], D->level + 1, D->parents_final.p, false, ctx->stream);
    src = ctx->out_parent.p;
  }
  BFB_TRY(read_parents(ctx, src, n, out, ctx->stream));
  BFB_CUDA(cudaStreamSynchronize(ctx->stream));
  return BFB_OK;
}

int rank_parents_raw(bfb_ctx* ctx, uint32_t* out) {
  if (!ctx->want_parents) return fail(BFB_ERR_STATE, "engine set up without parents");
  const uint32_t* src = ctx->parts[0].parent.p;
  if (ctx->relabeled) {  // this node's claims at the caller's ids
    launch_output(ctx, ctx->parts[0], ctx->tables->level + 1, src, false, ctx->stream);
    BFB_CUDA(cudaStreamSynchronize(ctx->stream));
    src = ctx->out_parent.p;
  }
  BFB_CUDA(cudaMemcpy(out, src, ctx->g.n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return BFB_OK;
}


// ------------------------------------------- device-synchronised rank mode --
// rank_bfs runs a whole BFS for node `rank` with no host round trip inside a
// level: each butterfly round is publish -> signal -> wait -> merge, where
// signal writes {seq, snapshot size} into every peer's mailbox over NVLink
// (release at system scope) and wait spins (acquire) until every peer's slot
// in this node's mailbox reached seq -- the Synchronize() of PAPER.md:350 as a
// device barrier.  The merge then reads the scheduled sources' snapshot
// bitmaps in place and their sizes from the mailbox (empty sources skipped,
// SPEC.md:346).  The host syncs once per level, for the frontier count
// (termination): every node holds the same synchronized
// frontier after phase 2, so every rank reaches the same decision alone.
namespace {

__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}

// Mailbox slot of writer w: [kMail*w + parity] = snapshot size of w's last
// round of that parity, [kMail*w + 2] = w's last published round (seq),
// [kMail*w + 3/4] = w's owned share of the committed frontier and its edges
// (the per-level all-reduce; the edges pick the next level's mode).  The
// sizes are double-buffered like the snapshots: a writer can run one round
// ahead of a reader that is still merging, never two.

// One thread per peer: write this node's size and seq into its mailbox.
__global__ void k_signal(int64_t* const* peer_mail, int me, int num_nodes, int64_t seq,
                         const PartCounters* ctr, int parity) {
  const int g = threadIdx.x;
  if (g >= num_nodes || g == me) return;
  int64_t* slot = peer_mail[g] + kMail * me;
  slot[parity] = ((volatile const PartCounters*)ctr)->pub_count[parity];
  st_release_sys(slot + 2, seq);  // orders the snapshot and the size before seq
}

// Spin until every peer's seq in this node's mailbox reached `seq`; gives up
// after `timeout_ns` (sets *err) so a lost peer can never hang the GPU.
__global__ void k_wait(const int64_t* mail, int me, int num_nodes, int64_t seq, int32_t* err,
                       uint64_t timeout_ns) {
  const int g = threadIdx.x;
  if (g >= num_nodes || g == me) return;
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_sys(mail + kMail * g + 2) < seq) {
    if (globaltimer_ns() - t0 > timeout_ns) {
      atomicOr(err, 1);
      return;
    }
    __nanosleep(200);
  }
}

// Termination all-reduce (the north star's per-level frontier
// count reduction) over the same mailboxes: every node writes its owned share
// of the next frontier (slot 3) and the barrier seq into every peer's
// mailbox; after the barrier each node sums the shares and checks the sum
// against the frontier it committed itself (err bit 2 on disagreement).
__global__ void k_signal_count(int64_t* const* peer_mail, int me, int num_nodes, int64_t seq,
                               const PartCounters* ctr) {
  const int g = threadIdx.x;
  if (g >= num_nodes || g == me) return;
  int64_t* slot = peer_mail[g] + kMail * me;
  slot[3] = ((volatile const PartCounters*)ctr)->q_count;
  slot[4] = ((volatile const PartCounters*)ctr)->q_edges;
  st_release_sys(slot + 2, seq);
}

__global__ void k_check_count(const int64_t* mail, int me, int num_nodes, const PartCounters* ctr,
                              int32_t* err) {
  if (threadIdx.x) return;
  int64_t sum = ctr->q_count;
  for (int g = 0; g < num_nodes; ++g)
    if (g != me) sum += ld_acquire_sys(mail + kMail * g + 3);
  if (sum != ctr->frontier) atomicOr(err, 2);
}

struct RoundSrc {
  const uint32_t* pub[kMaxSrc];  // bitmap snapshot of this round's parity
  const uint32_t* q[kMaxSrc];    // queue-form snapshot of this round's parity
  int id[kMaxSrc];
  int n;
};

// Publish for the device-synchronised mode: the round-start snapshot
// visited & ~start as a bitmap (always) and, while it stays below qcap
// entries, also as a vertex queue; a reader pulls whichever is smaller
// (4 B per vertex vs n/8 B), so sparse rounds move only their vertices over
// NVLink.  One atomic per warp reserves queue space.
__global__ void __launch_bounds__(256) k_publish_q(PartView v, int parity, uint32_t* __restrict__ q,
                                                   int64_t qcap) {
  const int lane = threadIdx.x & 31;
  int64_t cnt = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nq = (v.nwords + 3) >> 2;
  const int64_t nq_round = (nq + 31) & ~(int64_t)31;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nq_round; c += stride) {
    uint4 p = make_uint4(0, 0, 0, 0);
    if (c < nq) {
      p = andnot4(ld4(v.visited + 4 * c), ld4(v.start + 4 * c));
      st4(v.pub + 4 * c, p);
    }
    const int n4 = popc4(p);
    cnt += n4;
    int incl = n4;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    if (tot == 0) continue;
    int64_t base = 0;
    if (lane == 31) base = (int64_t)atomicAdd((unsigned long long*)&v.ctr->pub_qpos[parity],
                                              (unsigned long long)tot);
    base = __shfl_sync(0xffffffffu, base, 31);
    if (base + tot > qcap) continue;  // dense snapshot: readers use the bitmap
    int64_t pos = base + incl - n4;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      for (uint32_t x = word4(p, k); x; x &= x - 1)
        q[pos++] = (uint32_t)(((4 * c + k) << 5) + __ffs(x) - 1);
  }
  __shared__ int64_t red[32];
  cnt = block_sum_i64(cnt, red);
  if (threadIdx.x == 0 && cnt)
    atomicAdd((unsigned long long*)&v.ctr->pub_count[parity], (unsigned long long)cnt);
}

// Queue-form sources of a round: set each listed vertex's bit (several
// sources and threads may hit one word, so atomically).
// Sparse levels (sq != nullptr): a vertex this merge sets for the first
// time is appended to the node's claim queue, which stays the node's whole
// new-vertex set (the next round's snapshot and the commit's input).
__global__ void k_merge_queue(RoundSrc R, const int64_t* mail, int parity, int64_t qcap,
                              uint32_t* __restrict__ vis, uint32_t* sq, PartCounters* ctr) {
  for (int i = 0; i < R.n; ++i) {
    const int64_t k = mail[kMail * R.id[i] + parity];
    if (k <= 0 || k > qcap) continue;
    const uint32_t* __restrict__ q = R.q[i];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k;
         j += (int64_t)gridDim.x * blockDim.x) {
      const uint32_t u = q[j];
      const uint32_t bit = 1u << (u & 31);
      if (vis[u >> 5] & bit) continue;
      const uint32_t old = atomicOr(&vis[u >> 5], bit);
      if (sq && !(old & bit)) append_claim(sq, &ctr->sq_claims, u);
    }
  }
}

// Sparse-level publish (rank mode): the round-start snapshot is the claim
// queue itself (phase-1 claims + earlier rounds' merges), copied into this
// round's queue slot -- O(snapshot) instead of a sweep over the bitmaps.  The
// snapshot stays below the queue cap (the level's frontier edges bound it),
// so readers never look at the bitmap form.
__global__ void k_publish_sparse(const uint32_t* __restrict__ sq, PartCounters* ctr, int parity,
                                 uint32_t* __restrict__ q) {
  const int64_t k = (int64_t)ctr->sq_claims;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k;
       j += (int64_t)gridDim.x * blockDim.x)
    q[j] = sq[j];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctr->pub_count[parity] = k;
    ctr->pub_qpos[parity] = k;
  }
}

// OR the non-empty sources' snapshots into visited (this node is the only
// writer of its bitmap during the merge).
__global__ void k_merge_mail(RoundSrc R, const int64_t* mail, int parity, int64_t qcap,
                             uint32_t* __restrict__ vis, int64_t nwords) {
  uint64_t live = 0;  // bitmap-form sources: non-empty and above the queue cap
  for (int i = 0; i < R.n; ++i)
    if (mail[kMail * R.id[i] + parity] > qcap) live |= 1ull << i;
  if (!live) return;
  const int64_t nq = (nwords + 3) >> 2;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nq;
       c += (int64_t)gridDim.x * blockDim.x) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (uint64_t m = live; m; m &= m - 1) {
      const uint4 x = ld4(R.pub[__ffsll((long long)m) - 1] + 4 * c);
      acc.x |= x.x;
      acc.y |= x.y;
      acc.z |= x.z;
      acc.w |= x.w;
    }
    if (acc.x | acc.y | acc.z | acc.w) {
      const uint4 cur = ld4(vis + 4 * c);
      const uint4 nb = andnot4(acc, cur);
      if (nb.x | nb.y | nb.z | nb.w)
        st4(vis + 4 * c, make_uint4(cur.x | acc.x, cur.y | acc.y, cur.z | acc.z, cur.w | acc.w));
    }
  }
}

// RunStats accounting of one round from the mailbox sizes (one thread).
__global__ void k_account_mail(RoundSrc R, const int64_t* mail, int parity, RunCounters* run,
                               int64_t* hw, int64_t bitmap_bytes, int64_t qcap) {
  if (threadIdx.x) return;
  int64_t msgs = 0, in = 0, bytes = 0;
  for (int i = 0; i < R.n; ++i) {
    const int64_t k = mail[kMail * R.id[i] + parity];
    if (k > 0) {
      ++msgs;
      in += k;
      bytes += k <= qcap ? 4 * k : bitmap_bytes;
    }
  }
  run->remote_messages += msgs;
  run->remote_vertices += in;
  run->exchange_bytes += bytes;
  if (in > *hw) *hw = in;
}

}  // namespace

int rank_bfs(bfb_ctx* ctx, int64_t root, int64_t* sizes_out, int64_t max_levels,
             bfb_run_stats* st) {
  EngineTables* D = ctx->tables;
  if (!D || D->rank < 0) return fail(BFB_ERR_STATE, "not in rank mode");
  const int P = ctx->num_parts, me = D->rank;
  for (int g = 0; g < P; ++g)
    if (!D->peer_mail[g]) return fail(BFB_ERR_STATE, "peer mailboxes not mapped");
  BFB_CUDA(cudaMemcpy(D->peer_mail_dev.p, D->peer_mail.data(), P * sizeof(int64_t*),
                      cudaMemcpyHostToDevice));
  BFB_TRY(rank_begin(ctx, root));
  cudaStream_t s = ctx->stream;
  Part& p = ctx->parts[0];
  const int64_t n = ctx->g.n, nwords = (n + 31) / 32;
  const int64_t* off = EG(ctx).offsets.p;
  const int sms = ctx->num_sms;
  const int64_t bytes_per_transfer = nwords * (int64_t)sizeof(uint32_t);
  const uint64_t timeout_ns = 60ull * 1000 * 1000 * 1000;
  // queue-form snapshots pay off below n/32 vertices (4 B each vs n/8 B)
  const int64_t qcap = (nwords + kWordPad - 1) / kWordPad * kWordPad + kWordPad;
  BFB_CUDA(cudaMemsetAsync(ctx->high_water.p, 0, sizeof(int64_t), s));
  std::vector<RoundSrc> rounds;
  for (auto& rnd : ctx->schedule) {
    RoundSrc R{};
    for (int src : rnd[me]) {
      R.pub[R.n] = nullptr;  // filled per parity below
      R.id[R.n++] = src;
    }
    rounds.push_back(R);
  }
  bool bottom_up = ctx->direction == 2;
  int64_t bu_levels = 0, prev_frontier = 1, nsizes = 1, launches = 0;
  int64_t seen_edges = 0;  // degree sum of every frontier so far (direction switch)
  int64_t switch_chk = 0;
  if (ctx->direction == 1) {
    int64_t ob[2];
    // the root's degree (the caller's graph: the relabel keeps degrees)
    BFB_CUDA(cudaMemcpy(ob, ctx->g.offsets.p + root, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    seen_edges = ob[1] - ob[0];
  }
  if (sizes_out && max_levels > 0) sizes_out[0] = 1;
  double t_expand = 0, t_exchange = 0, t_commit = 0;
  int64_t expand_launches = 0;
  // sparse levels (as engine_bfs), decided on the GLOBAL frontier edge count
  // (own share + the peers' shares from the count all-reduce), so every
  // snapshot of the level stays in queue form: phase 1 queues its claims,
  // each round publishes the claim queue (no sweep), merges append what they
  // set, and the commit works from the queue (no sweep of the non-owned words)
  const bool sparse_ok = ctx->sparse_mode && ctx->direction != 2 && p.sparse_q.p != nullptr;
  const int64_t sparse_cap = std::min<int64_t>((int64_t)p.sparse_q.n, qcap - 1);
  int64_t global_edges = ctx->g.max_degree;  // the root's degree, bounded
  int64_t sparse_levels = 0;
  while (true) {
    const bool sparse = sparse_ok && !bottom_up && global_edges <= sparse_cap;
    PartView v = view_of(ctx, p);
    if (ctx->timing) BFB_CUDA(cudaEventRecord(D->ev[2], s));
    // parent pass as in engine_bfs, decided from global quantities (every
    // node the same way: the owner's pass covers the vertices that the other
    // nodes' store-free phase 1 found)
    const bool parent_pass = ctx->want_parents && !bottom_up &&
                             prev_frontier >= std::max<int64_t>(1, n >> 12) &&
                             D->reached >= pass_min_reached(n);
    if (bottom_up) {
      const unsigned bg = grid_cap(std::max<int64_t>(1, v.whi - v.wlo), 256, sms, 8);
      unsigned long long* ex = (unsigned long long*)&ctx->run.p->edges_examined;
      if (ctx->want_parents)
        k_bottom_up<true><<<bg, 256, 0, s>>>(v, EG(ctx).adj_index(), ex);
      else
        k_bottom_up<false><<<bg, 256, 0, s>>>(v, EG(ctx).adj_index(), ex);
      ++bu_levels;
    } else {
      PartView ev = v;
      if (sparse) ev.sparse_q = p.sparse_q.p;
      if (ctx->want_parents && (!parent_pass || sparse))
        launch_expand<true>(ctx->expand_grid, ev, EG(ctx).adj_index(), s);
      else
        launch_expand<false>(ctx->expand_grid, ev, EG(ctx).adj_index(), s);
    }
    ++launches;
    ++expand_launches;
    if (ctx->timing) BFB_CUDA(cudaEventRecord(D->ev[3], s));
    for (RoundSrc R : rounds) {
      const int64_t seq = ++D->seq;
      const int parity = (int)(seq & 1);
      PartView pv = v;
      pv.pub = parity ? p.pub_alt.p : p.pub.p;
      for (int i = 0; i < R.n; ++i) {
        R.pub[i] = D->peer_pub[parity][R.id[i]];
        R.q[i] = D->peer_q[R.id[i]] + parity * qcap;
      }
      if (sparse) {
        k_publish_sparse<<<grid_cap(sparse_cap, 256, sms, 2), 256, 0, s>>>(
            p.sparse_q.p, p.ctr.p, parity, p.pub_q.p + parity * qcap);
      } else {
        BFB_CUDA(cudaMemsetAsync(&p.ctr.p->pub_count[parity], 0, sizeof(int64_t), s));
        BFB_CUDA(cudaMemsetAsync(&p.ctr.p->pub_qpos[parity], 0, sizeof(int64_t), s));
        k_publish_q<<<grid_cap(nwords, 256, sms, 4), 256, 0, s>>>(pv, parity,
                                                                  p.pub_q.p + parity * qcap, qcap);
      }
      k_signal<<<1, 64, 0, s>>>(D->peer_mail_dev.p, me, P, seq, p.ctr.p, parity);
      k_wait<<<1, 64, 0, s>>>(D->mail.p, me, P, seq, D->err.p, timeout_ns);
      k_account_mail<<<1, 32, 0, s>>>(R, D->mail.p, parity, ctx->run.p, ctx->high_water.p,
                                      bytes_per_transfer, qcap);
      launches += 4;
      if (R.n) {
        k_merge_queue<<<grid_cap(qcap, 256, sms, 2), 256, 0, s>>>(
            R, D->mail.p, parity, qcap, p.visited.p, sparse ? p.sparse_q.p : nullptr, p.ctr.p);
        k_merge_mail<<<grid_cap(nwords, 256, sms, 4), 256, 0, s>>>(R, D->mail.p, parity, qcap,
                                                                  p.visited.p, nwords);
        launches += 2;
      }
    }
    if (ctx->timing) BFB_CUDA(cudaEventRecord(D->ev[4], s));
    // commit: count pass, direction decision, write pass (as engine_bfs)
    const uint32_t next_level = (uint32_t)(D->level + 1);
    PartView cv = commit_view_of(ctx, p, next_level);
    cv.rest_degrees = ctx->direction == 1;
    k_commit_prep<<<1, 32, 0, s>>>(D->ctrs.p, 1);
    ++launches;
    if (ctx->direction) BFB_CUDA(cudaMemsetAsync(p.front.p, 0, nwords * sizeof(uint32_t), s));
    const bool light = ctx->direction != 0 && bottom_up;
    if (sparse) {
      PartView sv = view_of(ctx, p);
      sv.sparse_q = p.sparse_q.p;
      sv.rest_degrees = ctx->direction == 1;
      k_sparse_commit<<<grid_cap(sparse_cap, 256, sms, 8), 256, 0, s>>>(sv, off, next_level);
      k_sparse_finalize<<<1, 1, 0, s>>>(p.ctr.p, ctx->run.p);
      launches += 2;
      if (next_level < (uint32_t)kLevelBits) ctx->lvbits_valid &= ~(1u << next_level);
      ++sparse_levels;
    } else {
      if (p.whi > p.wlo) {
        if (light)
          launches += launch_commit_light_count(cv, off, next_level, ctx->run.p, sms, s);
        else
          launches += launch_commit_count(cv, off, ctx->run.p, sms, s, parent_pass);
      }
      if (nwords - (p.whi - p.wlo) > 0) {
        k_commit_rest<<<resident_grid(k_commit_rest, nwords, 256, sms), 256, 0, s>>>(cv, next_level);
        ++launches;
      }
    }
    bool next_bu = ctx->direction == 2;
    if (ctx->direction == 1) {
      // Beamer's rule on global quantities, so every node takes the same
      // direction: an edge (u on node g, v on node h) is traversed only if g
      // runs top-down or h bottom-up, so mixed directions would lose edges.
      // The next frontier's degree sum = owned part (count pass) + the
      // non-owned rest: the words outside [wlo, whi) (k_commit_rest) and the
      // neighbours' bits of the partial boundary words (count pass), so the
      // sum -- and the running sum -- is the same global number on all nodes.
      BFB_CUDA(cudaMemcpyAsync(ctx->pinned, p.ctr.p, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      BFB_CUDA(cudaMemcpyAsync(ctx->pinned + 3, &p.ctr.p->rest_edges, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
      BFB_CUDA(cudaStreamSynchronize(s));
      const int64_t frontier = ctx->pinned[2], mf = ctx->pinned[1] + ctx->pinned[3];
      seen_edges += mf;
      switch_chk += (D->level + 1) * mf;
      const double mu = (double)(ctx->g.m - seen_edges);
      next_bu = bottom_up;
      if (!bottom_up && (double)mf > mu / ctx->do_alpha && frontier > prev_frontier)
        next_bu = true;
      else if (bottom_up && (double)frontier < (double)n / ctx->do_beta && frontier < prev_frontier)
        next_bu = false;
    }
    if (p.whi > p.wlo && !sparse) {
      if (light) {
        if (!next_bu)
          launches += launch_commit_rebuild(cv, off, next_level, ctx->run.p, sms, s);
      } else {
        launches += launch_commit_write(cv, off, next_level, !next_bu, sms, s);
      }
    }
    // the level's frontier count, all-reduced over the nodes' owned shares
    // and checked against this node's own commit
    if (P > 1) {
      const int64_t cseq = ++D->seq;
      k_signal_count<<<1, 64, 0, s>>>(D->peer_mail_dev.p, me, P, cseq, p.ctr.p);
      k_wait<<<1, 64, 0, s>>>(D->mail.p, me, P, cseq, D->err.p, timeout_ns);
      k_check_count<<<1, 32, 0, s>>>(D->mail.p, me, P, p.ctr.p, D->err.p);
      launches += 3;
    }
    if (ctx->timing) BFB_CUDA(cudaEventRecord(D->ev[5], s));
    BFB_CUDA(cudaMemcpyAsync(ctx->pinned, p.ctr.p, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaMemcpyAsync(ctx->pinned + 4, D->err.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (P > 1 && sparse_ok)  // the peers' shares of the next frontier's edges
      BFB_CUDA(cudaMemcpyAsync(ctx->pinned + 8, D->mail.p, kMail * (size_t)P * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaStreamSynchronize(s));
    BFB_CUDA(cudaGetLastError());
    global_edges = ctx->pinned[1];
    for (int g = 0; g < P && sparse_ok; ++g)
      if (g != me) global_edges += ctx->pinned[8 + kMail * g + 4];
    const int32_t errs = *(int32_t*)(ctx->pinned + 4);
    if (errs & 1) return fail(BFB_ERR_CUDA, "peer barrier timed out (a rank stopped participating)");
    if (errs & 2)
      return fail(BFB_ERR_CAPACITY, "frontier disagreement: the nodes' owned shares do not sum "
                                    "to the committed frontier");
    if (ctx->timing) {
      float a = 0, b = 0, c = 0;
      BFB_CUDA(cudaEventElapsedTime(&a, D->ev[2], D->ev[3]));
      BFB_CUDA(cudaEventElapsedTime(&b, D->ev[3], D->ev[4]));
      BFB_CUDA(cudaEventElapsedTime(&c, D->ev[4], D->ev[5]));
      t_expand += a;
      t_exchange += b;
      t_commit += c;
    }
    const int64_t f = ctx->pinned[2];
    if (f == 0) break;
    bottom_up = next_bu;
    prev_frontier = f;
    ++D->level;
    ++D->levels;
    D->reached += f;
    ctx->last_sizes.push_back(f);
    if (sizes_out && nsizes < max_levels) sizes_out[nsizes] = f;
    ++nsizes;
    if (D->level > n) return fail(BFB_ERR_CAPACITY, "level count exceeded |V| (internal error)");
  }
  D->launches += launches;
  BFB_TRY(rank_finish(ctx, st));
  RunCounters rc;
  int64_t hw = 0;
  BFB_CUDA(cudaMemcpy(&rc, ctx->run.p, sizeof(rc), cudaMemcpyDeviceToHost));
  BFB_CUDA(cudaMemcpy(&hw, ctx->high_water.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (st) {
    st->remote_messages = rc.remote_messages;
    st->remote_vertices = rc.remote_vertices;
    st->exchange_bytes = rc.exchange_bytes;
    st->buffer_high_water_max = hw;
    st->edges_examined = rc.edges_examined;
    st->bottom_up_levels = bu_levels;
    st->expand_ms = t_expand;
    st->exchange_ms = t_exchange;
    st->commit_ms = t_commit;
    st->expand_launches = expand_launches;
    st->switch_checksum = switch_chk;
    st->sparse_levels = sparse_levels;
  }
  if (hw > (int64_t)ctx->fanout * n && ctx->strategy == BFB_STRATEGY_BUTTERFLY)
    return fail(BFB_ERR_CAPACITY, "buffer bound violated");
  return BFB_OK;
}

}  // namespace bfb
