// Internal declarations shared by the libbflybfs translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "bflybfs.h"

namespace bfb {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define BFB_CUDA(call)                                                  \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) return ::bfb::cuda_fail(e_, #call, __FILE__, __LINE__); \
  } while (0)

#define BFB_TRY(call)             \
  do {                            \
    int rc_ = (call);             \
    if (rc_ != BFB_OK) return rc_; \
  } while (0)

// ------------------------------------------------------- device buffers --
// Owning device allocation.  All engine buffers are created in setup calls;
// bfb_bfs itself never allocates -- every
// device and pinned-host allocation of the library bumps alloc_counter(),
// which the allocation-freedom test reads around bfb_bfs (bfb_alloc_count).
int64_t& alloc_counter();
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  int alloc(size_t count) {
    release();
    if (count == 0) count = 1;
    ++alloc_counter();
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return fail(BFB_ERR_OOM, "device allocation of " + std::to_string(count * sizeof(T)) +
                                   " bytes failed: " + cudaGetErrorString(e));
    }
    n = count;
    return BFB_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// ------------------------------------------------------------- PCG64 -----
// numpy's PCG64: 128-bit LCG, state stepped before output, XSL-RR output,
// random() = (next64 >> 11) * 2^-53.  An affine map x -> a*x + c (mod 2^128)
// represents "advance by k steps", so jump-ahead is square-and-multiply.
struct U128 {
  uint64_t hi, lo;
};

__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}

__host__ __device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

struct Affine {
  U128 a, c;  // x -> a*x + c
};

__host__ __device__ __forceinline__ U128 apply(const Affine& f, U128 x) {
  return add128(mul128(f.a, x), f.c);
}

// g after f
__host__ __device__ __forceinline__ Affine compose(const Affine& g, const Affine& f) {
  Affine r;
  r.a = mul128(g.a, f.a);
  r.c = add128(mul128(g.a, f.c), g.c);
  return r;
}

__host__ __device__ __forceinline__ Affine affine_pow(Affine step, uint64_t k) {
  Affine acc;
  acc.a = U128{0, 1};
  acc.c = U128{0, 0};
  while (k) {
    if (k & 1) acc = compose(step, acc);
    step = compose(step, step);
    k >>= 1;
  }
  return acc;
}

__host__ __device__ __forceinline__ uint64_t xsl_rr(U128 s) {
  uint64_t x = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr uint64_t kPcgMultHi = 0x2360ED051FC65DA4ULL;
constexpr uint64_t kPcgMultLo = 0x4385DF649FCCF645ULL;

// ------------------------------------------------------------ graph -------
struct DevGraph {
  int64_t n = 0, m = 0, max_degree = 0;
  DevBuf<int64_t> offsets;   // n+1 (always the whole graph)
  DevBuf<uint32_t> adj;      // adjacency of rows [row_lo, row_hi) (all m entries when full)
  // A partitioned build (one rank's share, bfb_graph_from_rmat_part) keeps
  // only its own rows' adjacency: entries [adj_lo, adj_lo + adj.n) of the
  // global adjacency; kernels index it with adj_index() and global offsets.
  int64_t row_lo = 0, row_hi = 0, adj_lo = 0;
  bool full() const { return row_lo == 0 && row_hi == n; }
  const uint32_t* adj_index() const { return adj.p - adj_lo; }
  DevBuf<uint32_t> nonisol;  // bitmap of degree > 0 (bottom-up candidates), built at engine setup
  DevBuf<uint16_t> deg16;    // min(degree, 65535) per vertex (commit degree sums), engine setup
  DevBuf<uint32_t> first_nbr; // lowest-id neighbour per vertex, then (second half) the second-lowest
                              // (parent pass / bottom-up first probes), engine setup
  bool valid = false;
};

// ------------------------------------------------------------ engine ------
// Device-resident counters of one node (compute node = part).
struct PartCounters {
  int64_t q_count;      // |q_local| (owned frontier)
  int64_t q_edges;      // sum of degrees over q_local
  int64_t frontier;     // |synchronized next frontier| counted at commit
  int64_t pub_count[2]; // published snapshot size, by round parity (phase 2)
  int64_t pub_qpos[2];  // queue-form snapshot fill (device-synchronised mode)
  int64_t work_next;    // commit write pass: next unit to hand out (dense levels)
  int64_t bu_next;      // bottom-up phase 1: next 32-word group to hand out
  int64_t ex_next;      // top-down phase 1: next tile to hand out (dense levels)
  int64_t rest_edges;   // degree sum of the new vertices outside the owned range
                        // (rank mode, direction-optimizing: the global switch)
  unsigned long long sq_claims;  // sparse level: claims appended to the claim queue
  unsigned long long sq_packed;  // sparse commit: (count << 40) + edges, block-aggregated
};

// Device-resident run statistics (RunStats).
struct RunCounters {
  int64_t edges_examined;  // bottom-up levels: edges actually checked
  int64_t remote_messages;
  int64_t remote_vertices;
  int64_t traversed_edges;
  int64_t reached;
  int64_t exchange_bytes;
  int64_t disagree;        // checks mode: words where a node's frontier differs from node 0's
};

// One compute node's private world (NodeState).
struct Part {
  int64_t lo = 0, hi = 0;          // owned vertex range [lo, hi)
  int64_t wlo = 0, whi = 0;        // words touching the owned range
  int64_t owned_edges = 0;
  int64_t tile_cap = 0;
  DevBuf<uint32_t> visited;        // replicated visited bitmap (n bits)
  DevBuf<uint32_t> start;          // visited as of the level start
  DevBuf<uint32_t> level;          // d_local (n)
  DevBuf<uint32_t> parent;         // phase-1 parents (n) when wanted
  DevBuf<uint32_t> pub;            // published round snapshot (n bits)
  DevBuf<uint32_t> pub_alt;        // odd-round snapshot (multi-process mode)
  DevBuf<uint32_t> pub_q;          // queue-form snapshots, 2 x nwords entries (by parity)
  DevBuf<uint32_t> front;          // level-L frontier bitmap (bottom-up phase 1)
  DevBuf<uint32_t> lvbits;         // per level 1..kLevelBits-1: that level's new-vertex bitmap
  DevBuf<uint32_t> sparse_q;       // sparse levels: phase-1 claims (single node, top-down)
  DevBuf<uint32_t> q_v;            // q_local vertex ids, ascending
  DevBuf<int64_t> q_pre;           // exclusive degree prefix over q_local
  DevBuf<int64_t> q_base;          // offsets[v] - q_pre (adjacency base per row)
  DevBuf<uint32_t> tile_vstart;    // q_local index owning edge t*TILE
  DevBuf<uint32_t> unit_u32;       // commit: owned new vertices per 32-word unit
  DevBuf<int64_t> unit_i64;        // commit: unit degree sums, prefixes, scan tiles
  DevBuf<PartCounters> ctr;
};

}  // namespace bfb

namespace bfb {
struct EngineTables;  // bfs_engine.cu: device-side pointer/schedule tables
struct SmallEngine;   // small_bfs.cu: the single-CTA engine's tables

// One single-CTA run's results (small_bfs.cu)
struct SmallResult {
  std::vector<int64_t> sizes;  // per_level_frontier_size
  int64_t remote_messages = 0, remote_vertices = 0, exchange_bytes = 0, traversed_edges = 0,
          reached = 0, disagree = 0;
};

struct ReadPool;  // host_out.cu: persistent widening threads of the read-out

// Result read-out (host_out.cu): a page-locked staging area for the packed
// D2H copy and one event per pipelined chunk.
struct HostStage {
  void* p = nullptr;
  size_t bytes = 0;
  std::vector<cudaEvent_t> ev;
  HostStage() = default;
  HostStage(const HostStage&) = delete;
  HostStage& operator=(const HostStage&) = delete;
  ~HostStage() { release(); }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
  }
};
}

struct bfb_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  bfb::DevGraph g;
  // engine
  bool engine_ready = false;
  int num_parts = 0, fanout = 1, strategy = 0, want_parents = 0;
  std::vector<int64_t> bounds;
  std::vector<std::vector<std::vector<int>>> schedule;  // [round][node] -> sources
  std::vector<bfb::Part> parts;
  bfb::DevBuf<bfb::RunCounters> run;
  bfb::DevBuf<int64_t> high_water;    // per node
  int64_t* pinned = nullptr;          // host scratch (pinned)
  bfb::EngineTables* tables = nullptr;
  int expand_grid = 0;
  bool timing = false;
  int checks = 0;                     // bfb_set_checks: 1 = frontier agreement after phase 2
  int direction = 0;                  // 0 top-down, 1 direction-optimizing, 2 bottom-up
  double do_alpha = 14.0, do_beta = 64.0;  // tuned at s29 / s24 (Beamer: 14, 24)
  bool have_run = false;
  int64_t last_root = -1;
  int64_t last_levels = 0;
  std::vector<int64_t> last_sizes;     // per_level_frontier_size of the last run
  int64_t launches = 0;
  cudaEvent_t timer[2] = {nullptr, nullptr};
  // text ingestion: edges parsed by bfb_parse_text, awaiting the CSR build
  bfb::DevBuf<uint2> parsed;
  int64_t parsed_m = 0;
  // result read-out: packed levels on device, staging in host memory
  bfb::DevBuf<uint32_t> packed;
  bfb::HostStage stage;
  bfb::ReadPool* pool = nullptr;
  // the engine's degree-ordered relabel of the graph (relabel.cu), kept
  // across engine setups with the same partition: eg = relabelled CSR,
  // perm = old -> new id, inv = new -> old id; results are mapped back to
  // the caller's ids into out_level / out_parent
  bool relabeled = false;
  std::vector<int64_t> relabel_bounds;
  bfb::DevGraph eg;
  bfb::DevBuf<uint32_t> perm, inv;
  bfb::DevBuf<uint32_t> out_level, out_parent;
  bfb::DevBuf<uint8_t> lv8;  // engine-id levels, one byte each, gathered by the un-permute
  // small graphs: the whole BFS in one single-CTA launch (small_bfs.cu);
  // built at engine setup when the graph qualifies, used for top-down runs
  // while small_mode is on (bfb_set_small_engine)
  uint32_t lvbits_valid = 0xFFFFFFFFu;  // levels whose new-vertex bitmap the last run wrote
  int sparse_mode = 1;                  // sparse levels committed from the claim queue
  uint32_t hot_limit = 0xFFFFFFFFu;  // phase-1 probes of ids below it cache in L1 (bfs_engine.cu)
  bfb::DevBuf<uint32_t> hot_mask;    // several parts: the parts' hub blocks (bfs_engine.cu)
  bfb::SmallEngine* small = nullptr;
  int small_mode = 1;
};

namespace bfb {

// graph_build.cu
int build_from_rmat(bfb_ctx* ctx, int scale, int64_t ef, U128 state, U128 inc,
                    const uint64_t thr[3]);
int build_from_edges(bfb_ctx* ctx, int64_t n, const uint32_t* host_edges, int64_t m,
                     bool symmetrize);
int rmat_to_host(bfb_ctx* ctx, int scale, int64_t ef, U128 state, U128 inc, const uint64_t thr[3],
                 uint32_t* out);
int load_csr(bfb_ctx* ctx, int64_t n, int64_t m, const int64_t* offsets, const uint32_t* adj);
int build_from_device_edges(bfb_ctx* ctx, int64_t n, DevBuf<uint2>& edges, int64_t m,
                            bool symmetrize);
// one rank's share of the RMAT graph: the whole offsets (every vertex's
// degree) and only the adjacency of its partition_1d(parts) rows
int build_from_rmat_part(bfb_ctx* ctx, int scale, int64_t ef, U128 state, U128 inc,
                         const uint64_t thr[3], int parts, int rank, int64_t* bounds_out);
// ingest.cu
int parse_text(bfb_ctx* ctx, const char* data, int64_t len, int fmt, int nl, int64_t line0,
               int64_t rows, int64_t cols, bfb_parse_result* res);
int parsed_copy(bfb_ctx* ctx, uint32_t* out);
int write_edge_list(const char* path, const uint32_t* edges, int64_t m);
int graph_save(bfb_ctx* ctx, const char* path);
int graph_load(bfb_ctx* ctx, const char* path);
int copy_edges(bfb_ctx* ctx, uint32_t* out);
int partition_1d(bfb_ctx* ctx, int parts, int64_t* out);
int count_nonisolated(bfb_ctx* ctx, int64_t* out);
// host_out.cu: levels / parents from device to host (packed, pipelined,
// unpacked by host threads)
int read_levels(bfb_ctx* ctx, const uint32_t* level, int64_t n, int64_t num_levels,
                uint32_t* out, cudaStream_t s);
int read_parents(bfb_ctx* ctx, const uint32_t* parent, int64_t n, int64_t* out, cudaStream_t s);
// the read-out's buffers (packed levels, pinned stage, events, host threads),
// allocated at engine setup so bfb_bfs allocates nothing
int readout_setup(bfb_ctx* ctx, int64_t n);
void readout_release(bfb_ctx* ctx);
int select_nonisolated(bfb_ctx* ctx, const int64_t* ranks, int64_t k, int64_t* out);

// relabel.cu: the engine's degree-ordered relabel (within the parts of `bounds`)
bool relabel_wanted(const bfb_ctx* ctx);
int relabel_build(bfb_ctx* ctx, const std::vector<int64_t>& bounds);
void relabel_release(bfb_ctx* ctx);
// segsort.cu: per-row ascending sort of rows[rowstart[v]..rowstart[v+1]) into
// out (hand-written warp bitonic / block radix); keys < key_bound; clobbers rows
int sort_rows(bfb_ctx* ctx, const int64_t* rowstart, int64_t n, int64_t total, uint32_t* rows,
              uint32_t* out, int64_t key_bound);

// small_bfs.cu: the single-CTA engine for small graphs
bool small_eligible(const bfb_ctx* ctx, int parts, int total_pairs);
int small_setup(bfb_ctx* ctx);  // after the schedule / bounds are set; no-op if not eligible
void small_release(bfb_ctx* ctx);
int small_bfs(bfb_ctx* ctx, int64_t root, uint32_t* level, uint32_t* parent, int64_t* high_water,
              int checks, cudaEvent_t ev0, cudaEvent_t ev1, SmallResult* res);

// scan.cu: exclusive scan of n values produced by a loader -> int64 out[0..n]
// (out[n] = total).  Work buffers are sized by the caller via scan_tmp_words.
size_t scan_tmp_words(int64_t n);
int scan_u32_to_i64(const uint32_t* in, int64_t n, int64_t* out, int64_t* tmp,
                    cudaStream_t s);
int scan_popc_to_i64(const uint32_t* words, int64_t n, int64_t* out, int64_t* tmp,
                     cudaStream_t s);

// bfs_engine.cu
int engine_setup(bfb_ctx* ctx, int parts, const int64_t* bounds, int fanout, int strategy,
                 int want_parents);
int engine_bfs(bfb_ctx* ctx, int64_t root, uint32_t* levels_out, int64_t* parents_out,
               int64_t* sizes_out, int64_t max_levels, int64_t* hw_out, bfb_run_stats* st);
int engine_copy_levels(bfb_ctx* ctx, uint32_t* out);
int engine_copy_parents(bfb_ctx* ctx, int64_t* out);
int engine_validate(bfb_ctx* ctx, int64_t root, int64_t* errs);
int validate_host(bfb_ctx* ctx, int64_t root, const uint32_t* levels, const int64_t* parents,
                  int64_t* errs);
int probe_peak(bfb_ctx* ctx, int64_t bytes, int64_t* probes_out, double* ms_out);
void engine_release(bfb_ctx* ctx);

// bfs_engine.cu, multi-process mode: this context is node `rank` of CN
int rank_setup(bfb_ctx* ctx, int parts, const int64_t* bounds, int fanout, int strategy,
               int want_parents, int rank);
int rank_ipc_handles(bfb_ctx* ctx, void* out);
int rank_open_peer(bfb_ctx* ctx, int peer, const void* handles);
int rank_begin(bfb_ctx* ctx, int64_t root);
int rank_expand(bfb_ctx* ctx);
int rank_publish(bfb_ctx* ctx, int parity, int64_t* count_out);
int rank_merge(bfb_ctx* ctx, int parity, const int32_t* srcs, const int64_t* counts, int nsrc);
int rank_commit(bfb_ctx* ctx, int64_t* frontier_out, int64_t* owned_out);
int rank_finish(bfb_ctx* ctx, bfb_run_stats* st);
int rank_bfs(bfb_ctx* ctx, int64_t root, int64_t* sizes_out, int64_t max_levels,
             bfb_run_stats* st);
int rank_parents(bfb_ctx* ctx, int64_t* out);
int rank_parents_raw(bfb_ctx* ctx, uint32_t* out);

// schedule (capi.cu)
int make_schedule(int cn, int fanout, int strategy, std::vector<std::vector<std::vector<int>>>& out);

}  // namespace bfb
