// C ABI of libbflybfs.so (include/bflybfs.h): argument checking, error
// reporting, the host-side butterfly schedule, and dispatch to the device code.
#include <cstdio>
#include <cstring>

#include "bfb_internal.cuh"

namespace bfb {

static thread_local std::string tl_error;

int64_t& alloc_counter() {
  static int64_t count = 0;  // bumped under the context mutex (or in setup-only paths)
  return count;
}

void set_error(const std::string& msg) { tl_error = msg; }

int fail(int code, const std::string& msg) {
  tl_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                cudaGetErrorString(e), what, file, line);
  cudaGetLastError();
  tl_error = buf;
  return e == cudaErrorMemoryAllocation ? BFB_ERR_OOM : BFB_ERR_CUDA;
}

// butterfly-schedule (decisions SPEC.md:245-250): radix
// r = 2 for fanout 1, else fanout; in round i node g pulls from the nodes that
// differ from g in base-r digit i; a missing source s >= CN is replaced by its
// subgroup representative s - s % r^i, dropped if that is >= CN or == g.
int make_schedule(int cn, int fanout, int strategy, std::vector<std::vector<std::vector<int>>>& out) {
  out.clear();
  if (cn < 1) return fail(BFB_ERR_INVALID, "num_nodes must be >= 1");
  if (fanout < 1) return fail(BFB_ERR_FANOUT, "fanout must be >= 1");
  if (fanout > cn) return fail(BFB_ERR_FANOUT, "fanout exceeds num_nodes");
  if (strategy == BFB_STRATEGY_ALL2ALL) {
    if (cn > 1) {  // one round, every peer
      std::vector<std::vector<int>> rnd(cn);
      for (int g = 0; g < cn; ++g)
        for (int s = 0; s < cn; ++s)
          if (s != g) rnd[g].push_back(s);
      out.push_back(std::move(rnd));
    }
    return BFB_OK;
  }
  if (strategy != BFB_STRATEGY_BUTTERFLY) return fail(BFB_ERR_INVALID, "unknown strategy");
  const int64_t r = fanout == 1 ? 2 : fanout;
  int64_t w = 1;
  while (w < cn) {
    std::vector<std::vector<int>> rnd(cn);
    for (int64_t g = 0; g < cn; ++g) {
      const int64_t cleared = g - ((g / w) % r) * w;
      for (int64_t digit = 0; digit < r; ++digit) {
        int64_t s = cleared + digit * w;
        if (s == g) continue;
        if (s >= cn) {
          s -= s % w;
          if (s >= cn || s == g) continue;
        }
        rnd[g].push_back((int)s);
      }
    }
    out.push_back(std::move(rnd));
    w *= r;
  }
  return BFB_OK;
}

}  // namespace bfb

using namespace bfb;

#define CTX_GUARD(ctx)                                               \
  if (!(ctx)) return fail(BFB_ERR_INVALID, "null context");          \
  std::lock_guard<std::mutex> lock_((ctx)->mu);                      \
  if (cudaSetDevice((ctx)->device) != cudaSuccess)                   \
    return fail(BFB_ERR_CUDA, "cudaSetDevice failed")

#define NEED_GRAPH(ctx) \
  if (!(ctx)->g.valid) return fail(BFB_ERR_STATE, "no graph loaded")
#define NEED_FULL_GRAPH(ctx)  \
  if (!(ctx)->g.full())       \
  return fail(BFB_ERR_STATE, "this context holds one rank's rows only (partitioned build)")

// The single-context entry points (bfb_bfs and its read-outs) index every
// node's buffers; after bfb_rank_setup the context holds one node only.
namespace bfb {
bool rank_mode(const bfb_ctx* ctx);
}
#define NOT_RANK_MODE(ctx)                                                      \
  if (bfb::rank_mode(ctx))                                                      \
  return fail(BFB_ERR_STATE, "context is in multi-process (rank) mode: use bfb_rank_*")
#define NEED_RANK_MODE(ctx) \
  if (!bfb::rank_mode(ctx)) return fail(BFB_ERR_STATE, "not in rank mode (bfb_rank_setup first)")

extern "C" {

const char* bfb_version(void) { return "bflybfs-b200 0.1 (sm_100a)"; }

const char* bfb_last_error(void) { return tl_error.c_str(); }

int bfb_device_count(int* count_out) {
  if (!count_out) return fail(BFB_ERR_INVALID, "null output");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count_out = 0;
    return fail(BFB_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  *count_out = c;
  return BFB_OK;
}

int bfb_host_alloc(size_t bytes, void** ptr_out) {
  if (!ptr_out) return fail(BFB_ERR_INVALID, "null output");
  *ptr_out = nullptr;
  cudaError_t e = cudaHostAlloc(ptr_out, bytes ? bytes : 1, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(BFB_ERR_OOM, std::string("cudaHostAlloc failed: ") + cudaGetErrorString(e));
  }
  return BFB_OK;
}

void bfb_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

int bfb_num_rounds(int num_nodes, int fanout, int* rounds_out) {
  std::vector<std::vector<std::vector<int>>> s;
  BFB_TRY(make_schedule(num_nodes, fanout, BFB_STRATEGY_BUTTERFLY, s));
  *rounds_out = (int)s.size();
  return BFB_OK;
}

int bfb_make_schedule(int num_nodes, int fanout, int strategy, int32_t* out, int64_t cap,
                      int64_t* len_out) {
  std::vector<std::vector<std::vector<int>>> s;
  BFB_TRY(make_schedule(num_nodes, fanout, strategy, s));
  int64_t len = 0;
  for (auto& rnd : s)
    for (auto& srcs : rnd) len += 1 + (int64_t)srcs.size();
  if (len_out) *len_out = len;
  if (!out || cap < len) return out ? fail(BFB_ERR_INVALID, "schedule buffer too small") : BFB_OK;
  int64_t k = 0;
  for (auto& rnd : s)
    for (auto& srcs : rnd) {
      out[k++] = (int32_t)srcs.size();
      for (int x : srcs) out[k++] = x;
    }
  return BFB_OK;
}

int bfb_message_count_paper(int num_nodes, int fanout, int64_t* out) {
  int rounds = 0;
  BFB_TRY(bfb_num_rounds(num_nodes, fanout, &rounds));
  *out = (int64_t)num_nodes * fanout * rounds;
  return BFB_OK;
}

int64_t bfb_buffer_bound(int64_t num_vertices, int fanout) { return (int64_t)fanout * num_vertices; }

int64_t bfb_alloc_count(void) { return alloc_counter(); }

int bfb_create(bfb_ctx** ctx_out, int device) {
  if (!ctx_out) return fail(BFB_ERR_INVALID, "null output");
  *ctx_out = nullptr;
  int count = 0;
  BFB_TRY(bfb_device_count(&count));
  if (device < 0 || device >= count)
    return fail(BFB_ERR_INVALID, "device " + std::to_string(device) + " not present");
  BFB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  BFB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(BFB_ERR_CUDA, std::string("libbflybfs is built for sm_100a; device is ") +
                                  prop.name);
  auto* ctx = new bfb_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return cuda_fail(e, "cudaStreamCreate", __FILE__, __LINE__);
  }
  *ctx_out = ctx;
  return BFB_OK;
}

void bfb_destroy(bfb_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  engine_release(ctx);
  relabel_release(ctx);
  readout_release(ctx);
  ctx->g = DevGraph();
  for (auto& e : ctx->timer)
    if (e) cudaEventDestroy(e);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int bfb_set_timing(bfb_ctx* ctx, int enabled) {
  CTX_GUARD(ctx);
  ctx->timing = enabled != 0;
  return BFB_OK;
}

int bfb_set_checks(bfb_ctx* ctx, int flags) {
  CTX_GUARD(ctx);
  if (flags < 0 || flags > 1) return fail(BFB_ERR_INVALID, "unknown check flags");
  ctx->checks = flags;
  return BFB_OK;
}

int bfb_set_small_engine(bfb_ctx* ctx, int enabled) {
  CTX_GUARD(ctx);
  ctx->small_mode = enabled != 0;
  return BFB_OK;
}

int bfb_set_sparse_levels(bfb_ctx* ctx, int enabled) {
  CTX_GUARD(ctx);
  ctx->sparse_mode = enabled != 0;
  return BFB_OK;
}

int bfb_small_engine_active(bfb_ctx* ctx) {
  if (!ctx) return 0;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return ctx->small && ctx->small_mode && ctx->direction == 0 ? 1 : 0;
}

int bfb_set_direction(bfb_ctx* ctx, int mode, double alpha, double beta) {
  CTX_GUARD(ctx);
  if (mode < 0 || mode > 2 || !(alpha > 0) || !(beta > 0))
    return fail(BFB_ERR_INVALID, "bad direction parameters");
  ctx->direction = mode;
  ctx->do_alpha = alpha;
  ctx->do_beta = beta;
  return BFB_OK;
}

int bfb_timer_start(bfb_ctx* ctx) {
  CTX_GUARD(ctx);
  if (!ctx->timer[0]) {
    BFB_CUDA(cudaEventCreate(&ctx->timer[0]));
    BFB_CUDA(cudaEventCreate(&ctx->timer[1]));
  }
  BFB_CUDA(cudaEventRecord(ctx->timer[0], ctx->stream));
  return BFB_OK;
}

int bfb_timer_stop(bfb_ctx* ctx, double* elapsed_ms_out) {
  CTX_GUARD(ctx);
  if (!ctx->timer[0]) return fail(BFB_ERR_STATE, "timer not started");
  BFB_CUDA(cudaEventRecord(ctx->timer[1], ctx->stream));
  BFB_CUDA(cudaEventSynchronize(ctx->timer[1]));
  float ms = 0;
  BFB_CUDA(cudaEventElapsedTime(&ms, ctx->timer[0], ctx->timer[1]));
  if (elapsed_ms_out) *elapsed_ms_out = ms;
  return BFB_OK;
}

static U128 u128_of(const uint64_t v[2]) { return U128{v[0], v[1]}; }

int bfb_rmat_edges(bfb_ctx* ctx, int scale, int64_t edge_factor, const uint64_t pcg_state[2],
                   const uint64_t pcg_inc[2], const uint64_t thresholds[3], uint32_t* edges_out) {
  CTX_GUARD(ctx);
  if (!pcg_state || !pcg_inc || !thresholds || !edges_out)
    return fail(BFB_ERR_INVALID, "null argument");
  return rmat_to_host(ctx, scale, edge_factor, u128_of(pcg_state), u128_of(pcg_inc), thresholds,
                      edges_out);
}

int bfb_graph_from_rmat(bfb_ctx* ctx, int scale, int64_t edge_factor, const uint64_t pcg_state[2],
                        const uint64_t pcg_inc[2], const uint64_t thresholds[3]) {
  CTX_GUARD(ctx);
  if (!pcg_state || !pcg_inc || !thresholds) return fail(BFB_ERR_INVALID, "null argument");
  return build_from_rmat(ctx, scale, edge_factor, u128_of(pcg_state), u128_of(pcg_inc),
                         thresholds);
}

int bfb_graph_from_rmat_part(bfb_ctx* ctx, int scale, int64_t edge_factor,
                             const uint64_t pcg_state[2], const uint64_t pcg_inc[2],
                             const uint64_t thresholds[3], int num_parts, int rank,
                             int64_t* boundaries_out) {
  CTX_GUARD(ctx);
  if (!pcg_state || !pcg_inc || !thresholds || !boundaries_out)
    return fail(BFB_ERR_INVALID, "null argument");
  return build_from_rmat_part(ctx, scale, edge_factor, u128_of(pcg_state), u128_of(pcg_inc),
                              thresholds, num_parts, rank, boundaries_out);
}

int bfb_graph_rows(bfb_ctx* ctx, int64_t* row_lo_out, int64_t* row_hi_out,
                   int64_t* adjacency_entries_out) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  if (row_lo_out) *row_lo_out = ctx->g.row_lo;
  if (row_hi_out) *row_hi_out = ctx->g.row_hi;
  if (adjacency_entries_out) *adjacency_entries_out = ctx->g.full() ? ctx->g.m : (int64_t)ctx->g.adj.n - 1;
  return BFB_OK;
}

int bfb_graph_from_edges(bfb_ctx* ctx, int64_t num_vertices, const uint32_t* edges, int64_t m,
                         int symmetrize) {
  CTX_GUARD(ctx);
  if (m && !edges) return fail(BFB_ERR_INVALID, "null edges");
  return build_from_edges(ctx, num_vertices, edges, m, symmetrize != 0);
}

int bfb_graph_load_csr(bfb_ctx* ctx, int64_t num_vertices, int64_t num_edges,
                       const int64_t* offsets, const uint32_t* adjacency) {
  CTX_GUARD(ctx);
  if (!offsets || (num_edges && !adjacency)) return fail(BFB_ERR_INVALID, "null argument");
  if (offsets[0] != 0 || offsets[num_vertices] != num_edges)
    return fail(BFB_ERR_INVALID, "offsets do not describe num_edges edges");
  return load_csr(ctx, num_vertices, num_edges, offsets, adjacency);
}

int bfb_graph_info(bfb_ctx* ctx, int64_t* n, int64_t* m, int64_t* maxdeg) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  if (n) *n = ctx->g.n;
  if (m) *m = ctx->g.m;
  if (maxdeg) *maxdeg = ctx->g.max_degree;
  return BFB_OK;
}

int bfb_graph_copy_csr(bfb_ctx* ctx, int64_t* offsets_out, uint32_t* adjacency_out) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  if (adjacency_out) NEED_FULL_GRAPH(ctx);
  if (offsets_out)
    BFB_CUDA(cudaMemcpy(offsets_out, ctx->g.offsets.p, (ctx->g.n + 1) * sizeof(int64_t),
                        cudaMemcpyDeviceToHost));
  if (adjacency_out && ctx->g.m)
    BFB_CUDA(cudaMemcpy(adjacency_out, ctx->g.adj.p, ctx->g.m * sizeof(uint32_t),
                        cudaMemcpyDeviceToHost));
  return BFB_OK;
}

int bfb_graph_copy_edges(bfb_ctx* ctx, uint32_t* edges_out) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  NEED_FULL_GRAPH(ctx);
  if (!edges_out && ctx->g.m) return fail(BFB_ERR_INVALID, "null output");
  return copy_edges(ctx, edges_out);
}

int bfb_partition_1d(bfb_ctx* ctx, int num_parts, int64_t* boundaries_out) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  if (!boundaries_out) return fail(BFB_ERR_INVALID, "null output");
  return partition_1d(ctx, num_parts, boundaries_out);
}

int bfb_count_nonisolated(bfb_ctx* ctx, int64_t* count_out) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  return count_nonisolated(ctx, count_out);
}

int bfb_select_nonisolated(bfb_ctx* ctx, const int64_t* ranks, int64_t k, int64_t* vertices_out) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  return select_nonisolated(ctx, ranks, k, vertices_out);
}

int bfb_engine_setup(bfb_ctx* ctx, int num_parts, const int64_t* boundaries, int fanout,
                     int strategy, int want_parents) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  if (!boundaries) return fail(BFB_ERR_INVALID, "null boundaries");
  return engine_setup(ctx, num_parts, boundaries, fanout, strategy, want_parents);
}

int bfb_bfs(bfb_ctx* ctx, int64_t root, uint32_t* levels_out, int64_t* parents_out,
            int64_t* frontier_sizes_out, int64_t max_levels, int64_t* buffer_high_water_out,
            bfb_run_stats* stats_out) {
  CTX_GUARD(ctx);
  NOT_RANK_MODE(ctx);
  NEED_GRAPH(ctx);
  return engine_bfs(ctx, root, levels_out, parents_out, frontier_sizes_out, max_levels,
                    buffer_high_water_out, stats_out);
}

int bfb_frontier_sizes(bfb_ctx* ctx, int64_t* out, int64_t cap, int64_t* len_out) {
  CTX_GUARD(ctx);
  const int64_t L = (int64_t)ctx->last_sizes.size();
  if (len_out) *len_out = L;
  for (int64_t i = 0; i < L && i < cap && out; ++i) out[i] = ctx->last_sizes[i];
  return BFB_OK;
}

int bfb_copy_levels(bfb_ctx* ctx, uint32_t* levels_out) {
  CTX_GUARD(ctx);
  return engine_copy_levels(ctx, levels_out);
}

int bfb_copy_parents(bfb_ctx* ctx, int64_t* parents_out) {
  CTX_GUARD(ctx);
  NOT_RANK_MODE(ctx);
  return engine_copy_parents(ctx, parents_out);
}

int bfb_validate(bfb_ctx* ctx, int64_t root, int64_t* errors_out) {
  CTX_GUARD(ctx);
  NOT_RANK_MODE(ctx);
  return engine_validate(ctx, root, errors_out);
}

int bfb_validate_host(bfb_ctx* ctx, int64_t root, const uint32_t* levels, const int64_t* parents,
                      int64_t* errors_out) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  if (!levels || !errors_out) return fail(BFB_ERR_INVALID, "null argument");
  if (root < 0 || root >= ctx->g.n) return fail(BFB_ERR_ROOT, "root out of range");
  return validate_host(ctx, root, levels, parents, errors_out);
}

int bfb_parse_text(bfb_ctx* ctx, const char* data, int64_t len, int fmt, int newline,
                   int64_t first_line_no, int64_t rows, int64_t cols, bfb_parse_result* result) {
  CTX_GUARD(ctx);
  if (!result || len < 0 || (len && !data) || (fmt != 0 && fmt != 1) || first_line_no < 0 ||
      (newline != 0 && newline != 1))
    return fail(BFB_ERR_INVALID, "bad arguments");
  return parse_text(ctx, data, len, fmt, newline, first_line_no, rows, cols, result);
}

int bfb_parsed_edges(bfb_ctx* ctx, uint32_t* edges_out) {
  CTX_GUARD(ctx);
  if (!edges_out && ctx->parsed_m) return fail(BFB_ERR_INVALID, "null output");
  return parsed_copy(ctx, edges_out);
}

int bfb_graph_from_parsed(bfb_ctx* ctx, int64_t num_vertices, int symmetrize) {
  CTX_GUARD(ctx);
  if (!ctx->parsed.p) return fail(BFB_ERR_STATE, "no parsed edges");
  bfb::DevBuf<uint2> edges(std::move(ctx->parsed));
  const int64_t m = ctx->parsed_m;
  ctx->parsed_m = 0;
  return build_from_device_edges(ctx, num_vertices, edges, m, symmetrize != 0);
}

int bfb_write_edge_list(const char* path, const uint32_t* edges, int64_t num_edges) {
  if (!path || num_edges < 0 || (num_edges && !edges)) return fail(BFB_ERR_INVALID, "bad arguments");
  return write_edge_list(path, edges, num_edges);
}

int bfb_graph_save(bfb_ctx* ctx, const char* path) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  NEED_FULL_GRAPH(ctx);
  if (!path) return fail(BFB_ERR_INVALID, "null path");
  return graph_save(ctx, path);
}

int bfb_graph_load(bfb_ctx* ctx, const char* path) {
  CTX_GUARD(ctx);
  if (!path) return fail(BFB_ERR_INVALID, "null path");
  return graph_load(ctx, path);
}

int bfb_probe_peak(bfb_ctx* ctx, int64_t bytes, int64_t* probes_out, double* ms_out) {
  CTX_GUARD(ctx);
  if (!probes_out || !ms_out || bytes <= 0) return fail(BFB_ERR_INVALID, "bad arguments");
  return probe_peak(ctx, bytes, probes_out, ms_out);
}

int bfb_rank_setup(bfb_ctx* ctx, int num_parts, const int64_t* boundaries, int fanout,
                   int strategy, int want_parents, int rank) {
  CTX_GUARD(ctx);
  NEED_GRAPH(ctx);
  if (!boundaries) return fail(BFB_ERR_INVALID, "null boundaries");
  return rank_setup(ctx, num_parts, boundaries, fanout, strategy, want_parents, rank);
}

int bfb_rank_ipc_handles(bfb_ctx* ctx, void* handles_out) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  if (!handles_out) return fail(BFB_ERR_INVALID, "null output");
  return rank_ipc_handles(ctx, handles_out);
}

int bfb_rank_open_peer(bfb_ctx* ctx, int peer, const void* handles) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  if (!handles) return fail(BFB_ERR_INVALID, "null handles");
  return rank_open_peer(ctx, peer, handles);
}

int bfb_rank_begin(bfb_ctx* ctx, int64_t root) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  return rank_begin(ctx, root);
}

int bfb_rank_expand(bfb_ctx* ctx) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  return rank_expand(ctx);
}

int bfb_rank_publish(bfb_ctx* ctx, int parity, int64_t* count_out) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  if (!count_out || (parity != 0 && parity != 1)) return fail(BFB_ERR_INVALID, "bad argument");
  return rank_publish(ctx, parity, count_out);
}

int bfb_rank_merge(bfb_ctx* ctx, int parity, const int32_t* sources, const int64_t* counts,
                   int num_sources) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  if (num_sources < 0 || (num_sources && (!sources || !counts)) || (parity != 0 && parity != 1))
    return fail(BFB_ERR_INVALID, "bad argument");
  return rank_merge(ctx, parity, sources, counts, num_sources);
}

int bfb_rank_commit(bfb_ctx* ctx, int64_t* frontier_out, int64_t* owned_out) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  if (!frontier_out || !owned_out) return fail(BFB_ERR_INVALID, "null output");
  return rank_commit(ctx, frontier_out, owned_out);
}

int bfb_rank_finish(bfb_ctx* ctx, bfb_run_stats* stats_out) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  return rank_finish(ctx, stats_out);
}

int bfb_rank_bfs(bfb_ctx* ctx, int64_t root, int64_t* sizes_out, int64_t max_levels,
                 bfb_run_stats* stats_out) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  if (max_levels < 0) return fail(BFB_ERR_INVALID, "bad argument");
  return rank_bfs(ctx, root, sizes_out, max_levels, stats_out);
}

int bfb_rank_parents(bfb_ctx* ctx, int64_t* parents_out) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  if (!parents_out) return fail(BFB_ERR_INVALID, "null output");
  return rank_parents(ctx, parents_out);
}

int bfb_rank_parents_raw(bfb_ctx* ctx, uint32_t* parents_out) {
  CTX_GUARD(ctx);
  NEED_RANK_MODE(ctx);
  if (!parents_out) return fail(BFB_ERR_INVALID, "null output");
  return rank_parents_raw(ctx, parents_out);
}

}  // extern "C"
