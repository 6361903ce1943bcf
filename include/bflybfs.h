/*
 * bflybfs.h -- C ABI of libbflybfs.so, the B200 (sm_100a) ButterFly BFS path.
 *
 * This library fills the native-kernel slot the reference declares but does
 * not ship (`bflybfs._kernels._ext`, pkg/setup.py:5-15; "compiled kernels are
 * built for uint32", pkg/src/bflybfs/graphs.py:11-12).  Every entry point
 * below names the reference interface it replaces.  Plain pointers and sizes
 * only; host arrays are borrowed for the duration of a call; the context owns
 * all device memory.  Return value 0 = success, negative = error (see codes);
 * bfb_last_error() gives the message of the last failure on this thread.
 *
 * Vertex ids are uint32 (graphs.py:13 VID), distances use UNREACHED =
 * 0xFFFFFFFF (graphs.py:17), offsets are int64 (graphs.py:59).
 */
#ifndef BFLYBFS_H_
#define BFLYBFS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes: the Python wrapper maps them to the reference's exceptions */
#define BFB_OK 0
#define BFB_ERR_INVALID (-1)        /* ValueError: bad argument                        */
#define BFB_ERR_ROOT (-2)           /* ValueError: root out of range */
#define BFB_ERR_PARTITION (-3)      /* ValueError: partition/graph mismatch */
#define BFB_ERR_FANOUT (-4)         /* ValueError: fanout > CN           */
#define BFB_ERR_SELF_EDGE (-5)      /* ValueError: graphs.py:240                       */
#define BFB_ERR_DUPLICATE (-6)      /* ValueError: graphs.py:244                       */
#define BFB_ERR_NO_REVERSE (-7)     /* ValueError: graphs.py:247                       */
#define BFB_ERR_RANGE (-8)          /* ValueError: endpoint >= num_vertices (graphs.py:44-45) */
#define BFB_ERR_STATE (-9)          /* RuntimeError: call order (no graph / no engine) */
#define BFB_ERR_CAPACITY (-10)      /* RuntimeError: buffer-bound violation */
#define BFB_ERR_PARSE (-11)         /* ValueError (ParseError): malformed text graph, see bfb_parse_result */
#define BFB_ERR_IO (-12)            /* OSError: file open/read/write failure           */
#define BFB_ERR_CUDA (-20)          /* RuntimeError: CUDA failure                      */
#define BFB_ERR_OOM (-21)           /* MemoryError: device allocation failed           */

#define BFB_STRATEGY_BUTTERFLY 0    /* SPEC.md:280 strategy = butterfly                */
#define BFB_STRATEGY_ALL2ALL 1      /* SPEC.md:280 strategy = all-to-all */

typedef struct bfb_ctx bfb_ctx;

/* RunStats plus device-side phase timings. */
typedef struct bfb_run_stats {
  int64_t levels;                    /* non-empty frontiers, = 1 + eccentricity       */
  int64_t rounds_executed;           /* butterfly rounds summed over levels           */
  int64_t remote_messages;           /* non-empty scheduled transfers   */
  int64_t remote_vertices;           /* sum of transferred snapshot sizes             */
  int64_t traversed_edges;           /* sum of deg(v) over reached v    */
  int64_t reached;                   /* vertices with a finite distance               */
  int64_t buffer_high_water_max;     /* max over nodes of per-round incoming vertices */
  int64_t exchange_bytes;            /* bytes the exchange moved between nodes        */
  double elapsed_ms;                 /* device time, root injection -> termination    */
  double expand_ms;                  /* phase 1 kernels (timing mode only)            */
  double exchange_ms;                /* phase 2 kernels (timing mode only)            */
  double commit_ms;                  /* level commit / frontier build (timing mode)   */
  int64_t expand_launches;           /* expand kernel launches in this run            */
  int64_t kernel_launches;           /* all kernels this library launched in the run  */
  int64_t edges_examined;            /* bottom-up levels: edges actually checked      */
  int64_t bottom_up_levels;          /* levels whose phase 1 ran bottom-up            */
  double expand_max_part_ms;         /* timing mode, CN > 1 in one context: sum over
                                        levels of the slowest node's phase 1 (the
                                        critical path if each node had its own GPU) */
  int64_t switch_checksum;           /* direction-optimizing: sum over levels of
                                        (level + 1) x the next frontier's degree sum
                                        that fed Beamer's rule -- equal on every node
                                        (rank mode) and to the one-context run */
  int64_t sparse_levels;             /* levels committed from the claim queue
                                        (bfb_set_sparse_levels)                       */
} bfb_run_stats;

/* Outcome of bfb_parse_text (graphs.py:96-202 ParseError carries the line). */
typedef struct bfb_parse_result {
  int64_t num_lines;     /* text lines parsed by the device                      */
  int64_t num_edges;     /* edge lines (entries) kept                            */
  int64_t max_id_plus1;  /* "edges": 1 + largest vertex id (0 if no edges)      */
  int64_t err_line;      /* 1-based line of the first error, 0 if none          */
  int32_t err_code;      /* 2 tokens, 3 non-integer id, 4 negative id, 5/6 src/dst
                            id > MAX_VID, 7 mtx entry tokens, 8 mtx non-integer,
                            9 mtx coordinate outside rows x cols                 */
  int32_t pad;
  int64_t err_begin, err_end;  /* byte range of the offending line in `data`    */
} bfb_parse_result;

/* ---- library ---------------------------------------------------------- */
const char* bfb_version(void);
const char* bfb_last_error(void);
int bfb_device_count(int* count_out);

/* Page-locked host memory for result arrays (fast D2H of levels/parents). */
int bfb_host_alloc(size_t bytes, void** ptr_out);
void bfb_host_free(void* ptr);

/* ---- butterfly-schedule (host-only, no GPU needed) ------ */
/* num_rounds(CN, f): SPEC.md:202-210 */
int bfb_num_rounds(int num_nodes, int fanout, int* rounds_out);
/* make_schedule(CN, f) or the all2all pattern.
 * Flattened into `out`: for each round, for each node g: count c, then c source ids.
 * *len_out = int32 entries written (or needed, if cap is too small -> BFB_ERR_INVALID). */
int bfb_make_schedule(int num_nodes, int fanout, int strategy, int32_t* out, int64_t cap,
                      int64_t* len_out);
/* message_count_paper */
int bfb_message_count_paper(int num_nodes, int fanout, int64_t* out);
/* buffer_bound */
int64_t bfb_buffer_bound(int64_t num_vertices, int fanout);

/* Allocation tracking (SPEC.md acceptance 4): device and pinned-host
 * allocations the library has made so far; equal before and after a
 * bfb_bfs / bfb_rank_bfs call, read-out included (allocation-freedom). */
int64_t bfb_alloc_count(void);

/* ---- context ----------------------------------------------------------- */
int bfb_create(bfb_ctx** ctx_out, int device);
void bfb_destroy(bfb_ctx* ctx);
/* Record per-phase CUDA events inside bfb_bfs (fills *_ms of bfb_run_stats). */
int bfb_set_timing(bfb_ctx* ctx, int enabled);
/* Instrumentation (SPEC.md acceptance 8): flags 1 = after every phase 2,
 * check that all nodes' visited bitmaps (levels so far + the synchronized
 * frontier) are identical; bfb_bfs then fails with BFB_ERR_CAPACITY on a
 * disagreement.  (Rank mode always all-reduces and checks the per-level
 * frontier count.)  0 = off (default). */
int bfb_set_checks(bfb_ctx* ctx, int flags);
/* Small graphs (|V| <= 2^15, |E| <= 2^21, CN <= 64, whole graph resident):
 * top-down runs execute every level of every node inside ONE single-CTA
 * kernel launch (no per-level launches or host round trips; deep graphs such
 * as SPEC.md:446's path(10000) are bound by them otherwise).  Same
 * DistanceArray, frontier sizes and RunStats counters as the level-synchronous
 * engine, except exchange_bytes (4 B per listed vertex: list snapshots).
 * enabled = 1 (default) uses it whenever the engine setup built its tables;
 * 0 forces the level-synchronous engine.  Applies from the next bfb_bfs. */
int bfb_set_small_engine(bfb_ctx* ctx, int enabled);
/* Sparse levels (top-down phase 1, also inside direction-optimizing runs; one
 * node, several nodes of one context, and rank mode): a level whose frontier
 * has few edges (at most max(|V|/64, 2^16), capped at 2^23) queues its
 * phase-1 claims and is exchanged and committed from that queue instead of by
 * sweeps over the whole visited bitmap.  With one node and top-down runs,
 * levels of at most 2^13 frontier edges run back to back in single-CTA
 * launches of up to 4096 levels.  enabled = 1 (default) / 0 (every level by
 * bitmap sweeps).  Results are identical either way. */
int bfb_set_sparse_levels(bfb_ctx* ctx, int enabled);
/* 1 if the next top-down bfb_bfs runs on the single-CTA engine. */
int bfb_small_engine_active(bfb_ctx* ctx);
/* Phase-1 direction (paper contribution 3; SPEC.md:172 keeps
 * the slot): 0 = top-down (Alg. 2, default), 1 = direction-optimizing with
 * Beamer's switch (TD->BU when frontier edges > unexplored edges / alpha,
 * BU->TD when frontier < |V| / beta; defaults alpha 14, beta 64, tuned on
 * Kronecker s29 ef8 and s24 ef16 -- Beamer's CPU values are 14 and 24), 2 = bottom-up at every
 * level (testing).
 * Levels, frontier sizes and traversed edges are identical in all modes (the
 * exchange volumes differ: bottom-up discoveries are owned vertices only).
 * Applies from the next bfb_bfs. */
int bfb_set_direction(bfb_ctx* ctx, int mode, double alpha, double beta);
/* Device-side bracket timer on the context's stream: start records a CUDA
 * event, stop records another, synchronizes and returns the elapsed ms. */
int bfb_timer_start(bfb_ctx* ctx);
int bfb_timer_stop(bfb_ctx* ctx, double* elapsed_ms_out);

/* ---- text ingestion and the CSR cache (graphs.py:96-209) ----------------- */
/* load_edge_list's line parsing on device: `data` (host, len bytes) is copied
 * to HBM and split into lines (newline 0: universal newlines \n, \r\n, \r as
 * for a path source; 1: \n only, as an io.StringIO source iterates), each
 * line tokenised and its ids parsed with Python int() rules.  fmt 0 "edges": 'src dst' lines, '#'/'%'
 * comments.  fmt 1 "mtx": the coordinate entries of a Matrix Market file
 * (the caller has read the header and size line; `data` starts after them,
 * line numbers continue from first_line_no, rows/cols bound the entries).
 * The parsed edges stay in ctx for bfb_graph_from_parsed / bfb_parsed_edges.
 * A malformed line returns BFB_ERR_PARSE with result->err_* set. */
int bfb_parse_text(bfb_ctx* ctx, const char* data, int64_t len, int fmt, int newline,
                   int64_t first_line_no, int64_t rows, int64_t cols, bfb_parse_result* result);
/* Copy the parsed edges out: 2 * num_edges uint32 (src, dst pairs). */
int bfb_parsed_edges(bfb_ctx* ctx, uint32_t* edges_out);
/* CSR from the parsed edges without leaving the device: symmetrize = 1 is
 * build_csr(symmetrize(el)) (graphs.py:218-251), 0 is build_csr(el). */
int bfb_graph_from_parsed(bfb_ctx* ctx, int64_t num_vertices, int symmetrize);
/* write_edge_list (graphs.py:205-209): 'u v\n' lines, byte-identical. */
int bfb_write_edge_list(const char* path, const uint32_t* edges, int64_t num_edges);
/* Binary CSR cache of the resident graph ("BFBCSR01", n, m, offsets, adjacency):
 * save after a build, load instead of re-generating / re-parsing. */
int bfb_graph_save(bfb_ctx* ctx, const char* path);
int bfb_graph_load(bfb_ctx* ctx, const char* path);

/* ---- graph-core on device (graphs.py) ------------------------------------ */
/* generate_rmat (graphs.py:254-285): raw edges to a HOST buffer of 2*m uint32
 * (m = edge_factor << scale).  pcg_state/pcg_inc = numpy PCG64 initial state of
 * default_rng(seed) as {hi, lo}; thresholds = ceil(p * 2^53) for
 * (p_bottom, p_right_top, p_right_bottom) of graphs.py:273-275. */
int bfb_rmat_edges(bfb_ctx* ctx, int scale, int64_t edge_factor, const uint64_t pcg_state[2],
                   const uint64_t pcg_inc[2], const uint64_t thresholds[3], uint32_t* edges_out);
/* generate_rmat -> symmetrize -> build_csr fused on device; the CSR stays
 * resident in ctx (replaces graphs.py:218-251 for synthetic inputs). */
int bfb_graph_from_rmat(bfb_ctx* ctx, int scale, int64_t edge_factor,
                        const uint64_t pcg_state[2], const uint64_t pcg_inc[2],
                        const uint64_t thresholds[3]);
/* symmetrize (graphs.py:218-230) when `symmetrize` != 0, else build_csr's
 * validation (graphs.py:238-247) of an already symmetrized list.  Edges are
 * 2*m uint32 host values (src, dst) pairs; the CSR stays resident in ctx. */
int bfb_graph_from_edges(bfb_ctx* ctx, int64_t num_vertices, const uint32_t* edges, int64_t m,
                         int symmetrize);
/* One rank's share of the generate_rmat -> symmetrize -> build_csr graph
 * (SURVEY §8 e: GPU g owns offsets[b[g]..b[g+1]] and that adjacency slice):
 * the context keeps the whole offsets (every vertex's degree) and only the
 * adjacency of rows [b[rank], b[rank+1]) of partition_1d(num_parts) of the
 * final graph, whose num_parts+1 boundaries go to boundaries_out.  Rows are
 * built slice by slice under a bounded edge budget (the generator re-runs
 * per slice), so a rank never holds the whole edge set.  Such a context runs
 * bfb_rank_setup for that rank; whole-graph calls (CSR / edge copies, save,
 * bfb_engine_setup, certificates) return BFB_ERR_STATE. */
int bfb_graph_from_rmat_part(bfb_ctx* ctx, int scale, int64_t edge_factor,
                             const uint64_t pcg_state[2], const uint64_t pcg_inc[2],
                             const uint64_t thresholds[3], int num_parts, int rank,
                             int64_t* boundaries_out);
/* Rows whose adjacency this context holds ([0, n) unless partitioned) and
 * the number of adjacency entries resident. */
int bfb_graph_rows(bfb_ctx* ctx, int64_t* row_lo_out, int64_t* row_hi_out,
                   int64_t* adjacency_entries_out);
/* Upload an existing CSR (reference Graph, graphs.py:53-64). */
int bfb_graph_load_csr(bfb_ctx* ctx, int64_t num_vertices, int64_t num_edges,
                       const int64_t* offsets, const uint32_t* adjacency);
int bfb_graph_info(bfb_ctx* ctx, int64_t* num_vertices_out, int64_t* num_edges_out,
                   int64_t* max_degree_out);
/* D2H of the resident CSR (offsets n+1 int64, adjacency m uint32); either may be NULL. */
int bfb_graph_copy_csr(bfb_ctx* ctx, int64_t* offsets_out, uint32_t* adjacency_out);
/* D2H of the resident graph as the sorted, deduplicated (src, dst) list (2*m uint32). */
int bfb_graph_copy_edges(bfb_ctx* ctx, uint32_t* edges_out);
/* partition_1d (graphs.py:288-305) on the resident CSR: num_parts+1 int64. */
int bfb_partition_1d(bfb_ctx* ctx, int num_parts, int64_t* boundaries_out);
/* Number of vertices with degree > 0, and the vertices at the given ranks among
 * them (ascending id order): device form of flatnonzero(degrees > 0)[ranks]. */
int bfb_count_nonisolated(bfb_ctx* ctx, int64_t* count_out);
int bfb_select_nonisolated(bfb_ctx* ctx, const int64_t* ranks, int64_t k, int64_t* vertices_out);

/* ---- engine ------------------------------------------- */
/* init's allocation step: CN = num_parts nodes over the
 * resident graph with the given partition (num_parts+1 boundaries), all
 * per-node buffers allocated once here (no allocation inside bfb_bfs). */
int bfb_engine_setup(bfb_ctx* ctx, int num_parts, const int64_t* boundaries, int fanout,
                     int strategy, int want_parents);
/* run: one BFS from root.  levels_out (n uint32) and
 * parents_out (n int64, -1 unreached, root->root) are host buffers and may be
 * NULL (results stay on device).  frontier_sizes_out holds up to max_levels
 * entries (per_level_frontier_size); buffer_high_water_out holds num_parts
 * entries (may be NULL). */
int bfb_bfs(bfb_ctx* ctx, int64_t root, uint32_t* levels_out, int64_t* parents_out,
            int64_t* frontier_sizes_out, int64_t max_levels, int64_t* buffer_high_water_out,
            bfb_run_stats* stats_out);
/* per_level_frontier_size of the last run (all levels; bfb_bfs's array may be
 * capped by max_levels): writes min(cap, levels) entries, *len_out = levels. */
int bfb_frontier_sizes(bfb_ctx* ctx, int64_t* out, int64_t cap, int64_t* len_out);
/* D2H of the last run's results (node 0's view). */
int bfb_copy_levels(bfb_ctx* ctx, uint32_t* levels_out);
int bfb_copy_parents(bfb_ctx* ctx, int64_t* parents_out);
/* Device-side certificate of the last run's levels and
 * parents: *errors_out = bitmask (1 root, 2 reachability mismatch on an edge,
 * 4 edge spans >1 level, 8 reached vertex without predecessor, 16 bad parent). */
int bfb_validate(bfb_ctx* ctx, int64_t root, int64_t* errors_out);
/* The same certificate for caller-supplied results (host arrays: n uint32
 * levels, and n int64 parents with -1 = none, or NULL): checks any levels /
 * parents against the resident graph -- the verify command's device check
 * and the certificate's own negative tests.  Allocates its device copies. */
int bfb_validate_host(bfb_ctx* ctx, int64_t root, const uint32_t* levels, const int64_t* parents,
                      int64_t* errors_out);

/* Measurement helper (bench.py roofline, not part of the reference API): the
 * random-probe ceiling of phase 1 -- random 4-byte loads over a `bytes`-sized
 * device buffer (the visited bitmap's size).  *probes_out loads took *ms_out. */
int bfb_probe_peak(bfb_ctx* ctx, int64_t bytes, int64_t* probes_out, double* ms_out);

/* ---- multi-process mode: one process per GPU (torchrun), node = rank -----
 * The host driver (paper_2103_13577_b200/dist.py) sequences one level as
 * expand -> for each butterfly round: publish, [barrier + snapshot-size
 * allgather], merge -> commit.  Peers' round snapshots are read in place from
 * their HBM through CUDA IPC mappings (NVLink peer loads), fused with the OR
 * merge; the reference's CopyFrontier(Q_global[srcCN]) without
 * a staging copy. */
/* init's allocation step for node `rank` only (global partition boundaries). */
int bfb_rank_setup(bfb_ctx* ctx, int num_parts, const int64_t* boundaries, int fanout,
                   int strategy, int want_parents, int rank);
/* 320 bytes: the IPC handles of this node's two (round-parity) snapshot
 * bitmaps, its mailbox and its queue-form snapshots (device-synchronised
 * mode), and its parents (zero without parents). */
int bfb_rank_ipc_handles(bfb_ctx* ctx, void* handles_out);
int bfb_rank_open_peer(bfb_ctx* ctx, int peer, const void* handles);
int bfb_rank_begin(bfb_ctx* ctx, int64_t root);
int bfb_rank_expand(bfb_ctx* ctx);
/* Snapshot this node's q_global_next (round start); returns its size. */
int bfb_rank_publish(bfb_ctx* ctx, int parity, int64_t* count_out);
/* Merge the given sources' snapshots (sizes from the allgather; empty skipped). */
int bfb_rank_merge(bfb_ctx* ctx, int parity, const int32_t* sources, const int64_t* counts,
                   int num_sources);
/* Commit the level; returns the synchronized frontier size (0 = terminate)
 * and this node's owned share of it (|q_local|; sums to the frontier). */
int bfb_rank_commit(bfb_ctx* ctx, int64_t* frontier_out, int64_t* owned_out);
/* End of run: device elapsed time and this node's counters. */
int bfb_rank_finish(bfb_ctx* ctx, bfb_run_stats* stats_out);
/* This node's phase-1 parents (uint32, 0xFFFFFFFF = none): min over nodes is
 * a valid parent array. */
/* One whole BFS for this node with device-side synchronisation: per round,
 * publish -> signal {seq, snapshot size} into every peer's mailbox (NVLink
 * stores, release) -> spin on this node's mailbox (acquire) -> merge the
 * sources' snapshots in place.  No host round trip inside a level; the host
 * reads the frontier count once per level.  Every rank calls it with the same
 * root.  sizes_out[0..max_levels) = per_level_frontier_size; stats_out as
 * bfb_rank_finish plus this node's exchange accounting.  Honours
 * bfb_set_direction (each node applies Beamer's rule to its own rows). */
int bfb_rank_bfs(bfb_ctx* ctx, int64_t root, int64_t* sizes_out, int64_t max_levels,
                 bfb_run_stats* stats_out);
/* Output parents of the last BFS (int64, -1 unreached, root -> root): min over
 * every node's phase-1 parents, read from the peers' HBM (IPC mappings); call
 * after all ranks finished the BFS. */
int bfb_rank_parents(bfb_ctx* ctx, int64_t* parents_out);
int bfb_rank_parents_raw(bfb_ctx* ctx, uint32_t* parents_out);

#ifdef __cplusplus
}
#endif
#endif /* BFLYBFS_H_ */
