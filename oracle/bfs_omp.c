/* Top-down BFS oracle in C + OpenMP -- TEST INFRASTRUCTURE ONLY (and the
 * timed CPU baseline of bench.py / --impl reference).
 *
 * Restates SPEC.md:136-163 / Alg. 1: level-synchronous
 * top-down BFS with two swapped queues and a check-and-set on
 * the distance array, here an atomic compare-and-swap so the
 * frontier loop runs on all host threads (the paper's OpenMP worker model,
 * PAPER.md:585).  BFS levels are unique, so the output equals the numpy
 * oracle (oracle/bfs.py) bit-exactly; tests/test_oracle_bfs.py checks it.
 *
 * Build: oracle/Makefile -> oracle/_build/libbfs_omp.so (gcc -O3 -fopenmp).
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define UNREACHED 0xFFFFFFFFu

static double now_s(void) { return omp_get_wtime(); }

/* Returns 0 on success, -1 on bad root, -2 on allocation failure.
 * levels: uint32[n] output.  budget_s > 0 stops the search once the budget
 * is crossed (checked every 256 frontier vertices): *scanned = edges examined,
 * *seconds = elapsed, *done = 1 iff the BFS completed.  nthreads <= 0: all. */
int ob_bfs_top_down(int64_t n, const int64_t *off, const uint32_t *adj, int64_t root,
                    uint32_t *levels, int nthreads, double budget_s, int64_t *scanned,
                    double *seconds, int *done) {
  if (root < 0 || root >= n) return -1;
  if (nthreads > 0) omp_set_num_threads(nthreads);
  uint32_t *cur = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  uint32_t *next = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  if (!cur || !next) {
    free(cur);
    free(next);
    return -2;
  }
  const double t0 = now_s();
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) levels[i] = UNREACHED;
  levels[root] = 0;
  cur[0] = (uint32_t)root;
  int64_t ncur = 1, total = 0;
  uint32_t level = 0;
  int stopped = 0;
  while (ncur > 0 && !stopped) {
    int64_t nnext = 0, lvl_edges = 0;
    const int64_t chunk = 1024;
#pragma omp parallel reduction(+ : lvl_edges)
    {
      /* per-thread staging buffer, flushed to the shared queue in blocks */
      uint32_t buf[4096];
      int nb = 0;
#pragma omp for schedule(dynamic, chunk)
      for (int64_t i = 0; i < ncur; ++i) {
        if (__atomic_load_n(&stopped, __ATOMIC_RELAXED)) continue;
        if (budget_s > 0 && (i & 255) == 0 && now_s() - t0 > budget_s)
          __atomic_store_n(&stopped, 1, __ATOMIC_RELAXED);
        const uint32_t v = cur[i];
        const int64_t b = off[v], e = off[(int64_t)v + 1];
        lvl_edges += e - b;
        for (int64_t j = b; j < e; ++j) {
          const uint32_t u = adj[j];
          uint32_t expect = UNREACHED;
          /* check-and-set */
          if (__atomic_load_n(&levels[u], __ATOMIC_RELAXED) == UNREACHED &&
              __atomic_compare_exchange_n(&levels[u], &expect, level + 1, 0, __ATOMIC_RELAXED,
                                          __ATOMIC_RELAXED)) {
            buf[nb++] = u;
            if (nb == 4096) {
              const int64_t at = __atomic_fetch_add(&nnext, nb, __ATOMIC_RELAXED);
              memcpy(next + at, buf, sizeof(uint32_t) * (size_t)nb);
              nb = 0;
            }
          }
        }
      }
      if (nb) {
        const int64_t at = __atomic_fetch_add(&nnext, nb, __ATOMIC_RELAXED);
        memcpy(next + at, buf, sizeof(uint32_t) * (size_t)nb);
      }
    }
    total += lvl_edges;
    uint32_t *t = cur;
    cur = next;
    next = t;
    ncur = nnext;
    ++level;
  }
  if (scanned) *scanned = total;
  if (seconds) *seconds = now_s() - t0;
  if (done) *done = !stopped || ncur == 0;
  free(cur);
  free(next);
  return 0;
}

int ob_max_threads(void) { return omp_get_max_threads(); }
