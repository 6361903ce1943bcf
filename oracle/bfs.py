"""Top-down BFS oracle, restated from SPEC.md:122-176 / Alg. 1.
TEST INFRASTRUCTURE ONLY (and the timed CPU baseline of bench.py).

Level-synchronous with two swapped queues; the check-and-set of
SPEC.md:163 becomes "keep the first occurrence of each undiscovered neighbour"
in vectorised form, which yields the identical set per level.
"""

from __future__ import annotations

import time

import numpy as np

UNREACHED = np.uint32(0xFFFFFFFF)

# Edges gathered per vectorised chunk: bounds temporary memory (8 B per edge).
CHUNK_EDGES = 1 << 24


def _expand_chunks(offsets, frontier, chunk_edges=CHUNK_EDGES):
    """Yield (vertex_index_in_frontier, adjacency_positions) chunks covering all
    edges of ``frontier`` with about ``chunk_edges`` edges each."""
    starts = offsets[frontier]
    degs = offsets[frontier + 1] - starts
    cum = np.cumsum(degs)
    lo = 0
    while lo < frontier.size:
        base = cum[lo] - degs[lo]
        hi = int(np.searchsorted(cum, base + chunk_edges, side="right"))
        hi = max(hi, lo + 1)
        d = degs[lo:hi]
        tot = int(d.sum())
        if tot:
            seg_start = np.repeat(starts[lo:hi] - (np.cumsum(d) - d), d)
            pos = seg_start + np.arange(tot, dtype=np.int64)
            yield lo, hi, d, pos
        lo = hi


def bfs_top_down(offsets, adjacency, root, time_budget_s=None):
    """SPEC.md:136-144.  Returns uint32 distances (UNREACHED if no path).

    With ``time_budget_s`` the search stops after the first chunk that crosses
    the budget and returns (d, edges_scanned, seconds, completed) -- the bounded
    CPU-baseline sample of bench.py.  Without it returns d only."""
    offsets = np.asarray(offsets, dtype=np.int64)
    n = offsets.size - 1
    if not (0 <= int(root) < n):
        raise ValueError(f"root {root} out of range [0, {n})")
    d = np.full(n, UNREACHED, dtype=np.uint32)
    d[root] = 0
    frontier = np.array([root], dtype=np.int64)
    level = 0
    scanned = 0
    t0 = time.perf_counter()
    stopped = False
    while frontier.size and not stopped:
        found = []
        for lo, hi, degs, pos in _expand_chunks(offsets, frontier):
            nbrs = adjacency[pos]
            scanned += pos.size
            fresh = nbrs[d[nbrs] == UNREACHED]
            if fresh.size:
                fresh = np.unique(fresh)
                d[fresh] = level + 1  # check-and-set: set before the next chunk
                found.append(fresh.astype(np.int64))
            if time_budget_s is not None and time.perf_counter() - t0 > time_budget_s:
                stopped = True
                break
        frontier = np.concatenate(found) if found else np.empty(0, dtype=np.int64)
        level += 1
    if time_budget_s is None:
        return d
    return d, scanned, time.perf_counter() - t0, not stopped


def frontier_sizes(offsets, adjacency, root):
    """number of vertices at each distance."""
    d = bfs_top_down(offsets, adjacency, root)
    return level_sizes(d)


def level_sizes(d):
    reached = d[d != UNREACHED]
    if reached.size == 0:
        return []
    return np.bincount(reached.astype(np.int64)).tolist()


def traversed_edges(offsets, d):
    """SPEC RunStats.traversed_edges: sum of degrees of reached vertices."""
    offsets = np.asarray(offsets, dtype=np.int64)
    deg = np.diff(offsets)
    return int(deg[d != UNREACHED].sum())
