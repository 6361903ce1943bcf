"""Lockstep ButterFly BFS engine restated from SPEC.md:267-367 / Alg. 2
(PAPER.md:279-374).  TEST INFRASTRUCTURE ONLY.

CN simulated nodes, each with a full-length distance view ``d_local`` and
pre-allocated append-only queues.  Phase 1 traverses the
owned frontier; phase 2 runs the butterfly rounds pulling
round-start snapshots of the scheduled sources' ``q_global_next``
(SPEC.md:307-315,347), skipping empty sources.  Node 0's view
is returned.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import schedule as sched_mod

UNREACHED = np.uint32(0xFFFFFFFF)


@dataclass
class OracleStats:
    """Mirror of RunStats."""

    levels: int = 0
    per_level_frontier_size: list = field(default_factory=list)
    remote_messages: int = 0
    remote_vertices_transferred: int = 0
    rounds_executed: int = 0
    buffer_high_water: list = field(default_factory=list)
    traversed_edges: int = 0
    frontier_agreement: bool = True


class _Node:
    def __init__(self, g, lo, hi, n):
        self.g, self.lo, self.hi = g, lo, hi
        self.d = np.full(n, UNREACHED, dtype=np.uint32)
        # Pre-allocated to |V| each: no growth during a run.
        self.q_local = np.empty(n, dtype=np.int64)
        self.n_local = 0
        self.q_local_next = np.empty(n, dtype=np.int64)
        self.n_local_next = 0
        self.q_global_next = np.empty(n, dtype=np.int64)
        self.n_global_next = 0

    def claim(self, cand, level):
        """Check-and-set on d_local for a batch of candidates in arrival order:
        first arrival of each undiscovered vertex wins."""
        cand = cand[self.d[cand] == UNREACHED]
        if cand.size == 0:
            return
        _, first = np.unique(cand, return_index=True)
        new = cand[np.sort(first)]
        self.d[new] = level + 1
        k = new.size
        self.q_global_next[self.n_global_next:self.n_global_next + k] = new
        self.n_global_next += k
        own = new[(new >= self.lo) & (new < self.hi)]
        self.q_local_next[self.n_local_next:self.n_local_next + own.size] = own
        self.n_local_next += own.size


def run(offsets, adjacency, boundaries, root, fanout=1, strategy="butterfly",
        check_agreement=False):
    """SPEC.md:316-324.  Returns (d uint32[n] of node 0, OracleStats)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    boundaries = np.asarray(boundaries, dtype=np.int64)
    n = offsets.size - 1
    cn = boundaries.size - 1
    if not (0 <= int(root) < n):
        raise ValueError(f"root {root} out of range [0, {n})")
    if boundaries[0] != 0 or boundaries[-1] != n or np.any(np.diff(boundaries) < 0):
        raise ValueError("partition does not match graph")
    if strategy == "butterfly":
        schedule = sched_mod.make_schedule(cn, fanout)
    elif strategy == "all2all":
        sched_mod.make_schedule(cn, fanout)  # same fanout validation
        schedule = sched_mod.all_to_all_schedule(cn)
    else:
        raise ValueError(f"unknown strategy {strategy!r}")

    nodes = [_Node(g, int(boundaries[g]), int(boundaries[g + 1]), n) for g in range(cn)]
    for nd in nodes:  # init
        nd.d[root] = 0
        if nd.lo <= root < nd.hi:
            nd.q_local[0] = root
            nd.n_local = 1
    stats = OracleStats(buffer_high_water=[0] * cn)
    deg = np.diff(offsets)
    level = 0
    frontier_size = 1
    while frontier_size:
        stats.per_level_frontier_size.append(frontier_size)
        # Phase 1
        for nd in nodes:
            nd.n_global_next = 0
            nd.n_local_next = 0
            q = nd.q_local[:nd.n_local]
            if q.size == 0:
                continue
            stats.traversed_edges += int(deg[q].sum())
            starts = offsets[q]
            dq = deg[q]
            tot = int(dq.sum())
            if tot:
                pos = np.repeat(starts - (np.cumsum(dq) - dq), dq) + np.arange(tot, dtype=np.int64)
                nd.claim(adjacency[pos].astype(np.int64), level)
        # Phase 2
        for rnd in schedule:
            snap = [nd.n_global_next for nd in nodes]  # round-start snapshot
            for nd, srcs in zip(nodes, rnd):
                incoming = 0
                for s in srcs:
                    k = snap[s]
                    if k == 0:
                        continue  # empty-buffer suppression
                    stats.remote_messages += 1
                    stats.remote_vertices_transferred += k
                    incoming += k
                    nd.claim(nodes[s].q_global_next[:k], level)
                stats.buffer_high_water[nd.g] = max(stats.buffer_high_water[nd.g], incoming)
            stats.rounds_executed += 1
        if check_agreement:
            ref = set(nodes[0].q_global_next[:nodes[0].n_global_next].tolist())
            for nd in nodes[1:]:
                if set(nd.q_global_next[:nd.n_global_next].tolist()) != ref:
                    stats.frontier_agreement = False
        # swap queues; termination on node 0
        for nd in nodes:
            nd.q_local, nd.q_local_next = nd.q_local_next, nd.q_local
            nd.n_local = nd.n_local_next
        frontier_size = nodes[0].n_global_next
        level += 1
    stats.levels = len(stats.per_level_frontier_size)
    return nodes[0].d.copy(), stats
