"""Butterfly schedule restated from SPEC.md:178-265 (TEST INFRASTRUCTURE ONLY).

Receive-oriented: ``rounds[i][g]`` is the ordered tuple of nodes g pulls from in
round i.  Radix r = 2 for fanout 1, else r = fanout.  In round
i, g's desired sources vary base-r digit i of g.  A desired source
s >= CN is redirected to its subgroup representative, the lowest id sharing s's
digits at positions >= i, i.e. ``s - s % r**i``; it is dropped when that is
>= CN or equals g.
"""

from __future__ import annotations


def _check(num_nodes, fanout):
    if num_nodes < 1:
        raise ValueError("num_nodes must be >= 1")
    if fanout < 1:
        raise ValueError("fanout must be >= 1")
    if fanout > num_nodes:
        raise ValueError("fanout exceeds num_nodes")


def radix(fanout):
    return 2 if fanout == 1 else fanout


def num_rounds(num_nodes, fanout):
    """ceil(log_r CN), 0 for CN = 1."""
    _check(num_nodes, fanout)
    r, k, span = radix(fanout), 0, 1
    while span < num_nodes:
        span *= r
        k += 1
    return k


def make_schedule(num_nodes, fanout):
    """SPEC.md:193-201.  Returns a list of rounds; each round is a list (index
    g) of tuples of source node ids."""
    nr = num_rounds(num_nodes, fanout)
    r = radix(fanout)
    rounds = []
    for i in range(nr):
        w = r ** i
        per_node = []
        for g in range(num_nodes):
            base = g - ((g // w) % r) * w  # g with digit i cleared
            srcs = []
            for digit in range(r):
                s = base + digit * w
                if s == g:
                    continue
                if s >= num_nodes:
                    s -= s % w  # subgroup representative
                    if s >= num_nodes or s == g:
                        continue
                srcs.append(s)
            per_node.append(tuple(srcs))
        rounds.append(per_node)
    return rounds


def message_count_paper(num_nodes, fanout):
    """CN * f * ceil(log_max(f,2) CN) -- the paper's accounting."""
    return num_nodes * fanout * num_rounds(num_nodes, fanout)


def message_count_remote(schedule):
    """Total scheduled cross-node transfers."""
    return sum(len(srcs) for rnd in schedule for srcs in rnd)


def buffer_bound(num_vertices, fanout):
    """f * |V| incoming capacity per node."""
    return fanout * num_vertices


def knows_closure(schedule, num_nodes):
    """Information-flow closure of SPEC.md:240: knows(g) grows by knows(src)
    per round, from round-start snapshots."""
    knows = [{g} for g in range(num_nodes)]
    for rnd in schedule:
        snap = [set(k) for k in knows]
        for g, srcs in enumerate(rnd):
            for s in srcs:
                knows[g] |= snap[s]
    return knows


def all_to_all_schedule(num_nodes):
    """The all2all strategy as one round pulling every peer."""
    if num_nodes <= 1:
        return []
    return [[tuple(s for s in range(num_nodes) if s != g) for g in range(num_nodes)]]
