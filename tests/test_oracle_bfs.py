"""bfs-oracle and engine-oracle checks:
SPEC examples, golden levels (independent scipy BFS in make_golden.py), and
the acceptance sweeps at CPU-friendly sizes."""

import numpy as np
import pytest

from oracle import bfs as ob
from oracle import engine as oe
from oracle import graphs as og
from oracle import validate as ov
from tests import util

U = 0xFFFFFFFF


def test_spec_examples():
    off, adj = util.path_graph(3)
    assert ob.bfs_top_down(off, adj, 0).tolist() == [0, 1, 2]
    off, adj = util.csr_of_undirected(4, [(0, 1), (2, 3)])
    assert ob.bfs_top_down(off, adj, 0).tolist() == [0, 1, U, U]
    off, adj = util.star_graph(5)
    assert ob.frontier_sizes(off, adj, 0) == [1, 5]
    off, adj = util.path_graph(4)
    assert ob.frontier_sizes(off, adj, 0) == [1, 1, 1, 1]
    with pytest.raises(ValueError):
        ob.bfs_top_down(off, adj, 4)


def test_naive_bfs_gnp():
    # random G(200, 0.03) vs an independent naive queue BFS
    off, adj = util.gnp_graph(200, 0.03)
    d = ob.bfs_top_down(off, adj, 5)
    ref = np.full(200, U, dtype=np.uint32)
    ref[5] = 0
    q = [5]
    while q:
        v = q.pop(0)
        for u in adj[off[v]:off[v + 1]]:
            if ref[u] == U:
                ref[u] = ref[v] + 1
                q.append(int(u))
    assert np.array_equal(d, ref)
    assert not ov.check_levels(off, adj, 5, d)


def test_golden_levels(golden):
    for key in ("s12_ef8", "s16_ef8"):
        e = golden[key]
        off, adj = util.rmat_graph(e["scale"], e["edge_factor"], e["seed"])
        for r, want in e["bfs"].items():
            d = ob.bfs_top_down(off, adj, int(r))
            assert util.sha16(d) == want["levels_sha"], (key, r)
            assert ob.level_sizes(d) == want["sizes"]
            assert ob.traversed_edges(off, d) == want["traversed_edges"]


def test_c_oracle_golden_levels(golden):
    # the C/OpenMP restatement (bench.py's CPU baseline) against the same
    # golden levels, on 1 thread and on all host threads
    from oracle import cbfs

    for key in ("s12_ef8", "s16_ef8"):
        e = golden[key]
        off, adj = util.rmat_graph(e["scale"], e["edge_factor"], e["seed"])
        for r, want in e["bfs"].items():
            for threads in (1, 0):
                d = cbfs.bfs_top_down(off, adj, int(r), threads=threads)
                assert util.sha16(d) == want["levels_sha"], (key, r, threads)
    off, adj = util.path_graph(3)
    assert cbfs.bfs_top_down(off, adj, 0).tolist() == [0, 1, 2]
    off, adj = util.csr_of_undirected(4, [(0, 1), (2, 3)])
    assert cbfs.bfs_top_down(off, adj, 0).tolist() == [0, 1, U, U]
    with pytest.raises(ValueError):
        cbfs.bfs_top_down(off, adj, 4)
    off, adj = util.rmat_graph(14)
    d, scanned, secs, done = cbfs.bfs_top_down(off, adj, 0, time_budget_s=60)
    assert done and scanned == ob.traversed_edges(off, d)


def test_time_budget_sample():
    off, adj = util.rmat_graph(14)
    d, scanned, secs, done = ob.bfs_top_down(off, adj, 0, time_budget_s=60)
    assert done and scanned == ob.traversed_edges(off, d)


def test_validators_catch_errors():
    off, adj = util.rmat_graph(10)
    d = ob.bfs_top_down(off, adj, 0)
    assert not ov.check_levels(off, adj, 0, d)
    bad = d.copy()
    v = int(np.flatnonzero(d == 2)[0])
    bad[v] = 3
    assert ov.check_levels(off, adj, 0, bad)
    # parents from the levels: smallest neighbour one level up
    par = np.full(d.size, -1, dtype=np.int64)
    par[0] = 0
    for x in np.flatnonzero((d != U) & (np.arange(d.size) != 0)):
        nb = adj[off[x]:off[x + 1]]
        par[x] = int(nb[d[nb] == d[x] - 1].min())
    assert not ov.check_parents(off, adj, 0, d, par)
    par2 = par.copy()
    par2[v] = v
    assert ov.check_parents(off, adj, 0, d, par2)


# ---- engine oracle: acceptance criteria 1, 3, 4, 7, 8 ----

def _graphs():
    yield "rmat12", util.rmat_graph(12)
    yield "gnp", util.gnp_graph(1500, 0.004)
    yield "path", util.path_graph(300)
    yield "star", util.star_graph(50)
    yield "components", util.components_graph()


@pytest.mark.parametrize("cn", [1, 2, 3, 4, 7, 8, 9, 12, 16])
def test_engine_oracle_equivalence_sweep(cn):
    rng = np.random.default_rng(cn)
    for name, (off, adj) in _graphs():
        n = off.size - 1
        if cn > n:
            continue
        b = og.partition_1d(off, cn)
        roots = rng.choice(n, 3, replace=False)
        for f in sorted({1, min(2, cn), min(4, cn), cn}):
            for r in roots:
                ref = ob.bfs_top_down(off, adj, int(r))
                d, st = oe.run(off, adj, b, int(r), fanout=f, check_agreement=True)
                assert np.array_equal(d, ref), (name, cn, f, r)
                assert st.frontier_agreement
                assert st.per_level_frontier_size == ob.level_sizes(ref)
                assert max(st.buffer_high_water) <= f * n  # buffer bound
                from oracle import schedule as osch

                assert st.rounds_executed == st.levels * osch.num_rounds(cn, f)
                assert st.traversed_edges == ob.traversed_edges(off, ref)


def test_engine_spec_examples():
    off, adj = util.path_graph(5)
    b = og.partition_1d(off, 2)
    d, st = oe.run(off, adj, b, 0, fanout=1)
    assert d.tolist() == [0, 1, 2, 3, 4] and st.levels == 5
    with pytest.raises(ValueError):
        oe.run(off, adj, b, 7)
    with pytest.raises(ValueError):
        oe.run(off, adj, b, 0, fanout=3)


def test_strategy_equivalence_and_message_reduction():
    # acceptance 7: CN=16 all2all = 240 transfers per level (when all sources
    # are non-empty) vs <= 64 (f=1) / <= 96 (f=4) for the butterfly.
    off, adj = util.gnp_graph(3000, 0.01)
    b = og.partition_1d(off, 16)
    da, sa = oe.run(off, adj, b, 0, strategy="all2all", fanout=1)
    d1, s1 = oe.run(off, adj, b, 0, fanout=1)
    d4, s4 = oe.run(off, adj, b, 0, fanout=4)
    assert np.array_equal(da, d1) and np.array_equal(da, d4)
    assert sa.per_level_frontier_size == s1.per_level_frontier_size == s4.per_level_frontier_size
    assert sa.remote_messages <= 240 * sa.levels
    assert s1.remote_messages <= 64 * s1.levels
    assert s4.remote_messages <= 96 * s4.levels
    assert sa.remote_messages > s4.remote_messages > 0
    # at least one level where every node had discoveries: exactly 240 there
    assert sa.remote_messages >= 240
