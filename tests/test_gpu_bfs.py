"""engine.run on B200 vs the oracle: levels bit-exact, RunStats identical to
the lockstep oracle engine, parents valid; SPEC.md acceptance criteria 1,3,4,
7,8 through the C ABI; full-size properties at scale 24."""

import numpy as np
import pytest

from oracle import bfs as ob
from oracle import engine as oe
from oracle import schedule as osch
from oracle import validate as ov
from paper_2103_13577_b200 import engine, graphs
from tests import util
from tests.util import sha16

pytestmark = pytest.mark.gpu
U = 0xFFFFFFFF


def _g(off, adj):
    return graphs.Graph(off.size - 1, adj.size, off.copy(), adj.copy())


def _same_stats(st, ost):
    return (st.per_level_frontier_size == ost.per_level_frontier_size
            and st.levels == ost.levels
            and st.remote_messages == ost.remote_messages
            and st.remote_vertices_transferred == ost.remote_vertices_transferred
            and st.rounds_executed == ost.rounds_executed
            and st.buffer_high_water == ost.buffer_high_water
            and st.traversed_edges == ost.traversed_edges)


def test_spec_examples():
    off, adj = util.path_graph(3)
    g = _g(off, adj)
    d, st = engine.run(g, graphs.partition_1d(g, 1), 0)
    assert d.d.tolist() == [0, 1, 2] and d.root == 0
    off, adj = util.csr_of_undirected(4, [(0, 1), (2, 3)])
    g = _g(off, adj)
    assert engine.run(g, graphs.partition_1d(g, 1), 0)[0].d.tolist() == [0, 1, U, U]
    off, adj = util.star_graph(5)
    g = _g(off, adj)
    assert engine.run(g, graphs.partition_1d(g, 1), 0)[1].per_level_frontier_size == [1, 5]
    off, adj = util.path_graph(5)
    g = _g(off, adj)
    d, st = engine.run(g, graphs.partition_1d(g, 2), 0, engine.EngineConfig(fanout=1))
    assert d.d.tolist() == [0, 1, 2, 3, 4] and st.levels == 5


def test_errors():
    off, adj = util.path_graph(6)
    g = _g(off, adj)
    p = graphs.partition_1d(g, 2)
    with pytest.raises(ValueError):
        engine.run(g, p, 6)
    with pytest.raises(ValueError):
        engine.run(g, p, -1)
    with pytest.raises(ValueError):
        engine.run(g, p, 0, engine.EngineConfig(fanout=3))
    with pytest.raises(ValueError):
        engine.run(g, graphs.Partition(2, [0, 3, 5]), 0)
    with pytest.raises(ValueError):
        engine.EngineConfig(strategy="ring")


def test_golden_levels_s16(golden):
    e = golden["s16_ef8"]
    g = graphs.kronecker(16, 8, 1)
    p = graphs.partition_1d(g, 1)
    for r, want in e["bfs"].items():
        d, st = engine.run(g, p, int(r), engine.EngineConfig(parents=True))
        assert sha16(d.d) == want["levels_sha"], r
        assert st.per_level_frontier_size == want["sizes"]
        assert st.traversed_edges == want["traversed_edges"]
        assert g.device.validate(int(r)) == 0
        assert not ov.check_parents(g.offsets, g.adjacency, int(r), d.d, d.parents)


def test_golden_levels_s20(golden):
    e = golden["s20_ef8"]
    g = graphs.kronecker(20, 8, 1)
    for P, f in ((1, 1), (4, 2), (8, 8)):
        p = graphs.partition_1d(g, P)
        for r, want in list(e["bfs"].items())[:4]:
            d, st = engine.run(g, p, int(r), engine.EngineConfig(fanout=f))
            assert sha16(d.d) == want["levels_sha"], (P, f, r)
            assert st.per_level_frontier_size == want["sizes"]


def _sweep_graphs():
    yield "rmat13", util.rmat_graph(13)
    yield "gnp", util.gnp_graph(5000, 0.002)
    yield "path", util.path_graph(1500)
    yield "star", util.star_graph(300)
    yield "components", util.components_graph()


@pytest.mark.parametrize("small", [True, False], ids=["single-cta", "level-sync"])
@pytest.mark.parametrize("cn", [1, 2, 3, 4, 7, 8, 9, 12, 16])
def test_acceptance_sweep_vs_oracle_engine(cn, small):
    """Acceptance 1,3,4,7,8 at reduced root counts: levels
    equal bfs_top_down, RunStats equal the lockstep oracle engine's for both
    strategies, buffer high-water within f*|V|, rounds = levels*num_rounds.
    Both engines: the single-CTA one these small graphs get by default and
    the level-synchronous one (forced)."""
    rng = np.random.default_rng(100 + cn)
    for name, (off, adj) in _sweep_graphs():
        n = off.size - 1
        g = _g(off, adj)
        graphs.device_graph(g).set_small_engine(small)
        p = graphs.partition_1d(g, cn)
        roots = rng.choice(n, 3, replace=False)
        for f in sorted({1, min(2, cn), min(4, cn), cn}):
            for r in roots:
                r = int(r)
                ref = ob.bfs_top_down(off, adj, r)
                for strat in ("butterfly", "all2all"):
                    d, st = engine.run(g, p, r, engine.EngineConfig(fanout=f, strategy=strat,
                                                                  parents=True))
                    assert np.array_equal(d.d, ref), (name, cn, f, r, strat)
                    assert graphs.device_graph(g).small_engine_active == small
                    _, ost = oe.run(off, adj, p.boundaries, r, fanout=f, strategy=strat)
                    assert _same_stats(st, ost), (name, cn, f, r, strat, st, ost)
                    assert max(st.buffer_high_water) <= f * n or strat == "all2all"
                    if strat == "butterfly":
                        assert st.rounds_executed == st.levels * osch.num_rounds(cn, f)
                    assert not ov.check_parents(off, adj, r, d.d, d.parents)


@pytest.mark.parametrize("direction", ["optimizing", "bottom-up"])
@pytest.mark.parametrize("cn", [1, 3, 8])
def test_direction_optimizing_identical_results(direction, cn):
    """Bottom-up / direction-optimizing phase 1: levels, frontier
    sizes, rounds and traversed edges identical to the top-down oracle engine
    (the exchange volumes differ: bottom-up discoveries are owned vertices)."""
    rng = np.random.default_rng(7 + cn)
    for name, (off, adj) in _sweep_graphs():
        n = off.size - 1
        g = _g(off, adj)
        p = graphs.partition_1d(g, cn)
        for r in rng.choice(n, 2, replace=False):
            r = int(r)
            f = min(2, cn)
            d, st = engine.run(g, p, r, engine.EngineConfig(fanout=f, parents=True,
                                                          direction=direction))
            assert np.array_equal(d.d, ob.bfs_top_down(off, adj, r)), (name, cn, direction, r)
            _, ost = oe.run(off, adj, p.boundaries, r, fanout=f)
            assert st.per_level_frontier_size == ost.per_level_frontier_size
            assert (st.levels, st.rounds_executed, st.traversed_edges) == \
                (ost.levels, ost.rounds_executed, ost.traversed_edges), (name, cn, direction, r)
            assert max(st.buffer_high_water) <= f * n
            assert not ov.check_parents(off, adj, r, d.d, d.parents)
            if direction == "bottom-up" and st.levels > 1:
                assert st.bottom_up_levels == st.levels


def test_direction_optimizing_switches_on_kronecker(golden):
    e = golden["s16_ef8"]
    g = graphs.kronecker(16, 8, 1)
    p = graphs.partition_1d(g, 1)
    for r, want in e["bfs"].items():
        d, st = engine.run(g, p, int(r), engine.EngineConfig(direction="optimizing", parents=True))
        assert sha16(d.d) == want["levels_sha"]
        assert st.traversed_edges == want["traversed_edges"]
        if len(want["sizes"]) > 3:
            assert st.bottom_up_levels >= 1 and st.edges_examined < st.traversed_edges


def test_all2all_message_reduction_cn16():
    off, adj = util.gnp_graph(3000, 0.01)
    g = _g(off, adj)
    p = graphs.partition_1d(g, 16)
    da, sa = engine.run(g, p, 0, engine.EngineConfig(strategy="all2all"))
    d1, s1 = engine.run(g, p, 0, engine.EngineConfig(fanout=1))
    d4, s4 = engine.run(g, p, 0, engine.EngineConfig(fanout=4))
    assert np.array_equal(da.d, d1.d) and np.array_equal(da.d, d4.d)
    assert sa.remote_messages >= 240 > 0
    assert s1.remote_messages <= 64 * s1.levels and s4.remote_messages <= 96 * s4.levels


def test_isolated_root_and_determinism():
    g = graphs.kronecker(14, 8, 1)
    off = g.offsets
    iso = int(np.flatnonzero(np.diff(off) == 0)[0])
    p = graphs.partition_1d(g, 4)
    d, st = engine.run(g, p, iso, engine.EngineConfig(fanout=2))
    assert st.per_level_frontier_size == [1] and (d.d != U).sum() == 1
    a, _ = engine.run(g, p, 3, engine.EngineConfig(fanout=2))
    b, _ = engine.run(g, p, 3, engine.EngineConfig(fanout=2))
    assert np.array_equal(a.d, b.d)


def test_reference_graph_objects(reference_objects):
    """The drop-in (SURVEY §8 b): engine.run on the reference's Graph /
    Partition objects (graphs.py:53-93), 3 nodes, fanout 2; levels equal the
    independent scipy BFS of the fixture and the oracle."""
    rg, rp, levels, _ = reference_objects("s12_ef8_seed3")
    for r, want in levels.items():
        for cfg in (engine.EngineConfig(fanout=2, parents=True),
                    engine.EngineConfig(fanout=1, strategy="all2all"),
                    engine.EngineConfig(fanout=3, direction="optimizing")):
            d, st = engine.run(rg, rp, r, cfg)
            assert np.array_equal(d.d, want), (r, cfg)
            assert np.array_equal(d.d, ob.bfs_top_down(rg.offsets, rg.adjacency, r))
            assert st.per_level_frontier_size == ob.level_sizes(want)
            if cfg.parents:
                assert not ov.check_parents(rg.offsets, rg.adjacency, r, d.d, d.parents)


@pytest.mark.slow
def test_scale24_full_size_properties():
    """Full-size (s24 ef16) checks without a CPU BFS: device certificate
    (SPEC.md:130-132 + parent validity), run-to-run determinism, CN=1 vs CN=4
    agreement, and frontier sizes summing to the reached count."""
    g = graphs.kronecker(24, 16, 1)
    dg = g.device
    roots = graphs.sample_roots(g, 3)
    dg.setup(dg.partition_1d(1), 1, "butterfly", parents=True)
    ref = {}
    for r in roots:
        lv, _, sizes, st, _ = dg.bfs(int(r))
        assert dg.validate(int(r)) == 0
        assert sum(sizes) == st.reached == int((lv != U).sum())
        ref[int(r)] = sha16(lv)
        lv2, _, _, _, _ = dg.bfs(int(r))
        assert sha16(lv2) == ref[int(r)]
    dg.setup(dg.partition_1d(4), 2, "butterfly", parents=True)
    for r in roots:
        lv, _, _, _, _ = dg.bfs(int(r))
        assert sha16(lv) == ref[int(r)]
        assert dg.validate(int(r)) == 0


@pytest.mark.slow
def test_scale24_golden(golden):
    e = golden.get("s24_ef16")
    if e is None:
        pytest.skip("s24 golden not generated")
    g = graphs.kronecker(24, 16, 1)
    assert g.num_edges == e["num_edges"]
    dg = g.device
    off, adj = dg.csr()
    assert sha16(off) == e["offsets_sha"] and sha16(adj) == e["adjacency_sha"]
    assert dg.partition_1d(8).tolist() == e["partitions"]["8"]
    dg.setup(dg.partition_1d(1), 1, "butterfly")
    for r, want in e["bfs"].items():
        lv, _, sizes, st, _ = dg.bfs(int(r))
        assert sha16(lv) == want["levels_sha"] and sizes == want["sizes"]


@pytest.mark.slow
def test_config3_s27_ef16_butterfly_parts():
    """BASELINE config 3 at full size (Kronecker s27 ef16, fanout 2) with 2,
    4 and 8 butterfly nodes as parts of one GPU: levels identical to the
    single-node run, device certificate, rounds = levels x ceil(log2 CN), and
    the per-round incoming snapshot within the f * |V| bound."""
    g = graphs.kronecker(27, 16, 1)
    dg = g.device
    r = int(graphs.sample_roots(g, 1)[0])
    dg.setup(dg.partition_1d(1), 1, "butterfly", parents=True)
    ref, _, sizes, _, _ = dg.bfs(r)
    assert dg.validate(r) == 0
    want = sha16(ref)
    del ref
    for cn in (2, 4, 8):
        dg.setup(dg.partition_1d(cn), 2, "butterfly", parents=True)
        lv, _, s2, st, hw = dg.bfs(r)
        assert sha16(lv) == want and s2 == sizes
        assert dg.validate(r) == 0
        assert st.rounds_executed == len(sizes) * {2: 1, 4: 2, 8: 3}[cn]
        assert max(hw) <= 2 * g.num_vertices


@pytest.mark.slow
def test_config4_s28_ef8_fanout_sweep():
    """BASELINE config 4 at full size (Kronecker s28 ef8, 8 nodes) on one GPU
    (8 parts): fanout 2/4/8 give the same levels and frontier sizes, rounds
    per level 3/2/1, and fanout 8 (all-to-all) moves CN*(CN-1) transfers per
    non-trivial level at most."""
    g = graphs.kronecker(28, 8, 1)
    dg = g.device
    r = int(graphs.sample_roots(g, 1)[0])
    b = dg.partition_1d(8)
    ref = None
    for f, rounds in ((2, 3), (4, 2), (8, 1)):
        dg.setup(b, f, "butterfly")
        lv, _, sizes, st, _ = dg.bfs(r)
        key = (sha16(lv), tuple(sizes))
        ref = ref or key
        assert key == ref, f
        assert st.rounds_executed == len(sizes) * rounds
        assert st.remote_messages <= len(sizes) * 8 * 7
        assert dg.validate(r) == 0


@pytest.mark.parametrize("small", [True, False], ids=["single-cta", "level-sync"])
@pytest.mark.parametrize("cn", [1, 3])
def test_deep_graph_levels_past_the_level_bitmaps(cn, small):
    """Levels 0..31 are materialised from per-level bitmaps at termination,
    deeper ones written directly (kLevelBits = 32): a 300-vertex path plus a
    cycle and an isolated vertex, from both ends and the middle, all parts,
    parents on, in every phase-1 direction."""
    edges = [(i, i + 1) for i in range(299)] + [(300, 301), (301, 302), (302, 300)]
    off, adj = util.csr_of_undirected(304, edges)
    g = _g(off, adj)
    graphs.device_graph(g).set_small_engine(small)
    p = graphs.partition_1d(g, cn)
    for direction in ("top-down", "optimizing", "bottom-up"):
        for root in (0, 150, 299, 301, 303):
            cfg = engine.EngineConfig(fanout=1, parents=True, direction=direction)
            d, st = engine.run(g, p, root, cfg)
            ref = ob.bfs_top_down(off, adj, root)
            assert np.array_equal(d.d, ref), (cn, direction, root)
            assert not ov.check_parents(off, adj, root, d.d, d.parents)
            assert st.per_level_frontier_size == ob.level_sizes(ref)


@pytest.mark.parametrize("small", [True, False], ids=["single-cta", "level-sync"])
@pytest.mark.parametrize("direction", ["top-down", "optimizing"])
def test_tiny_and_ragged_graphs(direction, small):
    """Edge cases of the bitmap/word layout: a single vertex, one edge, a
    vertex count that is not a multiple of 32 (star centred on the last
    vertex, padded words), and 32 isolated vertices plus one edge at the end."""
    cases = [(1, []), (2, [(0, 1)]), (33, [(32, i) for i in range(32)]),
             (65, [(63, 64)]), (1025, [(i, i + 1) for i in range(1000, 1024)])]
    for n, edges in cases:
        off, adj = util.csr_of_undirected(n, edges)
        g = _g(off, adj)
        graphs.device_graph(g).set_small_engine(small)
        for cn in sorted({1, min(2, n), min(3, n)}):
            p = graphs.partition_1d(g, cn)
            for root in sorted({0, n - 1, n // 2}):
                cfg = engine.EngineConfig(fanout=1, parents=True, direction=direction)
                d, st = engine.run(g, p, root, cfg)
                ref = ob.bfs_top_down(off, adj, root)
                assert np.array_equal(d.d, ref), (n, cn, root)
                assert not ov.check_parents(off, adj, root, d.d, d.parents)
                assert st.per_level_frontier_size == ob.level_sizes(ref)


@pytest.mark.slow
def test_config5_s29_ef8_headline_properties():
    """BASELINE config 5 (the headline graph, Kronecker s29 ef8) at full size on
    one GPU: for three Graph500 roots the device certificate (SPEC.md:130-132 +
    parent validity) holds for top-down and direction-optimizing runs, both
    give identical levels (sha) and frontier sizes, and the sizes add up to
    the reached count."""
    g = graphs.kronecker(29, 8, 1)
    dg = g.device
    assert g.num_vertices == 1 << 29 and dg.max_degree > 0
    dg.setup(dg.partition_1d(1), 1, "butterfly", parents=True)
    for r in graphs.sample_roots(g, 3):
        out = {}
        for direction in ("top-down", "optimizing"):
            dg.set_direction(direction)
            lv, _, sizes, st, _ = dg.bfs(int(r))
            assert dg.validate(int(r)) == 0, direction
            assert sum(sizes) == st.reached == int((lv != U).sum())
            out[direction] = (sha16(lv), tuple(sizes), st.traversed_edges)
            del lv
        assert out["top-down"] == out["optimizing"], int(r)
    dg.set_direction("top-down")


@pytest.mark.parametrize("parents", [False, True])
def test_sparse_levels_identical(golden, parents):
    """One node, top-down: levels whose frontier has few edges queue their
    phase-1 claims and are committed from that queue (no sweep over the
    bitmaps; d_local written directly).  Levels, frontier sizes and traversed
    edges equal the golden files and the sweep-committed run; parents valid;
    the device certificate holds."""
    e = golden["s20_ef8"]
    g = graphs.kronecker(20, 8, 1)
    dg = g.device
    dg.setup(dg.partition_1d(1), 1, "butterfly", parents=parents)
    for r, want in list(e["bfs"].items())[:3]:
        r = int(r)
        out = {}
        for sparse in (True, False):
            dg.set_sparse_levels(sparse)
            lv, pa, sizes, st, _ = dg.bfs(r, parents=parents)
            assert (st.sparse_levels > 0) == sparse, (r, sparse, st.sparse_levels)
            assert sha16(lv) == want["levels_sha"] and sizes == want["sizes"], (r, sparse)
            assert dg.validate(r) == 0
            if parents:
                assert not ov.check_parents(g.offsets, g.adjacency, r, lv, pa)
            out[sparse] = st.traversed_edges
        assert out[True] == out[False]
    dg.set_sparse_levels(True)


def test_sparse_levels_deep_path():
    """A 40,000-vertex path (above the single-CTA engine's size) from its
    middle: every level is sparse, levels past kLevelBits are written directly
    too; equal to the oracle, parents valid."""
    off, adj = util.path_graph(40000)
    g = _g(off, adj)
    p = graphs.partition_1d(g, 1)
    for root in (0, 20000, 39999):
        d, st = engine.run(g, p, root, engine.EngineConfig(parents=True))
        ref = ob.bfs_top_down(off, adj, root)
        assert np.array_equal(d.d, ref), root
        assert not ov.check_parents(off, adj, root, d.d, d.parents)
        assert st.per_level_frontier_size == ob.level_sizes(ref)


def test_thin_levels_in_one_launch():
    """Thin levels (frontier edges <= 2^13; one node, top-down) run back to
    back inside single-CTA launches of up to 4096 levels, continuing from and
    handing back to the level-synchronous passes: a 200,000-vertex path from
    one end (49 launches), and a Kronecker s16 graph with a 5,000-vertex tail
    attached to vertex 0 (dense levels, then the thin tail).  Levels, sizes,
    traversed edges equal the oracle; parents valid; with the thin-level and
    sparse paths switched off the results are the same."""
    off, adj = util.path_graph(200000)
    g = _g(off, adj)
    p = graphs.partition_1d(g, 1)
    d, st = engine.run(g, p, 0, engine.EngineConfig(parents=True))
    ref = ob.bfs_top_down(off, adj, 0)
    assert np.array_equal(d.d, ref) and st.levels == 200000
    assert st.sparse_levels >= 199999
    assert not ov.check_parents(off, adj, 0, d.d, d.parents)
    # Kronecker core + a tail
    koff, kadj = util.rmat_graph(16)
    n0 = koff.size - 1
    src = np.repeat(np.arange(n0, dtype=np.int64), np.diff(koff))
    pairs = np.stack([src, kadj.astype(np.int64)], 1)
    pairs = pairs[pairs[:, 0] < pairs[:, 1]]
    tail = [(0, n0)] + [(n0 + i, n0 + i + 1) for i in range(4999)]
    off2, adj2 = util.csr_of_undirected(n0 + 5000, np.concatenate([pairs, np.asarray(tail)]))
    g2 = _g(off2, adj2)
    p2 = graphs.partition_1d(g2, 1)
    dg = graphs.device_graph(g2)
    for root in (1, n0 + 4999):
        ref = ob.bfs_top_down(off2, adj2, root)
        for sparse in (True, False):
            dg.set_sparse_levels(sparse)
            d, st = engine.run(g2, p2, root, engine.EngineConfig(parents=True))
            assert np.array_equal(d.d, ref), (root, sparse)
            assert st.per_level_frontier_size == ob.level_sizes(ref)
            assert st.traversed_edges == int(np.diff(off2)[ref != U].sum())
            assert not ov.check_parents(off2, adj2, root, d.d, d.parents)
    dg.set_sparse_levels(True)
