"""Parity pinned at the exact BASELINE.json configurations and at the edges of
the device engine's layout (SURVEY §8 c/d):

* C1 as written: Kronecker s16 ef8, 2 simulated nodes, fanout 2, root 0 and
  the first sampled Graph500 root -- levels / sizes / traversed edges against
  the golden files (reference graphs.py + scipy BFS), RunStats against the
  lockstep oracle engine;
* the device certificate (SPEC.md:130-132 + parents) rejects corrupted
  levels and parents -- each error bit has a case;
* a star with 2^26 leaves: max degree 2^26 switches the commit's 32-vertex
  degree sums to 64 bits (kWide) -- the only graph family that reaches it;
* C5 (s29 ef8) with 2/4/8 butterfly nodes (fanout 2) as parts of one GPU, and
  against a COMPLETE CPU BFS (oracle/bfs_omp.c, all host threads) on the
  host copy of the same CSR -- the headline graph's levels are not only
  self-certified.
"""

import numpy as np
import pytest

from oracle import bfs as ob
from oracle import cbfs
from oracle import engine as oe
from oracle import validate as ov
from paper_2103_13577_b200 import engine, graphs
from paper_2103_13577_b200.device import DeviceGraph
from tests.util import sha16

pytestmark = pytest.mark.gpu
U = 0xFFFFFFFF


def test_config1_exact(golden):
    """BASELINE config 1: s16 ef8, fanout 2, 2 simulated nodes, single source
    (root 0 and roots64[0], each run separately)."""
    e = golden["s16_ef8"]
    g = graphs.kronecker(16, 8, 1)
    p = graphs.partition_1d(g, 2)
    assert p.boundaries.tolist() == e["partitions"]["2"] == [0, 10241, 65536]
    off, adj = g.offsets, g.adjacency
    for r in (0, e["roots64"][0]):
        want = e["bfs"][str(r)]
        for direction in ("top-down", "optimizing"):
            d, st = engine.run(g, p, r, engine.EngineConfig(fanout=2, parents=True,
                                                          direction=direction))
            assert sha16(d.d) == want["levels_sha"], (r, direction)
            assert st.per_level_frontier_size == want["sizes"]
            assert st.traversed_edges == want["traversed_edges"]
            assert not ov.check_parents(off, adj, r, d.d, d.parents)
            if direction == "top-down":
                _, ost = oe.run(off, adj, p.boundaries, r, fanout=2)
                assert (st.levels, st.remote_messages, st.remote_vertices_transferred,
                        st.rounds_executed, st.buffer_high_water) == \
                    (ost.levels, ost.remote_messages, ost.remote_vertices_transferred,
                     ost.rounds_executed, ost.buffer_high_water), r


def test_certificate_rejects_corruption():
    """bfb_validate_host: the certificate the s27-s29 tests rely on flags
    every kind of wrong answer (and accepts the right one)."""
    g = graphs.kronecker(12, 8, 1)
    dg = g.device
    off, adj = g.offsets, g.adjacency
    r = 0
    ref = ob.bfs_top_down(off, adj, r)
    dg.setup(dg.partition_1d(1), 1, "butterfly", parents=True)
    lv, pa, _, _, _ = dg.bfs(r, levels=True, parents=True)
    assert np.array_equal(lv, ref)
    assert dg.validate_levels(r, lv, pa) == 0
    assert dg.validate_levels(r, lv) == 0
    deep = int(np.flatnonzero(ref == ref[ref != U].max())[0])  # a deepest vertex
    mid = int(np.flatnonzero(ref == 2)[0])
    for vertex, value, bit in ((r, 1, 1),      # root not at level 0
                               (mid, U, 2),    # a reached vertex reported unreached
                               (mid, 4, 4)):   # an edge spanning more than one level
        bad = lv.copy()
        bad[vertex] = value
        assert dg.validate_levels(r, bad) & bit, bit
    # a deepest vertex moved one level up: it has no neighbour at its new
    # level - 1 (all its neighbours sit at L - 1 or L)
    bad = lv.copy()
    bad[deep] = ref[deep] - 1
    assert dg.validate_levels(r, bad) & 8
    # a whole level shifted by one: every vertex still spans <= 1 level with
    # its neighbours only if the shift is consistent -- moving level 2 to 3
    # leaves level-3 vertices without a level-2 predecessor
    bad = lv.copy(); bad[lv == 2] = 3
    assert dg.validate_levels(r, bad) & (4 | 8)
    # parents: not a neighbour, wrong level, unreached vertex with a parent,
    # root's parent not the root
    bp = pa.copy(); bp[mid] = r
    assert dg.validate_levels(r, lv, bp) & 16
    bp = pa.copy(); bp[mid] = mid
    assert dg.validate_levels(r, lv, bp) & 16
    bp = pa.copy(); bp[r] = -1
    assert dg.validate_levels(r, lv, bp) & 16
    unreached = np.flatnonzero(ref == U)
    if unreached.size:
        bp = pa.copy(); bp[int(unreached[0])] = r
        assert dg.validate_levels(r, lv, bp) & 16


def test_wide_degree_star():
    """Max degree 2^26: the commit's 32-vertex degree sums overflow 32 bits
    on the level that holds the hub (kWide build); from a leaf the hub is a
    newly committed vertex, from the hub the 2^26 leaves are."""
    leaves = 1 << 26
    n = leaves + 1
    edges = np.empty((leaves, 2), dtype=np.uint32)
    edges[:, 0] = 0
    edges[:, 1] = np.arange(1, n, dtype=np.uint32)
    dg = DeviceGraph.from_edges(edges, n, symmetrize=True)
    del edges
    assert dg.max_degree == leaves and dg.num_edges == 2 * leaves
    for cn, fanout in ((1, 1), (2, 2)):
        dg.setup(dg.partition_1d(cn), fanout, "butterfly", parents=True)
        for direction in ("top-down", "optimizing"):
            dg.set_direction(direction)
            for root, want_sizes in ((0, [1, leaves]), (12345, [1, 1, leaves - 1])):
                lv, pa, sizes, st, _ = dg.bfs(root, levels=True, parents=True)
                assert sizes == want_sizes, (cn, direction, root)
                assert st.traversed_edges == 2 * leaves
                assert lv[root] == 0
                if root == 0:
                    assert int((lv == 1).sum()) == leaves and (pa[1:] == 0).all()
                else:
                    assert lv[0] == 1 and pa[0] == root
                    others = np.ones(n, dtype=bool)
                    others[[0, root]] = False
                    assert (lv[others] == 2).all() and (pa[others] == 0).all()
                assert dg.validate(root) == 0
    dg.set_direction("top-down")


@pytest.mark.slow
def test_config5_s29_parts_and_complete_cpu_bfs():
    """BASELINE config 5 (Kronecker s29 ef8) on one GPU: 1, 2, 4 and 8
    butterfly nodes (fanout 2) give the same levels (sha), frontier sizes and
    traversed edges, each certified on device; and for two Graph500 roots the
    levels equal a complete top-down BFS by oracle/bfs_omp.c on the host copy
    of the device-built CSR (every host thread)."""
    g = graphs.kronecker(29, 8, 1)
    dg = g.device
    roots = [int(r) for r in graphs.sample_roots(g, 2)]
    ref = {}
    dg.setup(dg.partition_1d(1), 1, "butterfly", parents=True)
    for r in roots:
        lv, _, sizes, st, _ = dg.bfs(r)
        assert dg.validate(r) == 0
        ref[r] = (sha16(lv), tuple(sizes), st.traversed_edges)
        del lv
    for cn in (2, 4, 8):
        dg.setup(dg.partition_1d(cn), 2, "butterfly", parents=True)
        for r in roots:
            lv, _, sizes, st, hw = dg.bfs(r)
            assert (sha16(lv), tuple(sizes), st.traversed_edges) == ref[r], (cn, r)
            assert dg.validate(r) == 0
            assert st.rounds_executed == len(sizes) * {2: 1, 4: 2, 8: 3}[cn]
            assert max(hw) <= 2 * g.num_vertices
            del lv
    dg.setup(dg.partition_1d(1), 1, "butterfly")
    off, adj = dg.csr()
    for r in roots:
        cpu = cbfs.bfs_top_down(off, adj, r, threads=cbfs.max_threads())
        assert sha16(cpu) == ref[r][0], r
        assert tuple(ob.level_sizes(cpu)) == ref[r][1]
        del cpu
