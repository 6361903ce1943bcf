"""Device graph-core (generate_rmat / symmetrize / build_csr / partition_1d)
vs the oracle and the reference's golden hashes.  Bit-exact."""

import numpy as np
import pytest

from oracle import graphs as og
from paper_2103_13577_b200 import graphs
from tests.util import sha16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale,ef,seed", [(1, 1, 0), (3, 2, 7), (10, 8, 1), (12, 8, 1), (13, 3, 42)])
def test_generate_rmat_bit_exact(scale, ef, seed):
    el = graphs.generate_rmat(scale, ef, seed)
    assert el.num_vertices == 1 << scale
    assert np.array_equal(el.edges, og.generate_rmat(scale, ef, seed))


def test_generate_rmat_custom_probs_and_errors():
    probs = (0.45, 0.15, 0.15, 0.25)
    el = graphs.generate_rmat(9, 4, 3, probs)
    assert np.array_equal(el.edges, og.generate_rmat(9, 4, 3, probs))
    with pytest.raises(ValueError):
        graphs.generate_rmat(0, 1, 1)
    with pytest.raises(ValueError):
        graphs.generate_rmat(33, 1, 1)
    with pytest.raises(ValueError):
        graphs.generate_rmat(4, 2, 1, (0.5, 0.5, 0.1, -0.1))


def test_golden_s16(golden):
    e = golden["s16_ef8"]
    el = graphs.generate_rmat(16, 8, 1)
    assert sha16(el.edges) == e["raw_sha"]
    g = graphs.kronecker(16, 8, 1)
    assert g.num_edges == e["num_edges"]
    assert sha16(g.offsets) == e["offsets_sha"]
    assert sha16(g.adjacency) == e["adjacency_sha"]
    assert g.max_degree == e["max_degree"]
    for P, b in e["partitions"].items():
        assert graphs.partition_1d(g, int(P)).boundaries.tolist() == b
    assert graphs.sample_roots(g).tolist() == e["roots64"]
    assert g.device.count_nonisolated() == e["nonisolated"]


def test_golden_s20(golden):
    e = golden["s20_ef8"]
    g = graphs.kronecker(20, 8, 1)
    assert g.num_edges == e["num_edges"]
    assert sha16(g.offsets) == e["offsets_sha"]
    assert sha16(g.adjacency) == e["adjacency_sha"]
    for P in ("2", "4", "8", "16"):
        assert graphs.partition_1d(g, int(P)).boundaries.tolist() == e["partitions"][P]
    assert graphs.sample_roots(g).tolist() == e["roots64"]


def test_symmetrize_and_build_csr_paths(s10):
    el = graphs.generate_rmat(10, 8, 1)
    sym = graphs.symmetrize(el)
    assert np.array_equal(sym.edges, og.symmetrize(s10["raw"], 1 << 10))
    g = graphs.build_csr(sym)
    assert np.array_equal(g.offsets, s10["offsets"])
    assert np.array_equal(g.adjacency, s10["adjacency"])
    # SPEC.md:63-64,72-73
    assert graphs.symmetrize(graphs.EdgeList([(0, 1)], 2)).edges.tolist() == [[0, 1], [1, 0]]
    assert graphs.symmetrize(graphs.EdgeList([(0, 0), (0, 1), (0, 1)], 2)).edges.tolist() == [[0, 1], [1, 0]]
    g2 = graphs.build_csr(graphs.EdgeList([(0, 1), (1, 0)], 2))
    assert g2.offsets.tolist() == [0, 1, 2] and g2.adjacency.tolist() == [1, 0]


def test_symmetrize_random_vs_oracle_and_idempotent():
    rng = np.random.default_rng(1)
    for n, m in ((50, 1000), (1000, 20000), (7, 3)):
        e = rng.integers(0, n, (m, 2)).astype(np.uint32)
        sym = graphs.symmetrize(graphs.EdgeList(e, n))
        assert np.array_equal(sym.edges, og.symmetrize(e, n))
        assert np.array_equal(graphs.symmetrize(sym).edges, sym.edges)
        g = graphs.build_csr(sym)
        off, adj = og.build_csr(sym.edges, n)
        assert np.array_equal(g.offsets, off) and np.array_equal(g.adjacency, adj)


def test_empty_inputs():
    assert graphs.symmetrize(graphs.EdgeList(np.empty((0, 2)), 5)).num_edges == 0
    g = graphs.build_csr(graphs.EdgeList(np.empty((0, 2)), 4))
    assert g.offsets.tolist() == [0, 0, 0, 0, 0] and g.num_edges == 0
    assert graphs.partition_1d(g, 2).boundaries.tolist() == og.partition_1d(g.offsets, 2).tolist()


@pytest.mark.parametrize("bad,msg", [
    ([(0, 0), (1, 2), (2, 1)], "self-edge"),
    ([(0, 1), (0, 1), (1, 0)], "duplicate"),
    ([(0, 1)], "missing reverse"),
])
def test_build_csr_rejects_non_symmetric(bad, msg):
    with pytest.raises(ValueError, match=msg):
        graphs.build_csr(graphs.EdgeList(np.array(bad, dtype=np.uint32), 3))


def test_partition_errors_and_spec_example():
    g = graphs.build_csr(graphs.symmetrize(graphs.EdgeList([(0, 1), (1, 2), (2, 3)], 4)))
    assert graphs.partition_1d(g, 1).boundaries.tolist() == [0, 4]
    assert graphs.partition_1d(g, 2).boundaries.tolist() == [0, 2, 4]
    with pytest.raises(ValueError):
        graphs.partition_1d(g, 0)
    with pytest.raises(ValueError):
        graphs.partition_1d(g, 5)


def test_reference_graph_types_accepted(reference_objects):
    rg, rp, _, _ = reference_objects("s10_ef8_seed1")
    assert np.array_equal(graphs.partition_1d(rg, 4).boundaries, rp.boundaries)
    dg = graphs.device_graph(rg)
    off, adj = dg.csr()
    assert np.array_equal(off, rg.offsets) and np.array_equal(adj, rg.adjacency)
