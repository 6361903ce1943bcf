"""Pin the graph-core restatement (oracle/graphs.py) against the reference
graphs.py (live, where /root/reference exists) and the committed golden
hashes, plus the SPEC.md examples of the graph-core module."""

import numpy as np
import pytest

from oracle import graphs as og
from tests.util import sha16


def test_golden_hashes_s16(golden):
    e = golden["s16_ef8"]
    raw = og.generate_rmat(16, 8, 1)
    assert sha16(raw) == e["raw_sha"]
    assert raw[:4].tolist() == e["raw_first"]
    sym = og.symmetrize(raw, 1 << 16)
    off, adj = og.build_csr(sym, 1 << 16)
    assert adj.size == e["num_edges"]
    assert sha16(off) == e["offsets_sha"]
    assert sha16(adj) == e["adjacency_sha"]
    for P, b in e["partitions"].items():
        assert og.partition_1d(off, int(P)).tolist() == b
    assert og.sample_roots(off).tolist() == e["roots64"]


def test_golden_fixture_s10(s10):
    raw = og.generate_rmat(10, 8, 1)
    assert np.array_equal(raw, s10["raw"])
    off, adj = og.build_csr(og.symmetrize(raw, 1 << 10), 1 << 10)
    assert np.array_equal(off, s10["offsets"])
    assert np.array_equal(adj, s10["adjacency"])


@pytest.mark.parametrize("scale,ef,seed", [(3, 2, 7), (8, 4, 3), (12, 8, 1), (14, 8, 5)])
def test_against_live_reference(reference_graphs, scale, ef, seed):
    R = reference_graphs
    el = R.generate_rmat(scale, ef, seed)
    raw = og.generate_rmat(scale, ef, seed)
    assert np.array_equal(el.edges, raw)
    sym = R.symmetrize(el)
    osym = og.symmetrize(raw, el.num_vertices)
    assert np.array_equal(sym.edges, osym)
    g = R.build_csr(sym)
    off, adj = og.build_csr(osym, el.num_vertices)
    assert np.array_equal(g.offsets, off) and np.array_equal(g.adjacency, adj)
    for P in (1, 2, 3, 8):
        assert np.array_equal(R.partition_1d(g, P).boundaries, og.partition_1d(off, P))


def test_live_reference_errors(reference_graphs):
    R = reference_graphs
    for bad in ([(0, 0)], [(0, 1), (0, 1), (1, 0)], [(0, 1)]):
        el = R.EdgeList(np.array(bad, dtype=np.uint32), 3)
        with pytest.raises(ValueError) as e1:
            R.build_csr(el)
        with pytest.raises(ValueError) as e2:
            og.build_csr(el.edges, 3)
        assert str(e1.value) == str(e2.value)


def test_spec_examples_symmetrize_build_csr_partition():
    # SPEC.md:63-64
    assert og.symmetrize([(0, 1)], 2).tolist() == [[0, 1], [1, 0]]
    assert og.symmetrize([(0, 0), (0, 1), (0, 1)], 2).tolist() == [[0, 1], [1, 0]]
    # SPEC.md:72-73
    off, adj = og.build_csr([(0, 1), (1, 0)], 2)
    assert off.tolist() == [0, 1, 2] and adj.tolist() == [1, 0]
    tri = og.symmetrize([(0, 1), (1, 2), (2, 0)], 3)
    assert og.build_csr(tri, 3)[0].tolist() == [0, 2, 4, 6]
    # SPEC.md:90-91
    path = og.symmetrize([(0, 1), (1, 2), (2, 3)], 4)
    poff, _ = og.build_csr(path, 4)
    assert og.partition_1d(poff, 1).tolist() == [0, 4]
    assert og.partition_1d(poff, 2).tolist() == [0, 2, 4]
    with pytest.raises(ValueError):
        og.partition_1d(poff, 0)
    with pytest.raises(ValueError):
        og.partition_1d(poff, 5)


def test_symmetrize_bruteforce_and_idempotent():
    # SPEC.md:65,95-96
    rng = np.random.default_rng(0)
    e = rng.integers(0, 50, (1000, 2)).astype(np.uint32)
    want = sorted({(int(a), int(b)) for a, b in e if a != b} | {(int(b), int(a)) for a, b in e if a != b})
    got = og.symmetrize(e, 50)
    assert [tuple(x) for x in got.tolist()] == want
    assert np.array_equal(og.symmetrize(got, 50), got)
    off, adj = og.build_csr(got, 50)
    src = np.repeat(np.arange(50), np.diff(off))
    assert np.array_equal(np.stack([src, adj], 1), got)


def test_rmat_quadrant_frequencies_and_determinism():
    # SPEC.md:81-83
    a = og.generate_rmat(3, 2, 7)
    assert a.shape == (16, 2) and int(a.max()) < 8
    assert np.array_equal(a, og.generate_rmat(3, 2, 7))
    e = og.generate_rmat(12, 8, 1)
    top_s = e[:, 0] >> 11
    top_d = e[:, 1] >> 11
    q = np.bincount(top_s * 2 + top_d, minlength=4) / e.shape[0]
    assert np.allclose(q, og.DEFAULT_PROBS, atol=0.02)
    with pytest.raises(ValueError):
        og.generate_rmat(0, 8, 1)
    with pytest.raises(ValueError):
        og.generate_rmat(33, 1, 1)
    with pytest.raises(ValueError):
        og.generate_rmat(4, 1, 1, (0.5, 0.5, 0.5, -0.5))


def test_pcg_draw_layout():
    # draw (2k+j)*m + e is the src (j=0) / dst (j=1) uniform of bit iteration k
    scale, ef, seed = 6, 2, 11
    m = ef << scale
    raw = og.generate_rmat(scale, ef, seed)
    (pb, prt, prb), ints = og.rmat_thresholds()
    for e in (0, 5, m - 1):
        for k in (0, scale - 1):
            bit = scale - 1 - k
            us = og.pcg64_draw(seed, (2 * k) * m + e)
            ud = og.pcg64_draw(seed, (2 * k + 1) * m + e)
            sb = us < pb
            db = ud < (prb if sb else prt)
            assert ((int(raw[e, 0]) >> bit) & 1) == sb
            assert ((int(raw[e, 1]) >> bit) & 1) == db
    # integer thresholds == float compare for every representable 53-bit draw edge
    for p, t in zip((pb, prt, prb), ints):
        assert (t - 1) * 2.0 ** -53 < p <= t * 2.0 ** -53


def test_parse_golden_matches_live_reference(reference_graphs, tmp_path):
    # the committed parse fixtures still equal the reference's own parser
    import base64
    import json
    import os

    from tests.util import sha16

    cases = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                        "parse_golden.json")))["cases"]
    for c in cases:
        p = tmp_path / c["name"]
        p.write_bytes(base64.b64decode(c["data_b64"]))
        try:
            el = reference_graphs.load_edge_list(str(p), c["fmt"])
            assert "error" not in c, c["name"]
            assert sha16(el.edges) == c["edges_sha"] and el.num_vertices == c["num_vertices"]
        except reference_graphs.ParseError as e:
            assert str(e) == c["error"], c["name"]
