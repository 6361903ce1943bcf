"""Text ingestion on device (graphs.py:96-209 restated as csrc/ingest.cu):
every golden case of tests/golden/parse_golden.json (made by the reference's
own load_edge_list / write_edge_list) -- edges, num_vertices, or the exact
ParseError line and message -- from a path and from a text stream; the
device text -> CSR path and the binary CSR cache."""

import base64
import hashlib
import io
import json
import os

import numpy as np
import pytest

from oracle import graphs as og
from paper_2103_13577_b200 import graphs
from tests import util

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "parse_golden.json")
CASES = json.load(open(GOLDEN))["cases"]


@pytest.mark.parametrize("case", CASES, ids=[f"{c['fmt']}-{c['name']}" for c in CASES])
def test_golden_path_source(case, tmp_path):
    path = tmp_path / case["name"]
    path.write_bytes(base64.b64decode(case["data_b64"]))
    if "error" in case:
        with pytest.raises(graphs.ParseError) as ei:
            graphs.load_edge_list(str(path), case["fmt"])
        assert str(ei.value) == case["error"]
        assert ei.value.line_no == case["line_no"]
        assert isinstance(ei.value, ValueError)
        return
    el = graphs.load_edge_list(str(path), case["fmt"])
    assert el.num_vertices == case["num_vertices"]
    assert el.num_edges == case["num_edges"]
    assert util.sha16(el.edges) == case["edges_sha"]
    out = tmp_path / (case["name"] + ".out")
    graphs.write_edge_list(el, str(out))
    assert hashlib.sha256(out.read_bytes()).hexdigest()[:16] == case["written_sha"]


STREAM = [c for c in CASES if "stream" in c]


@pytest.mark.parametrize("case", STREAM, ids=[f"{c['fmt']}-{c['name']}" for c in STREAM])
def test_golden_text_stream_source(case):
    src = io.StringIO(base64.b64decode(case["data_b64"]).decode("ascii"))
    want = case["stream"]
    if "error" in want:
        with pytest.raises(graphs.ParseError) as ei:
            graphs.load_edge_list(src, case["fmt"])
        assert str(ei.value) == want["error"]
        return
    el = graphs.load_edge_list(src, case["fmt"])
    assert el.num_vertices == want["num_vertices"]
    assert util.sha16(el.edges) == want["edges_sha"]


def test_binary_stream_and_unknown_format():
    el = graphs.load_edge_list(io.BytesIO(b"0 1\r2 3\n"))
    assert el.edges.tolist() == [[0, 1], [2, 3]]
    with pytest.raises(ValueError):
        graphs.load_edge_list(io.BytesIO(b"0 1\n"), "csv")


def test_rmat_text_roundtrip_and_device_csr(tmp_path):
    # s14 RMAT edges -> text -> device parse == the edges; text -> device CSR
    # == oracle build_csr(symmetrize(...)) == the device Kronecker build
    el = graphs.generate_rmat(14, 8, 1)
    path = tmp_path / "s14.txt"
    graphs.write_edge_list(el, str(path))
    back = graphs.load_edge_list(str(path))
    assert np.array_equal(back.edges, el.edges)
    assert back.num_vertices == int(el.edges.max()) + 1
    g = graphs.load_graph(str(path))
    n = back.num_vertices
    off, adj = og.build_csr(og.symmetrize(el.edges, n), n)
    assert np.array_equal(g.offsets, off) and np.array_equal(g.adjacency, adj)
    k = graphs.kronecker(14, 8, 1)
    assert np.array_equal(k.adjacency, adj)


def test_mtx_to_device_csr(tmp_path):
    path = tmp_path / "m.mtx"
    path.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n% c\n5 5 4\n"
                    "1 2\n2 3\n3 1\n5 4\n")
    g = graphs.load_graph(str(path), "mtx")
    assert g.num_vertices == 5
    assert g.offsets.tolist() == [0, 2, 4, 6, 7, 8]
    assert g.adjacency.tolist() == [1, 2, 0, 2, 0, 1, 4, 3]


def test_csr_cache_roundtrip(tmp_path):
    g = graphs.kronecker(12, 8, 1)
    path = tmp_path / "g.bfbcsr"
    graphs.save_csr(g, str(path))
    h = graphs.load_csr(str(path))
    assert h.num_vertices == g.num_vertices and h.num_edges == g.num_edges
    assert np.array_equal(h.offsets, g.offsets) and np.array_equal(h.adjacency, g.adjacency)
    bad = tmp_path / "bad.bfbcsr"
    bad.write_bytes(b"not a graph")
    with pytest.raises(OSError):
        graphs.load_csr(str(bad))
    with pytest.raises(OSError):
        graphs.load_csr(str(tmp_path / "missing.bfbcsr"))
