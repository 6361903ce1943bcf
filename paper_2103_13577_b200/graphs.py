"""Graph-core API of the reference (pkg/src/bflybfs/graphs.py), device-backed.

Same names, argument meaning and exceptions as the reference module; the
generator, symmetrize, CSR build and partition run as sm_100a kernels
(include/bflybfs.h).  Text ingestion (graphs.py:96-209) tokenises
and parses the file on device (csrc/ingest.cu); ``load_graph`` goes from text
to a device-resident CSR without the edges visiting the host, and
``save_csr`` / ``load_csr`` keep a binary CSR cache.
"""

from __future__ import annotations

import math

import numpy as np

from .device import DeviceGraph

VID = np.uint32                      # graphs.py:13
MAX_VID = int(np.iinfo(VID).max)     # graphs.py:14
UNREACHED = MAX_VID                  # graphs.py:17
RMAT_PROBS = (0.57, 0.19, 0.19, 0.05)  # graphs.py:21


class ParseError(ValueError):
    """Malformed graph input; carries the 1-based line number (graphs.py:24-29)."""

    def __init__(self, message, line_no):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


class EdgeList:
    """Directed (m, 2) edge pairs plus the vertex count (graphs.py:32-50)."""

    def __init__(self, edges, num_vertices):
        e = np.asarray(edges, dtype=VID).reshape(-1, 2)
        if e.size and int(e.max()) >= num_vertices:
            raise ValueError("edge endpoint exceeds num_vertices")
        self.edges = e
        self.num_vertices = int(num_vertices)

    @property
    def num_edges(self):
        return len(self.edges)

    def __repr__(self):
        return f"EdgeList(num_vertices={self.num_vertices}, num_edges={self.num_edges})"


class Graph:
    """Immutable CSR graph (graphs.py:53-75).

    ``offsets`` / ``adjacency`` are read-only numpy arrays.  A graph built on
    device keeps its ``DeviceGraph`` in ``device`` and copies the host arrays
    lazily on first access, so a scale-29 graph never has to visit the host.
    """

    def __init__(self, num_vertices, num_edges, offsets=None, adjacency=None, device=None):
        self.num_vertices = int(num_vertices)
        self.num_edges = int(num_edges)
        self.device = device
        self._offsets = offsets
        self._adjacency = adjacency
        for a in (offsets, adjacency):
            if a is not None:
                a.flags.writeable = False

    @classmethod
    def from_device(cls, dg):
        return cls(dg.num_vertices, dg.num_edges, device=dg)

    @property
    def offsets(self):
        if self._offsets is None:
            self._offsets = self.device.offsets()
            self._offsets.flags.writeable = False
        return self._offsets

    @property
    def adjacency(self):
        if self._adjacency is None:
            self._adjacency = self.device.adjacency()
            self._adjacency.flags.writeable = False
        return self._adjacency

    def neighbors(self, v):
        return self.adjacency[self.offsets[v]:self.offsets[v + 1]]

    @property
    def degrees(self):
        return np.diff(self.offsets)

    @property
    def max_degree(self):
        if self.device is not None:
            return self.device.max_degree
        return int(self.degrees.max()) if self.num_vertices else 0

    def __repr__(self):
        return f"Graph(num_vertices={self.num_vertices}, num_edges={self.num_edges})"


class Partition:
    """Contiguous vertex ranges, one per compute node (graphs.py:78-93)."""

    def __init__(self, num_parts, boundaries):
        self.num_parts = int(num_parts)
        self.boundaries = np.asarray(boundaries, dtype=np.int64)

    def owner_of(self, v):
        return int(np.searchsorted(self.boundaries[1:], v, side="right"))

    def part_range(self, g):
        return int(self.boundaries[g]), int(self.boundaries[g + 1])

    def edge_counts(self, graph):
        return np.diff(graph.offsets[self.boundaries])

    def __repr__(self):
        return f"Partition(num_parts={self.num_parts}, boundaries={self.boundaries.tolist()})"


def rmat_device_args(scale, edge_factor, seed, probs=RMAT_PROBS):
    """Validate like graphs.py:261-267 and return the device generator's
    inputs: PCG64 state/inc of default_rng(seed) and the integer thresholds
    ceil(p * 2^53) of graphs.py:273-275 (U < p <=> (next64 >> 11) < that)."""
    if scale < 1 or edge_factor < 1:
        raise ValueError("scale and edge_factor must be >= 1")
    if (1 << scale) - 1 > MAX_VID:
        raise ValueError(f"scale {scale} overflows the vertex-id range")
    a, b, c, d = (float(x) for x in probs)
    if min(a, b, c, d) < 0 or abs(a + b + c + d - 1.0) > 1e-9:
        raise ValueError("quadrant probabilities must be non-negative and sum to 1")
    st = np.random.PCG64(seed).state["state"]
    from ._lib import u64_pair

    thr = np.array([math.ceil(p * 2.0 ** 53) for p in (c + d, b / (a + b), d / (c + d))],
                   dtype=np.uint64)
    return u64_pair(st["state"]), u64_pair(st["inc"]), thr


def generate_rmat(scale, edge_factor, seed, probs=RMAT_PROBS, device=0):
    """graphs.py:254-285 on device; bit-identical to the reference's stream."""
    import ctypes

    from . import _lib

    state, inc, thr = rmat_device_args(scale, edge_factor, seed, probs)
    m = int(edge_factor) << int(scale)
    out = np.empty((m, 2), dtype=VID)
    dg = DeviceGraph(device)
    try:
        _lib.check(_lib.load().bfb_rmat_edges(dg.handle, int(scale), int(edge_factor),
                                              _lib.ptr(state, ctypes.c_uint64),
                                              _lib.ptr(inc, ctypes.c_uint64),
                                              _lib.ptr(thr, ctypes.c_uint64),
                                              _lib.ptr(out, ctypes.c_uint32)))
    finally:
        dg.close()
    return EdgeList(out, 1 << int(scale))


def symmetrize(el, device=0):
    """graphs.py:218-230 on device: mirror, drop self-loops and duplicates,
    sort by (src, dst)."""
    if el.num_edges == 0 or el.num_vertices == 0:
        return EdgeList(np.empty((0, 2), dtype=VID), el.num_vertices)
    dg = DeviceGraph.from_edges(el.edges, el.num_vertices, symmetrize=True, device=device)
    try:
        return EdgeList(dg.edges(), el.num_vertices)
    finally:
        dg.close()


def build_csr(el, device=0):
    """graphs.py:233-251 on device, with the same symmetry validation
    (ValueError on self-edge / duplicate / missing reverse).  The returned
    Graph keeps its device copy for the engine."""
    dg = DeviceGraph.from_edges(el.edges, el.num_vertices, symmetrize=False, device=device)
    off, adj = dg.csr()
    return Graph(el.num_vertices, adj.size, off, adj, device=dg)


def kronecker_part(scale, edge_factor, seed, num_parts, rank, probs=RMAT_PROBS, device=0):
    """One rank's share of kronecker(...) for the multi-process engine
    (SURVEY §8 e): the Graph's offsets are whole, its device adjacency holds
    only the rows of part ``rank`` of partition_1d(num_parts) (so host
    ``adjacency`` is unavailable).  Returns (Graph, Partition)."""
    dg = DeviceGraph.from_rmat_part(scale, edge_factor, seed, num_parts, rank, probs, device)
    return Graph.from_device(dg), Partition(num_parts, dg.boundaries)


def kronecker(scale, edge_factor, seed, probs=RMAT_PROBS, device=0):
    """build_csr(symmetrize(generate_rmat(...))) entirely on device; the host
    arrays are only materialised if accessed."""
    return Graph.from_device(DeviceGraph.from_rmat(scale, edge_factor, seed, probs, device))


def device_graph(g, device=0):
    """The DeviceGraph behind ``g`` (a Graph of this package or the
    reference's own graphs.Graph), uploading it once and caching it."""
    dg = getattr(g, "device", None)
    if isinstance(dg, DeviceGraph):
        return dg
    key = id(g)
    hit = _UPLOADS.get(key)
    if hit is not None:
        ref_off, ref_adj, dg = hit
        if ref_off is g.offsets and ref_adj is g.adjacency:
            return dg
    dg = DeviceGraph.from_csr(g.offsets, g.adjacency, device=device)
    _UPLOADS.clear()  # keep at most one uploaded foreign graph resident
    _UPLOADS[key] = (g.offsets, g.adjacency, dg)
    return dg


_UPLOADS = {}


def partition_1d(g, num_parts):
    """graphs.py:288-305 (searchsorted of round-half-up targets) on device."""
    if num_parts < 1:
        raise ValueError("num_parts must be >= 1")
    if g.num_vertices and num_parts > g.num_vertices:
        raise ValueError("num_parts exceeds the number of vertices")
    return Partition(num_parts, device_graph(g).partition_1d(num_parts))


def sample_roots(g, count=64, seed=2103):
    """Benchmark roots: default_rng(seed).choice(flatnonzero(deg > 0), count,
    replace=False), with the non-isolated selection on device."""
    dg = device_graph(g)
    pop = dg.count_nonisolated()
    k = min(int(count), pop)
    ranks = np.random.default_rng(seed).choice(pop, k, replace=False)
    return dg.select_nonisolated(ranks)


# ------------------------------------------------------------ text ingestion --
_FMT = {"edges": 0, "mtx": 1}


def _source_bytes(source):
    """(bytes, decode, newline mode) for a path, a text stream or a binary
    stream, read the way the reference reads it (graphs.py:96-101): paths and
    binary streams as ASCII with errors replaced and universal newlines; a
    text stream line by line as it iterates itself (io.StringIO splits on
    "\n" only)."""
    import io
    from pathlib import Path

    ascii_ = lambda b: b.decode("ascii", errors="replace")  # noqa: E731
    if isinstance(source, (str, Path)):
        with open(source, "rb") as fh:
            return fh.read(), ascii_, 0
    if isinstance(source, io.TextIOBase):
        text = "".join(source)
        return text.encode("utf-8"), lambda b: b.decode("utf-8", errors="replace"), 1
    return source.read(), ascii_, 0


def _next_line(data, pos, nl=0):
    """The line starting at pos: (line bytes, next pos); nl = 0 universal
    newlines, 1 "\n" only."""
    n = len(data)
    i = pos
    stops = (10, 13) if nl == 0 else (10,)
    while i < n and data[i] not in stops:
        i += 1
    if i >= n:
        return data[pos:n], n
    return data[pos:i], i + (2 if data[i] == 13 and i + 1 < n and data[i + 1] == 10 else 1)


def _mtx_prologue(data, decode, nl=0):
    """Header and size line of a Matrix Market file, as graphs.py:138-164.
    Returns (entry offset, line number of the size line, rows, cols, nnz)."""
    header, pos = _next_line(data, 0, nl) if data else (b"", 0)
    tokens = decode(header).strip().lower().split()
    if len(tokens) < 4 or tokens[0] != "%%matrixmarket" or tokens[1] != "matrix" \
            or tokens[2] != "coordinate":
        raise ParseError("expected '%%MatrixMarket matrix coordinate' header", 1)
    line_no = 1
    while pos < len(data):
        line, pos = _next_line(data, pos, nl)
        line_no += 1
        stripped = decode(line).strip()
        if not stripped or stripped[0] == "%":
            continue
        parts = stripped.split()
        if len(parts) != 3:
            raise ParseError("expected 'rows cols nnz' size line", line_no)
        try:
            rows, cols, nnz = (int(p) for p in parts)
        except ValueError:
            raise ParseError("non-integer size line", line_no) from None
        return pos, line_no, rows, cols, nnz
    raise ParseError("missing size line", line_no + 1)


def _raise_line_error(res, data, decode, rows=0, cols=0):
    """The reference's ParseError for the first malformed line the device
    found (graphs.py:109-134, 165-180)."""
    stripped = decode(bytes(data[res.err_begin:res.err_end])).strip()
    parts = stripped.split()
    code, ln = res.err_code, res.err_line
    if code == 2:
        raise ParseError(f"expected 'src dst', got {stripped!r}", ln)
    if code == 3:
        raise ParseError(f"non-integer vertex id in {stripped!r}", ln)
    if code == 4:
        raise ParseError(f"negative vertex id in {stripped!r}", ln)
    if code in (5, 6):
        raise ParseError(f"vertex id {int(parts[code - 5])} exceeds the representable range", ln)
    if code == 7:
        raise ParseError(f"expected coordinate entry, got {stripped!r}", ln)
    if code == 8:
        raise ParseError(f"non-integer coordinate in {stripped!r}", ln)
    if code == 9:
        i, j = int(parts[0]), int(parts[1])
        raise ParseError(f"coordinate ({i}, {j}) outside {rows}x{cols}", ln)
    raise RuntimeError(f"unknown parse error code {code} at line {ln}")


def _parse_on_device(dg, source, fmt):
    """Parse ``source`` into dg's parsed-edge buffer; returns (num_edges,
    num_vertices) with the reference's validation and errors."""
    import ctypes

    from . import _lib

    if fmt not in _FMT:
        raise ValueError(f"unknown format {fmt!r}")
    data, decode, nl = _source_bytes(source)
    start, line0, rows, cols, nnz = 0, 0, 0, 0, None
    if fmt == "mtx":
        start, line0, rows, cols, nnz = _mtx_prologue(data, decode, nl)
    region = np.frombuffer(data, dtype=np.uint8)[start:]
    clamp = 1 << 40  # any entry above 2^32 is outside the VID range anyway
    res = _lib.ParseResultC()
    rc = _lib.load().bfb_parse_text(dg.handle, region.ctypes.data if region.size else None,
                                    int(region.size), _FMT[fmt], nl, int(line0),
                                    max(-1, min(int(rows), clamp)), max(-1, min(int(cols), clamp)),
                                    ctypes.byref(res))
    if rc == _lib.ERR_PARSE:
        _raise_line_error(res, region, decode, rows, cols)
    _lib.check(rc)
    m = int(res.num_edges)
    if fmt == "edges":
        return m, int(res.max_id_plus1)
    if m != nnz:
        raise ParseError(f"declared {nnz} entries, found {m}", line0 + int(res.num_lines) + 1)
    top = max(rows, cols)
    if top and top - 1 > MAX_VID:
        raise ParseError(f"vertex id {top - 1} exceeds the representable range", 1)
    return m, (top if top else 0)


def load_edge_list(source, fmt="edges", device=0):
    """graphs.py:185-202: directed edges from a path or stream ("edges": 'src
    dst' lines, '#'/'%' comments, 0-based; "mtx": Matrix Market coordinate
    pattern, 1-based ids shifted).  Tokenising and integer parsing run on
    device; same EdgeList, num_vertices and ParseError (line numbers and
    messages) as the reference."""
    import ctypes

    from . import _lib

    dg = DeviceGraph(device)
    try:
        m, n = _parse_on_device(dg, source, fmt)
        out = np.empty((m, 2), dtype=VID)
        _lib.check(_lib.load().bfb_parsed_edges(dg.handle, _lib.ptr(out, ctypes.c_uint32)))
    finally:
        dg.close()
    return EdgeList(out, n)


def load_graph(source, fmt="edges", device=0):
    """build_csr(symmetrize(load_edge_list(source, fmt))) with the edges never
    leaving the device: parse, mirror/dedup and CSR all in HBM."""
    from . import _lib

    dg = DeviceGraph(device)
    try:
        m, n = _parse_on_device(dg, source, fmt)
        _lib.check(_lib.load().bfb_graph_from_parsed(dg.handle, int(n), 1))
        dg._refresh()
    except BaseException:
        dg.close()
        raise
    return Graph.from_device(dg)


def write_edge_list(el, path):
    """graphs.py:205-209: 'src dst' text lines, byte-identical output."""
    import ctypes

    from . import _lib

    e = np.ascontiguousarray(el.edges, dtype=VID)
    _lib.check(_lib.load().bfb_write_edge_list(str(path).encode(), _lib.ptr(e, ctypes.c_uint32),
                                               int(e.shape[0])))


def save_csr(g, path):
    """Binary CSR cache of ``g`` ("BFBCSR01" header, n, m, offsets, adjacency)."""
    from . import _lib

    _lib.check(_lib.load().bfb_graph_save(device_graph(g).handle, str(path).encode()))


def load_csr(path, device=0):
    """A Graph from a save_csr cache, resident on ``device``."""
    from . import _lib

    dg = DeviceGraph(device)
    try:
        _lib.check(_lib.load().bfb_graph_load(dg.handle, str(path).encode()))
        dg._refresh()
    except BaseException:
        dg.close()
        raise
    return Graph.from_device(dg)
