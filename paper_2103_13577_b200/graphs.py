"""Graph-core API of the reference (pkg/src/bflybfs/graphs.py), device-backed.

Same names, argument meaning and exceptions as the reference module; the
generator, symmetrize, CSR build and partition run as sm_100a kernels
(include/bflybfs.h).  Text ingestion (graphs.py:96-209) is outside the hot
path and is not provided.
"""

from __future__ import annotations

import math

import numpy as np

from .device import DeviceGraph

VID = np.uint32                      # graphs.py:13
MAX_VID = int(np.iinfo(VID).max)     # graphs.py:14
UNREACHED = MAX_VID                  # graphs.py:17
RMAT_PROBS = (0.57, 0.19, 0.19, 0.05)  # graphs.py:21


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
