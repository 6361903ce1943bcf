"""Stand-ins for the reference's Graph / Partition objects on GPU boxes,
where /root/reference (and so the reference's own classes) is absent.

They restate only the data layout the drop-in boundary reads --
``Graph(num_vertices, num_edges, offsets, adjacency)`` with read-only arrays
(pkg/src/bflybfs/graphs.py:53-64) and ``Partition(num_parts, boundaries)``
(graphs.py:78-83) -- and are deliberately NOT this package's types, so
engine.run must take them through the same duck-typed path it takes the
reference's.  The arrays come from tests/golden/ref_objects.npz, written by
tests/golden/make_ref_objects.py from the reference's own graphs.py.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

FIXTURE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_objects.npz")


@dataclass
class Graph:
    num_vertices: int
    num_edges: int
    offsets: np.ndarray
    adjacency: np.ndarray

    def __post_init__(self):
        self.offsets.flags.writeable = False
        self.adjacency.flags.writeable = False


@dataclass(frozen=True)
class Partition:
    num_parts: int
    boundaries: np.ndarray


def load(name):
    """(Graph, Partition, {root: levels}) of fixture case ``name``."""
    z = np.load(FIXTURE)
    off = z[f"{name}_offsets"].copy()
    adj = z[f"{name}_adjacency"].copy()
    b = z[f"{name}_boundaries"].copy()
    levels = {int(r): z[f"{name}_levels_{int(r)}"] for r in z[f"{name}_roots"]}
    return Graph(off.size - 1, adj.size, off, adj), Partition(b.size - 1, b), levels
