"""Certificates for BFS outputs (TEST INFRASTRUCTURE ONLY).

``check_levels`` restates the DistanceArray invariants of SPEC.md:130-132;
together (root at 0, |d[u]-d[v]| <= 1 and reachability agreement on every
edge, a predecessor at d-1 for every reached non-root) they imply d is the
exact BFS distance, so they certify levels at scales where no CPU BFS runs.
``check_parents`` checks Graph500-style parent validity.
"""

from __future__ import annotations

import numpy as np

UNREACHED = 0xFFFFFFFF


def _edge_src(offsets):
    deg = np.diff(offsets)
    return np.repeat(np.arange(offsets.size - 1, dtype=np.int64), deg)


def check_levels(offsets, adjacency, root, d):
    offsets = np.asarray(offsets, dtype=np.int64)
    d = np.asarray(d, dtype=np.uint32)
    errs = []
    if d[root] != 0:
        errs.append("d[root] != 0")
    src = _edge_src(offsets)
    dst = np.asarray(adjacency).astype(np.int64)
    ds, dt = d[src].astype(np.int64), d[dst].astype(np.int64)
    rs, rt = ds != UNREACHED, dt != UNREACHED
    if np.any(rs != rt):
        errs.append("edge with exactly one reached endpoint")
    both = rs & rt
    if np.any(np.abs(ds[both] - dt[both]) > 1):
        errs.append("edge spans more than one level")
    # every reached v != root has a neighbour at d[v]-1
    pred = both & (ds == dt - 1)
    has_pred = np.zeros(d.size, dtype=bool)
    has_pred[dst[pred]] = True
    reached = np.flatnonzero(d != UNREACHED)
    reached = reached[reached != root]
    if reached.size and not has_pred[reached].all():
        errs.append("reached vertex without a predecessor")
    if np.any(d[d != UNREACHED] > d.size):
        errs.append("level out of range")
    return errs


def check_parents(offsets, adjacency, root, d, parents):
    offsets = np.asarray(offsets, dtype=np.int64)
    parents = np.asarray(parents, dtype=np.int64)
    d = np.asarray(d, dtype=np.uint32)
    errs = []
    if parents[root] != root:
        errs.append("parents[root] != root")
    unreached = d == UNREACHED
    if np.any(parents[unreached] != -1):
        errs.append("unreached vertex with a parent")
    v = np.flatnonzero(~unreached)
    v = v[v != root]
    p = parents[v]
    if np.any((p < 0) | (p >= d.size)):
        errs.append("parent out of range")
        return errs
    if np.any(d[p].astype(np.int64) != d[v].astype(np.int64) - 1):
        errs.append("parent not one level up")
    # edge (p, v) must exist: binary search v in p's sorted row
    adj = np.asarray(adjacency)
    ok = np.zeros(v.size, dtype=bool)
    # vectorised per-row search via a global sorted key (src << 32 | dst)
    keys = (_edge_src(offsets).astype(np.uint64) << np.uint64(32)) | adj.astype(np.uint64)
    want = (p.astype(np.uint64) << np.uint64(32)) | v.astype(np.uint64)
    idx = np.searchsorted(keys, want)
    inb = idx < keys.size
    ok[inb] = keys[idx[inb]] == want[inb]
    if not ok.all():
        errs.append("parent edge missing from graph")
    return errs
