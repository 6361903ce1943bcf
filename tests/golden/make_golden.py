"""Regenerate tests/golden/golden.json and the small fixtures from the
REFERENCE itself (pkg/src/bflybfs/graphs.py imported from /root/reference)
plus an independent BFS (scipy.sparse.csgraph, unweighted shortest paths).

Run in the build container (the reference is not present on GPU boxes):
    python tests/golden/make_golden.py            # s10, s12, s16, s20
    python tests/golden/make_golden.py --s24      # adds s24 ef16 (~35 min, ~40 GB RAM)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import shortest_path

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
UNREACHED = 0xFFFFFFFF


def sha16(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def scipy_levels(offsets, adjacency, root):
    n = offsets.size - 1
    mat = sp.csr_matrix((np.ones(adjacency.size, dtype=np.int8), adjacency.astype(np.int64),
                         offsets), shape=(n, n))
    dist = shortest_path(mat, method="D", unweighted=True, indices=[root])[0]
    out = np.full(n, UNREACHED, dtype=np.uint32)
    fin = np.isfinite(dist)
    out[fin] = dist[fin].astype(np.uint32)
    return out


def level_sizes(d):
    r = d[d != UNREACHED]
    return np.bincount(r.astype(np.int64)).tolist() if r.size else []


def graph_entry(R, scale, ef, seed=1, roots_extra=(), bfs=True, nsample=4):
    t = time.time()
    el = R.generate_rmat(scale, ef, seed)
    g = R.build_csr(R.symmetrize(el))
    ent = {
        "scale": scale, "edge_factor": ef, "seed": seed,
        "raw_sha": sha16(el.edges), "raw_first": el.edges[:4].tolist(),
        "raw_last": el.edges[-2:].tolist(),
        "num_edges": int(g.num_edges), "offsets_sha": sha16(g.offsets),
        "adjacency_sha": sha16(g.adjacency), "max_degree": int(g.max_degree),
        "nonisolated": int((g.degrees > 0).sum()),
        "partitions": {str(P): R.partition_1d(g, P).boundaries.tolist()
                       for P in (1, 2, 3, 4, 7, 8, 9, 16)},
    }
    deg = g.degrees
    roots = np.random.default_rng(2103).choice(np.flatnonzero(deg > 0), 64, replace=False)
    ent["roots64"] = roots.tolist()
    if bfs:
        n = g.num_vertices
        pick = [0, 1, n - 1] + list(roots_extra) + roots[:nsample].tolist()
        ent["bfs"] = {}
        for r in dict.fromkeys(int(x) for x in pick):
            d = scipy_levels(g.offsets, g.adjacency, r)
            ent["bfs"][str(r)] = {"levels_sha": sha16(d), "sizes": level_sizes(d),
                                  "traversed_edges": int(deg[d != UNREACHED].sum())}
    ent["gen_seconds"] = round(time.time() - t, 1)
    return ent, el, g


def main():
    sys.path.insert(0, REF_SRC)
    from bflybfs import graphs as R  # the reference, unchanged

    path = os.path.join(HERE, "golden.json")
    gold = json.load(open(path)) if os.path.exists(path) else {}
    gold["_provenance"] = ("reference /root/reference/pkg/src/bflybfs/graphs.py "
                           f"(numpy {np.__version__}); levels from scipy.sparse.csgraph "
                           "shortest_path(unweighted); hashes = sha256(raw bytes)[:16]")
    for scale, ef in ((10, 8), (12, 8), (16, 8), (20, 8)):
        ent, el, g = graph_entry(R, scale, ef)
        gold[f"s{scale}_ef{ef}"] = ent
        print(f"s{scale} ef{ef}: {ent['num_edges']} edges, {ent['gen_seconds']} s", flush=True)
        if scale == 10:
            np.savez_compressed(os.path.join(HERE, "s10_ef8.npz"), raw=el.edges,
                                offsets=g.offsets, adjacency=g.adjacency)
    if "--s24" in sys.argv:
        ent, el, g = graph_entry(R, 24, 16, nsample=2)
        gold["s24_ef16"] = ent
        print(f"s24 ef16: {ent['num_edges']} edges, {ent['gen_seconds']} s", flush=True)
    # SPEC examples for small hand-checkable graphs live in the tests themselves.
    json.dump(gold, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
