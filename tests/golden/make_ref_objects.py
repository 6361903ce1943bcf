"""Fixture for the drop-in tests on a GPU box (where /root/reference is
absent): the arrays of REFERENCE Graph / Partition objects, produced here by
importing the reference's own graphs.py (pkg/src/bflybfs/graphs.py:212-305),
plus independent scipy BFS levels for the test roots.

    python tests/golden/make_ref_objects.py   ->  tests/golden/ref_objects.npz
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import REF_SRC, scipy_levels  # noqa: E402

CASES = {  # name: (scale, edge_factor, seed, num_parts, roots)
    "s12_ef8_seed3": (12, 8, 3, 3, (5, 0, 4095)),
    "s10_ef8_seed1": (10, 8, 1, 4, (0, 1)),
}


def main():
    sys.path.insert(0, REF_SRC)
    from bflybfs import graphs as R

    out = {}
    for name, (s, ef, seed, parts, roots) in CASES.items():
        g = R.build_csr(R.symmetrize(R.generate_rmat(s, ef, seed)))
        p = R.partition_1d(g, parts)
        out[f"{name}_offsets"] = np.asarray(g.offsets)
        out[f"{name}_adjacency"] = np.asarray(g.adjacency)
        out[f"{name}_boundaries"] = np.asarray(p.boundaries)
        out[f"{name}_roots"] = np.asarray(roots, dtype=np.int64)
        for r in roots:
            out[f"{name}_levels_{r}"] = scipy_levels(np.asarray(g.offsets), np.asarray(g.adjacency), r)
    np.savez_compressed(os.path.join(HERE, "ref_objects.npz"), **out)


if __name__ == "__main__":
    main()
