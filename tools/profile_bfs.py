"""Developer tool: one BFS on a device-built Kronecker graph, for ncu captures.

    python tools/profile_bfs.py [--scale 29] [--parents 0|1] [--direction top-down]

Builds the graph, runs one warm-up BFS from the first Graph500 root, then the
profiled BFS from the same root (ncu -s / -c select launches of the second).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2103_13577_b200 import graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=29)
ap.add_argument("--edge-factor", type=int, default=8)
ap.add_argument("--parents", type=int, default=1)
ap.add_argument("--direction", default="top-down")
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--levels", type=int, default=0, help="read the levels out after the last run")
a = ap.parse_args()
g = graphs.kronecker(a.scale, a.edge_factor, 1)
dg = g.device
root = int(graphs.sample_roots(g, 1)[0])
dg.setup(dg.partition_1d(1), 1, "butterfly", parents=bool(a.parents))
dg.set_direction(a.direction)
dg.set_timing(True)
for i in range(1 + a.runs):
    _, _, sizes, st, _ = dg.bfs(root, levels=bool(a.levels) and i == a.runs)
    print(f"root {root} levels {len(sizes)} sizes {sizes} ms {st.elapsed_ms:.2f} "
          f"expand {st.expand_ms:.2f} commit {st.commit_ms:.2f} edges {st.traversed_edges}",
          flush=True)
