import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2103_13577_b200 import engine, graphs
g = graphs.kronecker(29, 8, 1)
roots = graphs.sample_roots(g, 16)
p1 = graphs.Partition(1, [0, g.num_vertices])
cfg = engine.EngineConfig()
engine.run(g, p1, int(roots[0]), cfg)
ts = []
for r in roots:
    t = time.perf_counter(); d, st = engine.run(g, p1, int(r), cfg); ts.append((st.traversed_edges / (time.perf_counter() - t)) / 1e9)
print(os.environ.get("BFB_LIB", "libbflybfs.so"), "e2e hmean", len(ts) / sum(1 / x for x in ts))
