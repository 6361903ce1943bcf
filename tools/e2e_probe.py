"""Developer tool: where the end-to-end engine.run time goes (BFS vs levels
D2H vs host overhead) on a device-built Kronecker graph."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2103_13577_b200 import engine, graphs  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 29
g = graphs.kronecker(scale, 8, 1)
dg = g.device
roots = graphs.sample_roots(g, 8)
p1 = graphs.Partition(1, [0, g.num_vertices])
cfg = engine.EngineConfig()
engine.run(g, p1, int(roots[0]), cfg)
for r in roots[:4]:
    t = time.perf_counter()
    d, st = engine.run(g, p1, int(r), cfg)
    t1 = time.perf_counter()
    _, _, _, st2, _ = dg.bfs(int(r), levels=False)
    t2 = time.perf_counter()
    print(f"run {1e3 * (t1 - t):.1f} ms (device {st.elapsed * 1e3:.1f} ms)  bfs-no-levels "
          f"{1e3 * (t2 - t1):.1f} ms (device {st2.elapsed_ms:.1f})", flush=True)
