"""Tuning sweep (developer tool): one process per (library variant, env)
setting; s29 graph built on device; 6 roots; prints GTEP/s and phase times."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BODY = r'''
import sys, os
sys.path.insert(0, %r)
from paper_2103_13577_b200 import graphs
scale = int(os.environ.get("SW_SCALE", "29"))
g = graphs.kronecker(scale, 8, 1)
dg = g.device
roots = graphs.sample_roots(g, 6)
for parents, direction in ((False, "top-down"), (True, "top-down"), (True, "optimizing"), (False, "optimizing")):
    dg.setup(dg.partition_1d(1), 1, "butterfly", parents=parents)
    dg.set_direction(direction)
    dg.set_timing(True)
    dg.bfs(int(roots[0]), levels=False)
    t = []; ex = []; cm = []
    for r in roots:
        _, _, sizes, st, _ = dg.bfs(int(r), levels=False)
        t.append(st.traversed_edges / st.elapsed_ms / 1e6); ex.append(st.expand_ms); cm.append(st.commit_ms)
    hm = len(t) / sum(1 / x for x in t)
    print(f"{os.environ.get('SW_TAG')}: {direction} parents={parents} hmean={hm:.1f} GTEP/s expand={sum(ex)/len(ex):.2f} ms commit={sum(cm)/len(cm):.2f} ms bu_levels={st.bottom_up_levels} examined={st.edges_examined}", flush=True)
''' % ROOT

if __name__ == "__main__":
    settings = []
    for lib in sys.argv[1:] or ["libbflybfs.so"]:
        for persist in ("0",):
            settings.append((lib, persist))
    for lib, persist in settings:
        env = dict(os.environ, BFB_LIB=lib, BFB_L2_PERSIST=persist, SW_TAG=f"{lib} persist={persist}")
        subprocess.run([sys.executable, "-c", BODY], env=env, timeout=600)
