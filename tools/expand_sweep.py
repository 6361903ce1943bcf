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
g = graphs.kronecker(scale, int(os.environ.get("SW_EF", "8")), 1)
dg = g.device
roots = graphs.sample_roots(g, int(os.environ.get("SW_ROOTS", "6")))
for parents, direction in ((False, "top-down"), (True, "top-down"), (True, "optimizing"), (False, "optimizing")):
    P = int(os.environ.get("SW_PARTS", "1"))
    dg.setup(dg.partition_1d(P), min(2, P), "butterfly", parents=parents)
    dg.set_direction(direction, float(os.environ.get("SW_ALPHA", "14")), float(os.environ.get("SW_BETA", "64")))
    dg.set_timing(True)
    dg.bfs(int(roots[0]), levels=False)
    t = []; ex = []; cm = []; xc = []; mp = []
    for r in roots:
        _, _, sizes, st, _ = dg.bfs(int(r), levels=False)
        t.append(st.traversed_edges / st.elapsed_ms / 1e6); ex.append(st.expand_ms); cm.append(st.commit_ms); xc.append(st.exchange_ms); mp.append(st.expand_max_part_ms)
    hm = len(t) / sum(1 / x for x in t)
    print(f"{os.environ.get('SW_TAG')}: {direction} parents={parents} hmean={hm:.1f} GTEP/s expand={sum(ex)/len(ex):.2f} ms commit={sum(cm)/len(cm):.2f} ms exchange={sum(xc)/len(xc):.2f} ms expand_max_part={sum(mp)/len(mp):.2f} ms bu_levels={st.bottom_up_levels} examined={st.edges_examined}", flush=True)
''' % ROOT

if __name__ == "__main__":
    # each argument: LIB[:VAR=VALUE[,VAR=VALUE...]]
    for spec in sys.argv[1:] or ["libbflybfs.so"]:
        lib, _, extra = spec.partition(":")
        env = dict(os.environ, BFB_LIB=lib, SW_TAG=spec)
        for kv in filter(None, extra.split(",")):
            k, _, val = kv.partition("=")
            env[k] = val
        subprocess.run([sys.executable, "-c", BODY], env=env, timeout=600)
