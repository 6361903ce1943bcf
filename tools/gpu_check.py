"""Developer diagnostics for a gpurun box: parity at s16/s20 against the
golden hashes, then build/BFS timings at larger scales.  Not part of the
product; prints one line per check."""

from __future__ import annotations

import hashlib
import os
import sys
import time
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def stage(name, fn):
    t = time.time()
    try:
        fn()
        print(f"[ok] {name} ({time.time() - t:.1f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name} ({time.time() - t:.1f}s)", flush=True)
        traceback.print_exc()
        sys.stdout.flush()


def small():
    from oracle import bfs as obfs
    from oracle import engine as oeng
    from oracle import graphs as og
    from paper_2103_13577_b200 import engine, graphs

    el = graphs.generate_rmat(16, 8, 1)
    print("  raw sha", h(el.edges), "want bd4f8627a80e1335")
    g = graphs.kronecker(16, 8, 1)
    off, adj = g.device.csr()
    print("  csr sha", h(off), h(adj), "want 5f442686dbd20868 990b60349f90e4d0", g.num_edges)
    sym = graphs.symmetrize(el)
    g2 = graphs.build_csr(sym)
    print("  sym/build_csr path", np.array_equal(g2.offsets, off), np.array_equal(g2.adjacency, adj))
    for P in (1, 2, 4):
        p = graphs.partition_1d(g, P)
        print("  partition", P, p.boundaries.tolist())
    want = {0: "7bb61f53288997ac", 1: "e24b2aef12f45387", 65535: "c3734844c9c38e69"}
    p1 = graphs.partition_1d(g, 1)
    for r, w in want.items():
        d, st = engine.run(g, p1, r, engine.EngineConfig(parents=True))
        print("  root", r, h(d.d), w, st.per_level_frontier_size, st.elapsed * 1e3, "ms",
              "validate", g.device.validate(r))
    for P, f in ((2, 2), (4, 2), (4, 4), (3, 1), (8, 2), (8, 8)):
        p = graphs.partition_1d(g, P)
        for strat in ("butterfly", "all2all"):
            d, st = engine.run(g, p, 1, engine.EngineConfig(fanout=f, strategy=strat, parents=True))
            od, ost = oeng.run(off, adj, p.boundaries, 1, fanout=f, strategy=strat)
            same = (np.array_equal(d.d, od) and st.remote_messages == ost.remote_messages
                    and st.remote_vertices_transferred == ost.remote_vertices_transferred
                    and st.buffer_high_water == ost.buffer_high_water
                    and st.rounds_executed == ost.rounds_executed
                    and st.traversed_edges == ost.traversed_edges)
            print("  P", P, "f", f, strat, "match", same, st.remote_messages, ost.remote_messages,
                  st.remote_vertices_transferred, ost.remote_vertices_transferred,
                  st.buffer_high_water, ost.buffer_high_water, "val", g.device.validate(1))


def mid():
    from paper_2103_13577_b200 import engine, graphs

    t = time.time()
    g = graphs.kronecker(20, 8, 1)
    print("  s20 build", time.time() - t)
    off, adj = g.device.csr()
    print("  csr sha", h(off), h(adj), "want dbfc1afc32e5f78e 827868894e8c53a0", g.num_edges)
    p = graphs.partition_1d(g, 1)
    d, st = engine.run(g, p, 0, engine.EngineConfig())
    print("  root0", h(d.d), "want 4f4e988ed2954ba0", st.per_level_frontier_size)


def big(scale, ef, nroots=8):
    from paper_2103_13577_b200 import graphs

    def fn():
        t = time.time()
        g = graphs.kronecker(scale, ef, 1)
        dg = g.device
        print(f"  s{scale} ef{ef} build {time.time() - t:.2f}s n={dg.num_vertices} m={dg.num_edges}"
              f" maxdeg={dg.max_degree}", flush=True)
        roots = graphs.sample_roots(g, nroots)
        for parents in (False, True):
            dg.setup(dg.partition_1d(1), 1, "butterfly", parents=parents)
            dg.set_timing(True)
            teps = []
            for r in roots:
                _, _, sizes, st, _ = dg.bfs(int(r), levels=False)
                teps.append(st.traversed_edges / (st.elapsed_ms * 1e-3) / 1e9)
                print(f"   root {r} parents={parents} {st.elapsed_ms:.3f} ms levels={st.levels} "
                      f"E={st.traversed_edges} {teps[-1]:.1f} GTEP/s expand={st.expand_ms:.3f} "
                      f"commit={st.commit_ms:.3f} launches={st.kernel_launches}", flush=True)
            hm = len(teps) / sum(1 / x for x in teps)
            print(f"  harmonic mean GTEP/s parents={parents}: {hm:.1f}", flush=True)
            print("  validate", dg.validate(int(roots[-1])), flush=True)
        dg.close()
    return fn


if __name__ == "__main__":
    from __graft_entry__ import smoke

    which = sys.argv[1:] or ["smoke", "small", "mid", "s24", "s26"]
    for w in which:
        if w == "smoke":
            stage("smoke", smoke)
        elif w == "small":
            stage("small", small)
        elif w == "mid":
            stage("mid", mid)
        elif w.startswith("prof"):
            # prof<scale>: one parents=True BFS (profiling target)
            sc = int(w[4:6])
            from paper_2103_13577_b200 import graphs as _g

            gg = _g.kronecker(sc, 16 if sc in (24, 27) else 8, 1)
            gg.device.setup(gg.device.partition_1d(1), 1, "butterfly", parents=True)
            r = int(_g.sample_roots(gg, 1)[0])
            _, _, sz, st, _ = gg.device.bfs(r, levels=False)
            print("prof bfs", r, sz, st.elapsed_ms, flush=True)
        elif w.startswith("occ"):
            # occ<scale>: sweep expand blocks/SM (env knob read at setup)
            sc = int(w[3:5])
            for occ in ("2", "3", "4", "6", "8"):
                os.environ["BFB_EXPAND_OCC"] = occ
                print("BFB_EXPAND_OCC", occ, flush=True)
                stage(w + "/" + occ, big(sc, 16 if sc in (24, 27) else 8, nroots=3))
            os.environ.pop("BFB_EXPAND_OCC")
        elif w.startswith("s"):
            sc = int(w[1:3])
            ef = 16 if sc in (24, 27) else 8
            stage(w, big(sc, ef))
