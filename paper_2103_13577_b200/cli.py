"""cli module over the B200 engine.

    python -m paper_2103_13577_b200.cli bench    --kronecker 20 8 1 --nodes 4 --fanout 2
    python -m paper_2103_13577_b200.cli verify   --kronecker 16 8 1 --nodes 9 --fanout 1
    python -m paper_2103_13577_b200.cli schedule --nodes 16 --fanout 4
    python -m paper_2103_13577_b200.cli generate --kronecker 4 2 1 --out g.txt

bench follows SPEC.md:389-397: ``roots`` distinct roots sampled uniformly over
all vertices with ``seed``, one engine run per root, runs sorted by
time with ``trim`` fastest and slowest dropped, trimmed mean time, teps_nominal
= |E| / mean and teps_touched = traversed edges / mean, JSON on
stdout and optional per-run CSV.  verify runs
the CN-node engine per root and compares its full distance array with an
independent host BFS over the graph's host CSR (``_host_bfs``, the SPEC's
bfs_top_down, SPEC.md:136-163 -- no device code shared with the engine), and
always requires the device certificate of SPEC.md:130-132 as well; exit
status 1 with (root, vertex, expected, got) on the first mismatch.
"""

from __future__ import annotations

import argparse
import csv
import json
import sys

import numpy as np

from . import engine, graphs, schedule


def _load_graph(args):
    if args.kronecker:
        s, ef, seed = args.kronecker
        g = graphs.kronecker(int(s), int(ef), int(seed))
        return g, f"kronecker-s{s}-ef{ef}-seed{seed}"
    if not args.graph:
        raise SystemExit("need --graph PATH or --kronecker SCALE EF SEED")
    # parse -> symmetrize -> CSR on device (graphs.load_graph); a .bfbcsr
    # cache written by `generate --out NAME.bfbcsr` loads directly
    if args.graph.endswith(".bfbcsr"):
        return graphs.load_csr(args.graph), args.graph
    return graphs.load_graph(args.graph, args.format), args.graph


def sample_roots(n, count, seed):
    """Distinct roots uniform over all vertices; the same set
    for every (CN, fanout) configuration."""
    k = min(int(count), int(n))
    return np.random.default_rng(seed).choice(n, k, replace=False), k < int(count)


def cmd_bench(args):
    g, name = _load_graph(args)
    p = graphs.partition_1d(g, args.nodes)
    cfg = engine.EngineConfig(fanout=args.fanout, strategy=args.strategy)
    roots, short = sample_roots(g.num_vertices, args.roots, args.seed)
    if len(roots) <= 2 * args.trim:
        raise SystemExit("roots must exceed 2 * trim")
    runs = []
    for r in roots:
        _, st = engine.run(g, p, int(r), cfg)
        runs.append({"root": int(r), "elapsed_s": st.elapsed, "levels": st.levels,
                     "remote_messages": st.remote_messages,
                     "remote_vertices": st.remote_vertices_transferred,
                     "buffer_high_water_max": max(st.buffer_high_water),
                     "traversed_edges": st.traversed_edges,
                     "rounds_executed": st.rounds_executed,
                     "frontier_sizes": st.per_level_frontier_size})
    kept = sorted(runs, key=lambda x: x["elapsed_s"])
    kept = kept[args.trim:len(kept) - args.trim] if args.trim else kept
    mean_t = float(np.mean([x["elapsed_s"] for x in kept]))
    mean_trav = float(np.mean([x["traversed_edges"] for x in kept]))
    report = {
        "graph_name": name, "num_vertices": g.num_vertices, "num_edges": g.num_edges,
        "config": {"nodes": args.nodes, "fanout": args.fanout, "strategy": args.strategy},
        "roots_sampled": len(runs), "roots_kept": len(kept), "roots_short": bool(short),
        "mean_time": mean_t, "teps_nominal": g.num_edges / mean_t,
        "teps_touched": mean_trav / mean_t, "per_run": runs,
    }
    print(json.dumps(report))
    if args.csv:
        cols = ["root", "elapsed_s", "levels", "remote_messages", "remote_vertices",
                "buffer_high_water_max"]
        with open(args.csv, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(cols)
            for x in runs:
                w.writerow([x[c] for c in cols])
    return 0


def _host_bfs(offsets, adjacency, root):
    """verify's reference (SPEC.md:136-163 bfs_top_down): level-synchronous
    BFS on the host CSR in numpy, frontier expanded a level at a time.  It is
    the checker of the verify command, never a path that produces results."""
    n = offsets.size - 1
    d = np.full(n, graphs.UNREACHED, dtype=np.uint32)
    d[root] = 0
    frontier = np.array([root], dtype=np.int64)
    level = 0
    while frontier.size:
        starts, ends = offsets[frontier], offsets[frontier + 1]
        cnt = ends - starts
        idx = np.repeat(starts - np.concatenate(([0], np.cumsum(cnt)[:-1])), cnt) + \
            np.arange(int(cnt.sum()), dtype=np.int64)
        nb = np.unique(adjacency[idx])
        nb = nb[d[nb] == graphs.UNREACHED]
        level += 1
        d[nb] = level
        frontier = nb.astype(np.int64)
    return d


def cmd_verify(args):
    g, _ = _load_graph(args)
    p = graphs.partition_1d(g, args.nodes)
    roots, _ = sample_roots(g.num_vertices, args.roots, args.seed)
    cfg = engine.EngineConfig(fanout=args.fanout, strategy=args.strategy)
    off, adj = np.asarray(g.offsets), np.asarray(g.adjacency)
    for r in roots:
        r = int(r)
        ref = _host_bfs(off, adj, r)
        got, _ = engine.run(g, p, r, cfg)
        bad = np.flatnonzero(ref != got.d)
        if bad.size:
            v = int(bad[0])
            print(json.dumps({"ok": False, "root": r, "vertex": v, "expected": int(ref[v]),
                              "got": int(got.d[v])}))
            return 1
        cert = graphs.device_graph(g).validate(r)
        if cert:
            print(json.dumps({"ok": False, "root": r, "certificate_errors": int(cert)}))
            return 1
    print(json.dumps({"ok": True, "roots": len(roots), "nodes": args.nodes,
                      "fanout": args.fanout}))
    return 0


def cmd_schedule(args):
    s = schedule.make_schedule(args.nodes, args.fanout)
    print(json.dumps({
        "num_nodes": args.nodes, "fanout": args.fanout,
        "rounds": [[list(srcs) for srcs in rnd] for rnd in s],
        "num_rounds": schedule.num_rounds(args.nodes, args.fanout),
        "message_count_paper": schedule.message_count_paper(args.nodes, args.fanout),
        "message_count_remote": schedule.message_count_remote(s),
    }))
    return 0


def cmd_generate(args):
    s, ef, seed = args.kronecker
    g = graphs.kronecker(int(s), int(ef), int(seed))
    if args.out.endswith(".bfbcsr"):
        graphs.save_csr(g, args.out)  # binary CSR cache
    else:
        graphs.write_edge_list(graphs.EdgeList(g.device.edges(), g.num_vertices), args.out)
    print(json.dumps({"num_vertices": g.num_vertices, "num_edges": g.num_edges, "out": args.out}))
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="bflybfs-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def graph_args(sp):
        sp.add_argument("--graph")
        sp.add_argument("--format", default="edges", choices=["edges", "mtx"])
        sp.add_argument("--kronecker", nargs=3, type=int, metavar=("SCALE", "EF", "SEED"))

    b = sub.add_parser("bench")
    graph_args(b)
    b.add_argument("--nodes", type=int, default=1)
    b.add_argument("--fanout", type=int, default=1)
    b.add_argument("--strategy", default="butterfly", choices=["butterfly", "all2all"])
    b.add_argument("--roots", type=int, default=100)
    b.add_argument("--trim", type=int, default=25)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--csv")
    v = sub.add_parser("verify")
    graph_args(v)
    v.add_argument("--nodes", type=int, default=1)
    v.add_argument("--fanout", type=int, default=1)
    v.add_argument("--strategy", default="butterfly", choices=["butterfly", "all2all"])
    v.add_argument("--roots", type=int, default=20)
    v.add_argument("--seed", type=int, default=0)
    sc = sub.add_parser("schedule")
    sc.add_argument("--nodes", type=int, required=True)
    sc.add_argument("--fanout", type=int, required=True)
    gen = sub.add_parser("generate")
    gen.add_argument("--kronecker", nargs=3, type=int, required=True,
                     metavar=("SCALE", "EF", "SEED"))
    gen.add_argument("--out", required=True)
    args = ap.parse_args(argv)
    return {"bench": cmd_bench, "verify": cmd_verify, "schedule": cmd_schedule,
            "generate": cmd_generate}[args.cmd](args)


if __name__ == "__main__":
    sys.exit(main())
