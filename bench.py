"""ButterFly BFS benchmark (driver contract).

Workload: Kronecker scale 29, edge factor 8, seed 1 (BASELINE.json config 5),
built on device; 64 Graph500 roots (default_rng(2103) over non-isolated
vertices).  A step = one BFS from the next root (top-down ButterFly BFS,
parents on), the graph resident in HBM.  Metric = harmonic mean over the
timed roots of E_trav / t (GTEP/s), E_trav = sum of degrees of reached
vertices, t = device time from root injection to termination.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--impl reference times the reference's CPU path (oracle/bfs_omp.c: the
bfs-oracle of SPEC.md restated in C + OpenMP, on every host thread) on the
graph copied to host.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BFS GTEP/s (harmonic mean, 64 roots) Kronecker s29 ef8 at 1/2/4/8 B200"
UNIT = "GTEP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=29)
    ap.add_argument("--edge-factor", type=int, default=8)
    ap.add_argument("--fanout", type=int, default=0, help="0 = min(2, N)")
    ap.add_argument("--roots", type=int, default=64)
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU baseline work")
    ap.add_argument("--no-parents", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ peaks ---
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def committed_traffic(scale, ef):
    """DRAM bytes per expand launch from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "expand_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    return d.get(f"s{scale}_ef{ef}")


# ------------------------------------------------------------ distributed ---
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, local


def hmean(xs):
    xs = [x for x in xs if x > 0]
    return len(xs) / sum(1.0 / x for x in xs) if xs else 0.0


# -------------------------------------------------------------- CPU path ---
def cpu_threads():
    return len(os.sched_getaffinity(0))


def cpu_sample(off, adj, roots, budget_s, steps):
    """Reference CPU path on bounded samples: the oracle's top-down BFS
    restated in C + OpenMP (oracle/bfs_omp.c, the paper's
    OpenMP worker model) on every host thread; each step runs a BFS from the
    next root, stopping after budget_s / steps seconds; returns per-step
    (GTEP/s = edges scanned / time, edges, seconds, completed)."""
    from oracle import cbfs

    per = max(0.5, budget_s / max(1, steps))
    out = []
    for i in range(steps):
        _, scanned, secs, done = cbfs.bfs_top_down(off, adj, int(roots[i % len(roots)]),
                                                   time_budget_s=per, threads=cpu_threads())
        out.append((scanned / secs / 1e9 if secs > 0 else 0.0, scanned, secs, done))
    return out


def host_csr(dg):
    t = time.time()
    off, adj = dg.csr()
    return off, adj, time.time() - t


# ------------------------------------------------------------------- main ---
def main():
    args = parse()
    ws, rank, local = dist_env()
    n_gpus = max(args.gpus, ws)
    fanout = args.fanout or min(2, n_gpus)
    parents = not args.no_parents
    cfg = {
        "workload": f"kronecker s{args.scale} ef{args.edge_factor} seed1, {args.roots} Graph500 roots, "
                    "top-down ButterFly BFS (one step = one BFS)",
        "scale": args.scale, "edge_factor": args.edge_factor, "seed": 1, "roots": args.roots,
        "num_parts": n_gpus, "fanout": fanout, "strategy": "butterfly", "parents": parents,
        "parallelism": f"1D vertex partition x{n_gpus}",
        "l2": "inputs larger than L2 (CSR of s29 ~38 GB vs 126 MB L2)",
        "graph_build": "on device (bit-exact generator, CSR, partition)",
    }

    if args.impl == "reference":
        if rank != 0:
            return
        run_reference(args, cfg, n_gpus)
        return

    if ws > 1:
        line = main_rank(args, cfg)
        if rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
        return

    from paper_2103_13577_b200 import engine, graphs
    from paper_2103_13577_b200.device import levels_readout_bytes

    t0 = time.time()
    g = graphs.kronecker(args.scale, args.edge_factor, 1, device=local)
    dg = g.device
    build_s = time.time() - t0
    roots = graphs.sample_roots(g, args.roots)
    dg.setup(dg.partition_1d(1), 1, "butterfly", parents=parents)
    dg.set_timing(True)
    K, W = args.steps, args.warmup
    for i in range(W):
        dg.bfs(int(roots[(K + i) % len(roots)]), levels=False)
    teps, times, edges, launches = [], [], [], 0
    exp_ms, exp_launch, level_bytes = 0.0, 0, 0
    with ClockSampler(local) as clk:
        dg.timer_start()
        for i in range(K):
            _, _, sizes, st, _ = dg.bfs(int(roots[i % len(roots)]), levels=False)
            teps.append(st.traversed_edges / (st.elapsed_ms * 1e-3) / 1e9)
            times.append(st.elapsed_ms)
            edges.append(st.traversed_edges)
            launches += st.kernel_launches
            exp_ms += st.expand_ms
            exp_launch += st.expand_launches
            # expand algorithmic bytes: 4 B adjacency per edge + 20 B per
            # frontier vertex (q_pre 8, q_base 8, q_v 4); summed over levels =
            # per reached vertex.  Parents (4 B per vertex) are written by the
            # commit's parent pass on the dense levels, so they are not counted
            level_bytes += 4 * st.traversed_edges + 20 * st.reached
        bracket_ms = dg.timer_stop()
    value = hmean(teps)
    peak, peak_src = measured_peaks()
    # the expand's real ceiling: one random visited-bitmap probe per edge
    probe_peak = dg.probe_peak((g.num_vertices + 7) // 8)
    probe_achieved = sum(edges) / (exp_ms * 1e-3)
    achieved = level_bytes / (exp_ms * 1e-3) / 1e9 if exp_ms > 0 else 0.0
    traffic = committed_traffic(args.scale, args.edge_factor)

    # Direction-optimizing phase 1 (paper contribution 3) on the
    # same roots -- reported beside the top-down headline, not instead of it.
    dg.set_direction("optimizing")
    for i in range(W):
        dg.bfs(int(roots[(K + i) % len(roots)]), levels=False)
    do_teps, do_ms, do_bu, do_ex, do_edges = [], [], [], 0, 0
    for i in range(K):
        _, _, _, st, _ = dg.bfs(int(roots[i % len(roots)]), levels=False)
        do_teps.append(st.traversed_edges / (st.elapsed_ms * 1e-3) / 1e9)
        do_ms.append(st.elapsed_ms)
        do_bu.append(st.bottom_up_levels)
        do_ex += st.edges_examined
        do_edges += st.traversed_edges
    dg.set_direction("top-down")
    direction_opt = {"value": round(hmean(do_teps), 3), "unit": UNIT,
                     "bfs_ms_mean": round(float(np.mean(do_ms)), 4),
                     "bottom_up_levels_mean": round(float(np.mean(do_bu)), 2),
                     "bottom_up_edges_examined_per_traversed": round(do_ex / max(1, do_edges), 4),
                     "note": "same graph, roots, parents and levels (bit-identical); phase 1 switches "
                             "top-down/bottom-up by Beamer's rule (alpha 5, beta 1024, tuned on this graph; Beamer's CPU values are 14, 24); TEPS counts "
                             "the same E_trav"}

    # e2e: the public API call (engine.run) with host-resident results
    p1 = graphs.Partition(1, [0, g.num_vertices])
    e2e = []
    n_e2e = min(args.e2e_steps, K)
    h2d = 8  # the root id crosses to the device; the graph is resident
    d2h = 0  # DistanceArray.d: levels packed to 4/8 bits on device, widened on host
    ecfg = engine.EngineConfig(fanout=1)  # the reference's contract: levels only
    engine.run(g, p1, int(roots[0]), ecfg)  # untimed: engine setup for this config
    for i in range(n_e2e):
        r = int(roots[i % len(roots)])
        t = time.perf_counter()
        d, st = engine.run(g, p1, r, ecfg)
        dt = time.perf_counter() - t
        e2e.append(st.traversed_edges / dt / 1e9)
        d2h = max(d2h, levels_readout_bytes(g.num_vertices, st.levels))

    # CPU baseline (bounded sample of the same workload, 1 thread)
    off, adj, copy_s = host_csr(dg)
    cpu = cpu_sample(off, adj, roots, args.cpu_budget, 2)
    cpu_v = hmean([c[0] for c in cpu])
    del off, adj

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": 1, "steps": K,
        "warmup": W, "ms_per_step": round(bracket_ms / K, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": cfg,
        "aggregate_gteps": round(sum(edges) / (bracket_ms * 1e-3) / 1e9, 3),
        "bfs_ms_mean": round(float(np.mean(times)), 4),
        "graph": {"num_vertices": g.num_vertices, "num_edges": g.num_edges,
                  "build_s": round(build_s, 2), "max_degree": dg.max_degree},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": "k_expand (phase 1 top-down expansion)",
                     "achieved_def": "sum over levels of (4 B x edges + 20 B x frontier "
                                     "vertices) / sum of k_expand event time",
                     "peak_src": peak_src,
                     "expand_share": round(exp_ms / sum(times), 4),
                     "expand_launches_per_bfs": exp_launch / K,
                     "l2_probe": {"achieved": round(probe_achieved / 1e9, 2),
                                  "peak": round(probe_peak / 1e9, 2), "unit": "Gprobe/s",
                                  "frac": round(probe_achieved / probe_peak, 4),
                                  "def": "one random 4 B visited-bitmap load per traversed "
                                         "edge / k_expand time, vs random 4 B loads over a "
                                         "bitmap-sized (n/8 B) buffer, measured in this run "
                                         "(csrc/probe_peak.cu)"}},
        "cpu_baseline": {"value": round(cpu_v, 5), "unit": UNIT, "cores": cpu_threads(),
                         "kind": "port",
                         "sample": f"oracle/bfs_omp.c top-down BFS (C + OpenMP, {cpu_threads()} "
                                   f"threads) on the same s{args.scale} CSR copied to host "
                                   f"({copy_s:.1f} s), 2 roots x {args.cpu_budget / 2:.0f} s budget, "
                                   f"GTEP/s = edges scanned / time",
                         "host_threads_available": cpu_threads()},
        "e2e": {"value": round(hmean(e2e), 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": n_e2e,
                "path": "paper_2103_13577_b200.engine.run(g, p, root, EngineConfig()) -> DistanceArray "
                        "in host numpy (uint32), wall clock per call; levels cross PCIe "
                        "packed and are widened by host threads"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "direction_optimizing": direction_opt,
    }
    print(json.dumps(line), flush=True)


def main_rank(args, cfg):
    """N > 1 under torchrun: one rank per GPU, node = rank.  The s29 graph is
    built on every GPU (deterministic); each rank keeps its partition_1d rows.
    A step = one BFS through the device-synchronised engine (bfb_rank_bfs:
    per-round barrier and snapshot sizes through NVLink mailboxes, snapshots
    merged in place from peer HBM); t = max over ranks of the device time from
    root injection to termination.  Returns rank 0's JSON line."""
    import torch
    import torch.distributed as dist

    from paper_2103_13577_b200 import dist as bdist
    from paper_2103_13577_b200 import graphs
    from paper_2103_13577_b200.device import levels_readout_bytes

    ws, rank, local = dist_env()
    dev = int(os.environ.get("BFB_DEVICE", str(local)))
    torch.cuda.set_device(dev)
    if not dist.is_initialized():
        backend = os.environ.get("BFB_DIST_BACKEND", "nccl")  # gloo: several ranks per GPU
        if backend == "nccl":
            dist.init_process_group(backend="nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend=backend)
    comm = bdist.Comm()
    P = comm.size
    fanout = args.fanout or min(2, P)
    parents = not args.no_parents
    t0 = time.time()
    g = graphs.kronecker(args.scale, args.edge_factor, 1, device=dev)
    dg = g.device
    build_s = time.time() - t0
    b = dg.partition_1d(P)
    roots = graphs.sample_roots(g, args.roots)
    eng = bdist.RankEngine(dg, b, fanout, "butterfly", parents, comm)
    dg.set_timing(True)
    K, W = args.steps, args.warmup

    def timed(direction):
        dg.set_direction(direction)
        for i in range(W):
            eng.node.bfs(int(roots[(K + i) % len(roots)]))
        comm.barrier()
        out = {"teps": [], "edges": [], "t": [], "launches": 0, "expand": 0.0, "exchange": 0.0,
               "commit": 0.0, "bu": 0, "reached": 0, "nvl_rate": [], "nvl_bytes": 0}
        dg.timer_start()
        for i in range(K):
            sizes, st = eng.node.bfs(int(roots[i % len(roots)]))
            tmax = comm.allreduce(float(st.elapsed_ms), "max")
            e = int(comm.allreduce(int(st.traversed_edges)))
            out["teps"].append(e / (tmax * 1e-3) / 1e9)
            out["edges"].append(e)
            out["t"].append(tmax)
            out["launches"] += int(st.kernel_launches)
            out["expand"] += comm.allreduce(float(st.expand_ms), "max")
            out["exchange"] += comm.allreduce(float(st.exchange_ms), "max")
            # NVLink payload this rank pulled (queue or bitmap snapshots) and
            # its own exchange time; the rate is max over ranks
            out["nvl_rate"].append(comm.allreduce(
                float(st.exchange_bytes) / max(1e-9, float(st.exchange_ms) * 1e-3), "max"))
            out["nvl_bytes"] += int(comm.allreduce(int(st.exchange_bytes), "max"))
            out["commit"] += comm.allreduce(float(st.commit_ms), "max")
            out["bu"] += int(st.bottom_up_levels)
            out["reached"] += sum(sizes)
        out["bracket"] = comm.allreduce(dg.timer_stop(), "max")
        return out

    with ClockSampler(dev) as clk:
        td = timed("top-down")
    do = timed("optimizing")
    dg.set_direction("top-down")
    value = hmean(td["teps"])
    peak, peak_src = measured_peaks()
    # per-rank algorithmic expand bytes (4 B/edge + 24 B per owned reached
    # vertex, summed over ranks) over the slowest rank's expand time
    level_bytes = 4 * sum(td["edges"]) + (24 if parents else 20) * td["reached"]
    achieved = level_bytes / P / (td["expand"] * 1e-3) / 1e9 if td["expand"] > 0 else 0.0

    # e2e: the public multi-rank API (every rank calls RankEngine.run(root) and
    # gets the DistanceArray in host numpy); wall clock, max over ranks
    e2e = []
    d2h = 0
    eng.run(int(roots[0]), parents=False)
    for i in range(min(args.e2e_steps, K)):
        r = int(roots[i % len(roots)])
        comm.barrier()
        t = time.perf_counter()
        d, st = eng.run(r, parents=False)  # the reference's contract: levels only
        dt = comm.allreduce(time.perf_counter() - t, "max")
        e2e.append(st.traversed_edges / dt / 1e9)
        d2h = max(d2h, levels_readout_bytes(g.num_vertices, st.levels))

    cfg = dict(cfg, fanout=fanout, num_parts=P)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": P, "steps": K,
        "warmup": W, "ms_per_step": round(td["bracket"] / K, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": cfg,
        "aggregate_gteps": round(sum(td["edges"]) / (td["bracket"] * 1e-3) / 1e9, 3),
        "bfs_ms_mean": round(float(np.mean(td["t"])), 4),
        "phase_ms_mean_max_over_ranks": {k: round(td[k] / K, 4)
                                         for k in ("expand", "exchange", "commit")},
        "graph": {"num_vertices": g.num_vertices, "num_edges": g.num_edges,
                  "build_s": round(build_s, 2), "max_degree": dg.max_degree},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None,
                     "kernel": "k_expand_w (phase 1 top-down expansion), per GPU",
                     "achieved_def": "(4 B x edges + 24 B x reached vertices) / N per GPU / "
                                     "slowest rank's expand time",
                     "peak_src": peak_src},
        "cpu_baseline": None,
        "e2e": {"value": round(hmean(e2e), 3), "unit": UNIT, "h2d_bytes_per_step": 8 * P,
                "d2h_bytes_per_step": d2h * P, "steps": len(e2e),
                "path": "paper_2103_13577_b200.dist.RankEngine.run(root) on every rank -> "
                        "DistanceArray in host numpy, wall clock max over ranks"},
        "gpu_launches": td["launches"],
        "clocks": clk.summary(),
        "exchange": "device-synchronised butterfly: per round publish -> NVLink mailbox signal "
                    "-> spin-wait -> in-place merge of the sources' snapshot bitmaps (CUDA IPC)",
        "roofline_nvlink": {"bound": "nvlink", "unit": "GB/s", "peak": 900.0,
                            "achieved": round(float(np.mean(td["nvl_rate"])) / 1e9, 1),
                            "frac": round(float(np.mean(td["nvl_rate"])) / 900e9, 4),
                            "bytes_per_bfs_max_rank": td["nvl_bytes"] // K,
                            "def": "per rank: snapshot bytes pulled from peers (4 B per queued "
                                   "vertex or n/8 B per bitmap) / that rank's phase-2 time "
                                   "(publish + barrier + merge), max over ranks, mean over "
                                   "BFS; peak = NVLink 5 per direction per GPU (nominal)"},
        "direction_optimizing": {"value": round(hmean(do["teps"]), 3), "unit": UNIT,
                                 "bfs_ms_mean": round(float(np.mean(do["t"])), 4),
                                 "bottom_up_levels_mean_per_rank": round(do["bu"] / K, 2)},
    }
    return line if comm.rank == 0 else None


def run_reference(args, cfg, n_gpus):
    """Reference arm: the reference's CPU path (oracle port of SPEC.md's BFS)
    on the host cores, bounded samples per step; rank 0 only."""
    from paper_2103_13577_b200 import graphs

    t0 = time.time()
    g = graphs.kronecker(args.scale, args.edge_factor, 1)
    roots = graphs.sample_roots(g, args.roots)
    off, adj, copy_s = host_csr(g.device)
    g.device.close()
    build_s = time.time() - t0
    K, W = args.steps, args.warmup
    budget = min(args.cpu_budget, 150.0) / max(1, K + W)  # whole run within a few minutes
    cpu_sample(off, adj, roots[K:K + W] if len(roots) > K else roots, budget * W, W)
    t = time.perf_counter()
    res = cpu_sample(off, adj, roots, budget * K, K)
    wall = time.perf_counter() - t
    value = hmean([r[0] for r in res])
    line = {
        "metric": METRIC, "value": round(value, 5), "unit": UNIT, "n_gpus": n_gpus, "steps": K,
        "warmup": W, "ms_per_step": round(wall * 1e3 / K, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "impl": "reference", "config": cfg,
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": cpu_threads(),
                         "kind": "port",
                         "sample": f"each step: oracle/bfs_omp.c top-down BFS (C + OpenMP "
                                   f"restatement of SPEC.md:136-163, {cpu_threads()} threads) from "
                                   f"the next root, stopped after {budget:.2f} s; input graph "
                                   f"(generator, symmetrize, CSR) built on device outside the "
                                   f"timed region and copied to host "
                                   f"({build_s:.1f} s incl. {copy_s:.1f} s copy)",
                         "host_threads_available": cpu_threads()},
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
