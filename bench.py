"""ButterFly BFS benchmark (driver contract; see DESIGN.md §5 Measurement).

Workload: Kronecker scale 29, edge factor 8, seed 1 (BASELINE.json config 5),
built on device; the 64 Graph500 roots (default_rng(2103) over non-isolated
vertices).  ONE STEP = one pass over all 64 roots (64 top-down ButterFly
BFSs, parents on), the graph resident in HBM -- so every run times every
root.  Metric = harmonic mean over the timed BFSs of E_trav / t (GTEP/s),
E_trav = sum of degrees of the reached vertices, t = device time from root
injection to termination (levels and parents final on device).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
with N ranks (one per GPU; fails if fewer than N GPUs are visible).
--impl reference times the reference's CPU path (oracle/bfs_omp.c: the
bfs-oracle of SPEC.md restated in C + OpenMP, every host thread), one
COMPLETE BFS per step from the next root, on the graph copied to host.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
# algorithmic phase-1 bytes: 4 B of adjacency per traversed edge and 20 B per
# frontier vertex (q_pre 8, q_base 8, q_v 4); summed over levels = per reached
# vertex (parents come from the commit's parent pass on the dense levels)
BYTES_PER_EDGE, BYTES_PER_VERTEX = 4, 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=5, help="timed passes over the roots")
    ap.add_argument("--warmup", type=int, default=3, help="untimed passes over the roots")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=29)
    ap.add_argument("--edge-factor", type=int, default=8)
    ap.add_argument("--fanout", type=int, default=0, help="0 = min(2, N)")
    ap.add_argument("--roots", type=int, default=64)
    ap.add_argument("--cpu-roots", type=int, default=2, help="complete CPU BFSs for cpu_baseline")
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
    """(DRAM bytes per expand launch, bytes per expand launch algorithmic,
    source) from the committed ncu launch list of one s29 BFS, if any."""
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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(n):
    """--gpus N without torchrun: re-launch this script as N ranks (one per
    GPU).  BFB_SHARED_GPU=1 (with BFB_DIST_BACKEND=gloo) lets the ranks share
    cuda:0, for protocol runs on a one-GPU box."""
    import torch

    have = torch.cuda.device_count()
    shared = os.environ.get("BFB_SHARED_GPU") == "1"
    if have < n and not shared:
        print(json.dumps({"error": f"--gpus {n} requested but only {have} GPU(s) visible"}),
              flush=True)
        return 2
    env = dict(os.environ)
    if shared:
        env["BFB_DEVICE"] = "0"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def hmean(xs):
    xs = [x for x in xs if x > 0]
    return len(xs) / sum(1.0 / x for x in xs) if xs else 0.0


# -------------------------------------------------------------- CPU path ---
def cpu_threads():
    return len(os.sched_getaffinity(0))


def cpu_complete_bfs(off, adj, root):
    """The reference CPU path for one root: a COMPLETE top-down BFS by
    oracle/bfs_omp.c (SPEC.md:136-163 restated in C + OpenMP, the paper's
    OpenMP worker model) on every host thread.  Returns (levels, GTEP/s,
    seconds), GTEP/s = E_trav / time."""
    from oracle import cbfs

    t = time.perf_counter()
    d = cbfs.bfs_top_down(off, adj, int(root), threads=cpu_threads())
    secs = time.perf_counter() - t
    deg = np.diff(off)
    e = int(deg[d != 0xFFFFFFFF].sum())
    return d, e / secs / 1e9, secs


def sha16(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def cpu_baseline_leg(off, adj, roots, gpu_sha, copy_s):
    """cpu_baseline (untimed for the GPU line): complete CPU BFSs from the
    first roots, their levels compared with the GPU's for the same roots."""
    res = [cpu_complete_bfs(off, adj, r) for r in roots]
    match = all(sha16(d) == gpu_sha[int(r)] for (d, _, _), r in zip(res, roots))
    return {"value": round(hmean([x[1] for x in res]), 5), "unit": UNIT, "cores": cpu_threads(),
            "kind": "port",
            "sample": f"{len(roots)} complete top-down BFSs (roots {[int(r) for r in roots]}) by "
                      f"oracle/bfs_omp.c (C + OpenMP, {cpu_threads()} threads) on the same CSR "
                      f"copied to host ({copy_s:.1f} s), GTEP/s = E_trav / time, "
                      f"{sum(x[2] for x in res):.1f} s of CPU BFS",
            "levels_match_gpu": bool(match),
            "host_threads_available": cpu_threads()}


# ------------------------------------------------------------ the JSON line --
def base_line(args, cfg, n_gpus, K, W, value, bracket_ms):
    return {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": n_gpus, "steps": K,
        "warmup": W, "ms_per_step": round(bracket_ms / K, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": cfg,
    }


def config_of(args, n_gpus, fanout, parents):
    return {
        "workload": f"kronecker s{args.scale} ef{args.edge_factor} seed1, {args.roots} Graph500 "
                    "roots, top-down ButterFly BFS; one step = one pass over all the roots "
                    f"({args.roots} BFSs)",
        "scale": args.scale, "edge_factor": args.edge_factor, "seed": 1, "roots": args.roots,
        "roots_timed": args.roots, "num_parts": n_gpus, "fanout": fanout, "strategy": "butterfly",
        "parents": parents, "parallelism": f"1D vertex partition x{n_gpus}",
        "l2": f"inputs larger than L2 (CSR of s{args.scale} ef{args.edge_factor} "
              f"~{(8 * args.edge_factor + 8) * 2 ** args.scale / 1e9:.1f} GB vs 126 MB L2)",
        "graph_build": "on device (bit-exact generator, CSR, partition)",
    }


# ------------------------------------------------------------------- main ---
def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, max(args.gpus, ws))
        return 0
    if ws == 1 and args.gpus > 1:
        return spawn_ranks(args.gpus)
    if ws > 1:
        line = main_rank(args)
    else:
        line = main_single(args)
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


def main_single(args):
    from paper_2103_13577_b200 import engine, graphs
    from paper_2103_13577_b200.device import levels_readout_bytes

    _, _, local = dist_env()
    parents = not args.no_parents
    cfg = config_of(args, 1, 1, parents)
    t0 = time.time()
    g = graphs.kronecker(args.scale, args.edge_factor, 1, device=local)
    dg = g.device
    build_s = time.time() - t0
    roots = [int(r) for r in graphs.sample_roots(g, args.roots)]
    dg.setup(dg.partition_1d(1), 1, "butterfly", parents=parents)
    dg.set_timing(True)
    K, W = args.steps, args.warmup

    def passes(count, record):
        for _ in range(count):
            for r in roots:
                _, _, _, st, _ = dg.bfs(r, levels=False)
                if record is not None:
                    record.append(st)

    passes(W, None)
    td = []
    with ClockSampler(local) as clk:
        dg.timer_start()
        passes(K, td)
        bracket_ms = dg.timer_stop()
    teps = [st.traversed_edges / (st.elapsed_ms * 1e-3) / 1e9 for st in td]
    value = hmean(teps)
    exp_ms = sum(st.expand_ms for st in td)
    edges = sum(st.traversed_edges for st in td)
    level_bytes = sum(BYTES_PER_EDGE * st.traversed_edges + BYTES_PER_VERTEX * st.reached
                      for st in td)
    launches = sum(st.kernel_launches for st in td)
    exp_launch = sum(st.expand_launches for st in td)
    peak, peak_src = measured_peaks()
    probe_peak = dg.probe_peak((g.num_vertices + 7) // 8)
    achieved = level_bytes / (exp_ms * 1e-3) / 1e9 if exp_ms > 0 else 0.0

    # Direction-optimizing phase 1 (paper contribution 3) on the
    # same roots -- reported beside the top-down headline, not instead of it.
    dg.set_direction("optimizing")
    passes(1, None)
    do = []
    passes(K, do)
    dg.set_direction("top-down")
    do_edges = sum(st.traversed_edges for st in do)
    direction_opt = {
        "value": round(hmean([st.traversed_edges / (st.elapsed_ms * 1e-3) / 1e9 for st in do]), 3),
        "unit": UNIT, "bfs_ms_mean": round(float(np.mean([st.elapsed_ms for st in do])), 4),
        "bottom_up_levels_mean": round(float(np.mean([st.bottom_up_levels for st in do])), 2),
        "bottom_up_edges_examined_per_traversed":
            round(sum(st.edges_examined for st in do) / max(1, do_edges), 4),
        "note": "same graph, roots, parents and levels (bit-identical); phase 1 switches "
                "top-down/bottom-up by Beamer's rule (alpha 14, beta 64, tuned on this graph and s24 ef16; "
                "Beamer's CPU values are 14, 24); TEPS counts the same E_trav"}

    # e2e: the public API call (engine.run) with host-resident results, every
    # root once; the reference's contract returns levels only
    p1 = graphs.Partition(1, [0, g.num_vertices])
    ecfg = engine.EngineConfig(fanout=1)
    engine.run(g, p1, roots[0], ecfg)  # untimed: engine setup for this config
    e2e, d2h, gpu_sha = [], 0, {}
    for r in roots:
        t = time.perf_counter()
        d, st = engine.run(g, p1, r, ecfg)
        dt = time.perf_counter() - t
        e2e.append(st.traversed_edges / dt / 1e9)
        d2h = max(d2h, levels_readout_bytes(g.num_vertices, st.levels))
        if len(gpu_sha) < args.cpu_roots:
            gpu_sha[r] = sha16(d.d)
        del d

    # CPU baseline: complete BFSs of the reference's CPU path on host copies
    t = time.time()
    off, adj = dg.csr()
    copy_s = time.time() - t
    cpu = cpu_baseline_leg(off, adj, roots[:args.cpu_roots], gpu_sha, copy_s)
    del off, adj

    line = base_line(args, cfg, 1, K, W, value, bracket_ms)
    traffic = committed_traffic(args.scale, args.edge_factor)
    line.update({
        "aggregate_gteps": round(edges / (bracket_ms * 1e-3) / 1e9, 3),
        "bfs_ms_mean": round(float(np.mean([st.elapsed_ms for st in td])), 4),
        "bfs_per_step": len(roots),
        "graph": {"num_vertices": g.num_vertices, "num_edges": g.num_edges,
                  "build_s": round(build_s, 2), "max_degree": dg.max_degree},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4),
                     "traffic": traffic.get("dram_bytes_per_launch") if isinstance(traffic, dict)
                     else traffic,
                     "kernel": "k_expand_w (phase 1 top-down expansion)",
                     "achieved_def": f"sum over BFSs and levels of ({BYTES_PER_EDGE} B x edges + "
                                     f"{BYTES_PER_VERTEX} B x frontier vertices) / sum of "
                                     "k_expand_w event time (CUDA events on the engine stream)",
                     "peak_src": peak_src,
                     "expand_share": round(exp_ms / sum(st.elapsed_ms for st in td), 4),
                     "expand_launches_per_bfs": round(exp_launch / len(td), 2),
                     "l2_probe": {"achieved": round(edges / (exp_ms * 1e-3) / 1e9, 2),
                                  "peak": round(probe_peak / 1e9, 2), "unit": "Gprobe/s",
                                  "frac": round(edges / (exp_ms * 1e-3) / probe_peak, 4),
                                  "def": "one random 4 B visited-bitmap load per traversed "
                                         "edge / k_expand_w time, vs random 4 B loads over a "
                                         "bitmap-sized (n/8 B) buffer, measured in this run "
                                         "(csrc/probe_peak.cu)"}},
        "cpu_baseline": cpu,
        "e2e": {"value": round(hmean(e2e), 3), "unit": UNIT, "h2d_bytes_per_step": 8 * len(roots),
                "d2h_bytes_per_step": d2h * len(roots), "bfs": len(e2e),
                "path": "paper_2103_13577_b200.engine.run(g, p, root, EngineConfig()) -> "
                        "DistanceArray in host numpy (uint32), wall clock per call, every root "
                        "once; levels cross PCIe packed and are widened by host threads"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "direction_optimizing": direction_opt,
    })
    return line


def main_rank(args):
    """N > 1 under torchrun: one rank per GPU, node = rank.  Each rank builds
    its share of the s29 graph on its GPU (every vertex's degree + the
    adjacency of its partition_1d rows, graphs.kronecker_part).
    A step = one pass over the roots through the device-synchronised engine
    (bfb_rank_bfs: per-round barrier and snapshot sizes through NVLink
    mailboxes, snapshots merged in place from peer HBM); t = max over ranks of
    the device time from root injection to termination.  Returns rank 0's
    JSON line (None on the other ranks)."""
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
    cfg = config_of(args, P, fanout, parents)
    # each rank builds only its share: whole offsets + its own rows' adjacency
    t0 = time.time()
    g, part = graphs.kronecker_part(args.scale, args.edge_factor, 1, P, comm.rank, device=dev)
    dg = g.device
    build_s = comm.allreduce(time.time() - t0, "max")
    b = part.boundaries
    row_lo, row_hi, held = dg.rows()
    held_max = int(comm.allreduce(int(held), "max"))
    roots = [int(r) for r in graphs.sample_roots(g, args.roots)]
    eng = bdist.RankEngine(dg, b, fanout, "butterfly", parents, comm)
    dg.set_timing(True)
    K, W = args.steps, args.warmup

    def passes(count, out):
        for _ in range(count):
            for r in roots:
                sizes, st = eng.node.bfs(r)
                if out is None:
                    continue
                tmax = comm.allreduce(float(st.elapsed_ms), "max")
                e = int(comm.allreduce(int(st.traversed_edges)))
                out["teps"].append(e / (tmax * 1e-3) / 1e9)
                out["edges"] += e
                out["t"].append(tmax)
                out["reached"] += sum(sizes)
                out["launches"] += int(comm.allreduce(int(st.kernel_launches)))
                for k in ("expand", "exchange", "commit"):
                    out[k] += comm.allreduce(float(getattr(st, k + "_ms")), "max")
                # NVLink payload this rank pulled (queue or bitmap snapshots)
                # over its own exchange time; the rate is max over ranks
                out["nvl_rate"].append(comm.allreduce(
                    float(st.exchange_bytes) / max(1e-9, float(st.exchange_ms) * 1e-3), "max"))
                out["nvl_bytes"] += int(comm.allreduce(int(st.exchange_bytes), "max"))
                out["bu"] += int(st.bottom_up_levels)
                out["exp_launches"] += int(st.expand_launches)  # this rank's, one per level

    def timed(direction):
        dg.set_direction(direction)
        passes(W if direction == "top-down" else 1, None)
        comm.barrier()
        out = {"teps": [], "edges": 0, "t": [], "launches": 0, "expand": 0.0, "exchange": 0.0,
               "commit": 0.0, "bu": 0, "reached": 0, "nvl_rate": [], "nvl_bytes": 0,
               "exp_launches": 0}
        dg.timer_start()
        passes(K, out)
        out["bracket"] = comm.allreduce(dg.timer_stop(), "max")
        return out

    with ClockSampler(dev) as clk:
        td = timed("top-down")
    do = timed("optimizing")
    dg.set_direction("top-down")
    nb = len(td["t"])
    value = hmean(td["teps"])
    peak, peak_src = measured_peaks()
    level_bytes = BYTES_PER_EDGE * td["edges"] + BYTES_PER_VERTEX * td["reached"]
    achieved = level_bytes / P / (td["expand"] * 1e-3) / 1e9 if td["expand"] > 0 else 0.0

    # e2e: the public multi-rank API (every rank calls RankEngine.run(root)
    # and gets the DistanceArray in host numpy); wall clock, max over ranks
    e2e, d2h, gpu_sha = [], 0, {}
    eng.run(roots[0], parents=False)
    for r in roots:
        comm.barrier()
        t = time.perf_counter()
        d, st = eng.run(r, parents=False)
        dt = comm.allreduce(time.perf_counter() - t, "max")
        e2e.append(st.traversed_edges / dt / 1e9)
        d2h = max(d2h, levels_readout_bytes(g.num_vertices, st.levels))
        if len(gpu_sha) < args.cpu_roots:
            gpu_sha[r] = sha16(d.d)
        del d

    cpu = None
    if comm.rank == 0:  # the CPU path needs the whole CSR: built once more, copied, dropped
        t = time.time()
        full = graphs.kronecker(args.scale, args.edge_factor, 1, device=dev).device
        off, adj = full.csr()
        full.close()
        copy_s = time.time() - t
        cpu = cpu_baseline_leg(off, adj, roots[:args.cpu_roots], gpu_sha, copy_s)
        del off, adj
    comm.barrier()

    traffic = committed_traffic(args.scale, args.edge_factor)
    traffic_n = None
    if isinstance(traffic, dict) and traffic.get("algorithmic_bytes_per_launch"):
        # DRAM bytes per launch scale with the algorithmic bytes (ncu at N = 1)
        ratio = traffic["dram_bytes_per_launch"] / traffic["algorithmic_bytes_per_launch"]
        traffic_n = int(ratio * level_bytes / P / max(1, td["exp_launches"]))
    line = base_line(args, cfg, P, K, W, value, td["bracket"])
    line.update({
        "aggregate_gteps": round(td["edges"] / (td["bracket"] * 1e-3) / 1e9, 3),
        "bfs_ms_mean": round(float(np.mean(td["t"])), 4),
        "bfs_per_step": len(roots),
        "phase_ms_mean_max_over_ranks": {k: round(td[k] / nb, 4)
                                         for k in ("expand", "exchange", "commit")},
        "graph": {"num_vertices": g.num_vertices, "num_edges": g.num_edges,
                  "build_s": round(build_s, 2), "max_degree": dg.max_degree,
                  "storage": f"partitioned: each rank holds the whole offsets and its own rows' "
                             f"adjacency (max {held_max} of {g.num_edges} entries per rank)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic_n,
                     "traffic_src": "N = 1 ncu DRAM/algorithmic byte ratio of k_expand_w "
                                    "(profiles/expand_traffic.json) x this run's per-GPU "
                                    "algorithmic bytes per BFS",
                     "kernel": "k_expand_w (phase 1 top-down expansion), per GPU",
                     "achieved_def": f"({BYTES_PER_EDGE} B x edges + {BYTES_PER_VERTEX} B x "
                                     "reached vertices) / N per GPU / slowest rank's expand time",
                     "peak_src": peak_src},
        "cpu_baseline": cpu,
        "e2e": {"value": round(hmean(e2e), 3), "unit": UNIT, "h2d_bytes_per_step": 8 * P * len(roots),
                "d2h_bytes_per_step": d2h * P * len(roots), "bfs": len(e2e),
                "path": "paper_2103_13577_b200.dist.RankEngine.run(root) on every rank -> "
                        "DistanceArray in host numpy, wall clock max over ranks, every root once"},
        "gpu_launches": td["launches"],
        "clocks": clk.summary(),
        "exchange": "device-synchronised butterfly: per round publish -> NVLink mailbox signal "
                    "-> spin-wait -> in-place merge of the sources' snapshots (CUDA IPC)",
        "roofline_nvlink": {"bound": "nvlink", "unit": "GB/s", "peak": 900.0,
                            "achieved": round(float(np.mean(td["nvl_rate"])) / 1e9, 1),
                            "frac": round(float(np.mean(td["nvl_rate"])) / 900e9, 4),
                            "bytes_per_bfs_max_rank": td["nvl_bytes"] // nb,
                            "def": "per rank: snapshot bytes pulled from peers (4 B per queued "
                                   "vertex or n/8 B per bitmap) / that rank's phase-2 time "
                                   "(publish + barrier + merge), max over ranks, mean over "
                                   "BFSs; peak = NVLink 5 per direction per GPU (nominal)"},
        "direction_optimizing": {"value": round(hmean(do["teps"]), 3), "unit": UNIT,
                                 "bfs_ms_mean": round(float(np.mean(do["t"])), 4),
                                 "bottom_up_levels_mean_per_rank": round(do["bu"] / nb, 2)},
    })
    if os.environ.get("BFB_SHARED_GPU") == "1":
        line["note"] = "protocol run: all ranks share one GPU (BFB_SHARED_GPU=1); not a scaling number"
    return line if comm.rank == 0 else None


def run_reference(args, n_gpus):
    """Reference arm: the reference's CPU path (oracle port of SPEC.md's BFS,
    C + OpenMP on every host thread); each step one COMPLETE BFS from the next
    root; rank 0 only.  The input graph is built on device outside the timed
    region (the reference's numpy build cannot make s29 on a host) and copied
    to host."""
    from paper_2103_13577_b200 import graphs

    t0 = time.time()
    g = graphs.kronecker(args.scale, args.edge_factor, 1)
    roots = [int(r) for r in graphs.sample_roots(g, args.roots)]
    t = time.time()
    off, adj = g.device.csr()
    copy_s = time.time() - t
    g.device.close()
    build_s = time.time() - t0
    K, W = args.steps, args.warmup
    for i in range(W):
        cpu_complete_bfs(off, adj, roots[(K + i) % len(roots)])
    t = time.perf_counter()
    res = [cpu_complete_bfs(off, adj, roots[i % len(roots)]) for i in range(K)]
    wall = time.perf_counter() - t
    value = hmean([r[1] for r in res])
    cfg = config_of(args, n_gpus, args.fanout or min(2, n_gpus), not args.no_parents)
    cfg["roots_timed"] = min(K, len(roots))
    line = base_line(args, cfg, n_gpus, K, W, value, wall * 1e3)
    sample = (f"each step: one complete top-down BFS from the next root by oracle/bfs_omp.c "
              f"(C + OpenMP restatement of SPEC.md:136-163, {cpu_threads()} threads); input graph "
              f"(generator, symmetrize, CSR) built on device outside the timed region and copied "
              f"to host ({build_s:.1f} s incl. {copy_s:.1f} s copy)")
    line.update({
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": cpu_threads(),
                         "kind": "port", "sample": sample,
                         "host_threads_available": cpu_threads()},
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    })
    line["ms_per_step"] = round(wall * 1e3 / K, 3)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    sys.exit(main())
