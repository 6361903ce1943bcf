"""Multi-process ButterFly BFS: one process per GPU, compute node g = rank g.

The reference simulates CN workers in one process; here
each worker is a process driving its own B200 (torchrun, one rank per GPU).
``run_levels`` is the per-rank form of Alg. 2 /
SPEC.md:298-324:

    begin(root)                                 init
    repeat:
        expand()                                phase 1
        for my sources S_i of butterfly round i:    phase 2
            c = publish(parity)                 round-start snapshot
            counts = allgather(c)               Synchronize() + snapshot sizes
            merge(parity, S_i, counts[S_i])     pull + check-and-set
        f, owned = commit()
        f == allreduce_sum(owned)               termination all-reduce
    until f == 0

The snapshot payload never goes through the collective: ``merge`` reads the
sources' snapshot bitmaps in place from their HBM over NVLink (CUDA IPC
mappings set up once), fused with the OR-merge kernel.  The collective carries
one int64 per rank per round (barrier + sizes).  Snapshot buffers alternate by
round parity, so one barrier per round suffices (a node re-uses a parity only
after every peer has published the following round, which they do only after
finishing the previous merge).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import byref, c_int64

import numpy as np

from . import _lib
from ._lib import check, ptr
from .engine import DistanceArray, RunStats


# ------------------------------------------------------------------ comm ---
class Comm:
    """Host-side plumbing over torch.distributed: barrier + small allgathers on
    a gloo group (CPU tensors), large reductions on the default group."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        self.rank = dist.get_rank()
        self.size = dist.get_world_size()
        if group is None and dist.get_backend() != "gloo":
            group = dist.new_group(backend="gloo")
        self.group = group

    def allgather_i64(self, x):
        t = self.torch.tensor([int(x)], dtype=self.torch.int64)
        out = [self.torch.zeros(1, dtype=self.torch.int64) for _ in range(self.size)]
        self.dist.all_gather(out, t, group=self.group)
        return [int(o.item()) for o in out]

    def allreduce(self, x, op="sum"):
        torch = self.torch
        dt = torch.float64 if isinstance(x, float) else torch.int64
        t = torch.tensor([x], dtype=dt)
        ops = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX,
               "min": self.dist.ReduceOp.MIN}
        self.dist.all_reduce(t, op=ops[op], group=self.group)
        return t.item()

    def allgather_bytes(self, b):
        out = [None] * self.size
        self.dist.all_gather_object(out, bytes(b), group=self.group)
        return out

    def allreduce_min_u32(self, arr):
        """Element-wise min of a uint32 array across ranks (parents assembly)."""
        torch = self.torch
        t = torch.from_numpy(arr.astype(np.int64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return t.numpy()

    def barrier(self):
        self.dist.barrier(group=self.group)


# -------------------------------------------------------------- protocol ---
def my_rounds(num_nodes, fanout, strategy, rank):
    """This node's receive list per round (SPEC.md:193-201 / :325-333)."""
    from . import schedule

    if strategy == "butterfly":
        s = schedule.make_schedule(num_nodes, fanout)
    else:
        schedule.make_schedule(num_nodes, fanout)  # fanout validation
        s = schedule.all_to_all_schedule(num_nodes)
    return [list(rnd[rank]) for rnd in s]


def run_levels(node, rounds, comm, root):
    """One BFS on this rank.  ``node`` implements begin/expand/publish/merge/
    commit; returns per_level_frontier_size (identical on every rank)."""
    node.begin(root)
    sizes = [1]
    counter = 0
    while True:
        node.expand()
        for srcs in rounds:
            parity = counter & 1
            c = node.publish(parity)
            counts = comm.allgather_i64(c)
            node.merge(parity, srcs, [counts[s] for s in srcs])
            counter += 1
        f, owned = node.commit()
        total = int(comm.allreduce(int(owned), "sum"))
        if total != f:
            raise RuntimeError(f"frontier disagreement: local {f}, sum of owned {total}")
        if f == 0:
            return sizes
        sizes.append(f)


# ---------------------------------------------------------------- GPU node ---
class GpuNode:
    """This rank's node on its GPU (libbflybfs multi-process mode)."""

    def __init__(self, dg, boundaries, fanout, strategy, parents, comm):
        self.dg = dg
        self.comm = comm
        self.rank = comm.rank
        lib = _lib.load()
        b = np.ascontiguousarray(boundaries, dtype=np.int64)
        check(lib.bfb_rank_setup(dg.handle, b.size - 1, ptr(b, ctypes.c_int64), int(fanout),
                                 _lib.STRATEGY[strategy], 1 if parents else 0, self.rank))
        dg._engine_key = ("rank", tuple(b.tolist()), fanout, strategy, parents)
        h = (ctypes.c_uint8 * 128)()
        check(lib.bfb_rank_ipc_handles(dg.handle, h))
        allh = comm.allgather_bytes(bytes(h))
        for peer, hb in enumerate(allh):
            if peer != self.rank:
                buf = (ctypes.c_uint8 * 128).from_buffer_copy(hb)
                check(lib.bfb_rank_open_peer(dg.handle, peer, buf))
        self.parents = parents

    def begin(self, root):
        check(_lib.load().bfb_rank_begin(self.dg.handle, int(root)))

    def expand(self):
        check(_lib.load().bfb_rank_expand(self.dg.handle))

    def publish(self, parity):
        c = c_int64()
        check(_lib.load().bfb_rank_publish(self.dg.handle, parity, byref(c)))
        return c.value

    def merge(self, parity, srcs, counts):
        s = np.asarray(srcs, dtype=np.int32)
        c = np.asarray(counts, dtype=np.int64)
        check(_lib.load().bfb_rank_merge(self.dg.handle, parity, ptr(s, ctypes.c_int32),
                                         ptr(c, ctypes.c_int64), s.size))

    def commit(self):
        f, o = c_int64(), c_int64()
        check(_lib.load().bfb_rank_commit(self.dg.handle, byref(f), byref(o)))
        return f.value, o.value

    def finish(self):
        st = _lib.RunStatsC()
        check(_lib.load().bfb_rank_finish(self.dg.handle, byref(st)))
        return st

    def levels(self):
        return self.dg.levels()

    def parents_raw(self):
        out = np.empty(self.dg.num_vertices, dtype=np.uint32)
        check(_lib.load().bfb_rank_parents_raw(self.dg.handle, ptr(out, ctypes.c_uint32)))
        return out


class RankEngine:
    """engine.run for one rank of a torch.distributed job: every rank calls
    ``run(root)`` with the same root; each returns the same DistanceArray."""

    def __init__(self, dg, boundaries, fanout=1, strategy="butterfly", parents=False, comm=None):
        self.comm = comm or Comm()
        n = len(boundaries) - 1
        if n != self.comm.size:
            raise ValueError("partition must have one part per rank")
        if fanout > n:
            raise ValueError("fanout exceeds num_nodes")
        self.rounds = my_rounds(n, fanout, strategy, self.comm.rank)
        self.node = GpuNode(dg, boundaries, fanout, strategy, parents, self.comm)
        self.parents = parents

    def run(self, root, levels=True):
        sizes = run_levels(self.node, self.rounds, self.comm, root)
        st = self.node.finish()
        stats = aggregate_stats(self.comm, sizes, st)
        d = self.node.levels() if levels else None
        par = None
        if self.parents and levels:
            raw = self.node.parents_raw()
            m = self.comm.allreduce_min_u32(raw)
            par = np.where(m == 0xFFFFFFFF, -1, m).astype(np.int64)
        return DistanceArray(d, int(root), par), stats


def aggregate_stats(comm, sizes, st):
    """Global RunStats from per-rank counters (sums; high water per node)."""
    hw = comm.allgather_i64(st.buffer_high_water_max)
    return RunStats(
        levels=len(sizes),
        per_level_frontier_size=list(sizes),
        remote_messages=int(comm.allreduce(int(st.remote_messages))),
        remote_vertices_transferred=int(comm.allreduce(int(st.remote_vertices))),
        rounds_executed=int(st.rounds_executed),
        buffer_high_water=hw,
        elapsed=float(comm.allreduce(float(st.elapsed_ms), "max")) / 1e3,
        traversed_edges=int(comm.allreduce(int(st.traversed_edges))),
        reached=int(sum(sizes)),
        exchange_bytes=int(comm.allreduce(int(st.exchange_bytes))),
        device_ms={"total": float(st.elapsed_ms)},
        kernel_launches=int(st.kernel_launches),
    )


# ----------------------------------------------------------------- bench ---
def bench_rank(args, cfg, metric, unit):
    """bench.py at N > 1 under torchrun: one rank per GPU, s29 graph built on
    every GPU (deterministic), node = rank, K timed BFS; time per BFS = max over
    ranks of the device time; returns rank 0's JSON line."""
    import time

    import torch
    import torch.distributed as dist

    from . import graphs

    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = int(os.environ.get("BFB_DEVICE", str(local)))
    torch.cuda.set_device(dev)
    if not dist.is_initialized():
        backend = os.environ.get("BFB_DIST_BACKEND", "nccl")  # gloo: several ranks per GPU
        if backend == "nccl":
            dist.init_process_group(backend="nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend=backend)
    comm = Comm()
    P = comm.size
    fanout = args.fanout or min(2, P)
    parents = not args.no_parents
    t0 = time.time()
    g = graphs.kronecker(args.scale, args.edge_factor, 1, device=dev)
    dg = g.device
    build_s = time.time() - t0
    b = dg.partition_1d(P)
    roots = graphs.sample_roots(g, args.roots)
    eng = RankEngine(dg, b, fanout, "butterfly", parents, comm)
    K, W = args.steps, args.warmup
    for i in range(W):
        eng.run(int(roots[(K + i) % len(roots)]), levels=False)
    comm.barrier()
    teps, edges, tmax_all, launches = [], [], [], 0
    dg.timer_start()
    for i in range(K):
        sizes = run_levels(eng.node, eng.rounds, comm, int(roots[i % len(roots)]))
        st = eng.node.finish()
        tmax = comm.allreduce(float(st.elapsed_ms), "max")
        e = int(comm.allreduce(int(st.traversed_edges)))
        teps.append(e / (tmax * 1e-3) / 1e9)
        edges.append(e)
        tmax_all.append(tmax)
        launches += int(st.kernel_launches)
    bracket = comm.allreduce(dg.timer_stop(), "max")
    value = len(teps) / sum(1.0 / x for x in teps)
    cfg = dict(cfg, fanout=fanout, num_parts=P)
    line = {
        "metric": metric, "value": round(value, 3), "unit": unit, "n_gpus": P, "steps": K,
        "warmup": W, "ms_per_step": round(bracket / K, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": cfg, "aggregate_gteps": round(sum(edges) / (bracket * 1e-3) / 1e9, 3),
        "graph": {"num_vertices": g.num_vertices, "num_edges": g.num_edges,
                  "build_s": round(build_s, 2)},
        "gpu_launches": launches,
        "exchange": "CUDA-IPC peer snapshot reads fused with the OR-merge; gloo barrier+sizes",
    }
    return line if comm.rank == 0 else None
