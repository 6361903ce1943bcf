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

``run_levels`` is the host-sequenced form of the protocol (one host round trip
per round; it also drives the numpy test node of tests/).  ``RankEngine.run``
uses the device-synchronised form by default (``bfb_rank_bfs``): the same
rounds, with the barrier and the snapshot sizes exchanged through per-node
mailboxes in HBM that peers write over NVLink, so a level costs one host sync.
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
        h = (ctypes.c_uint8 * 320)()
        check(lib.bfb_rank_ipc_handles(dg.handle, h))
        allh = comm.allgather_bytes(bytes(h))
        for peer, hb in enumerate(allh):
            if peer != self.rank:
                buf = (ctypes.c_uint8 * 320).from_buffer_copy(hb)
                check(lib.bfb_rank_open_peer(dg.handle, peer, buf))
        comm.barrier()  # every peer mapped before any mailbox is written
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

    def bfs(self, root, max_levels=4096):
        """Whole BFS, device-synchronised (bfb_rank_bfs); returns (sizes, stats)."""
        sizes = np.zeros(max_levels, dtype=np.int64)
        st = _lib.RunStatsC()
        check(_lib.load().bfb_rank_bfs(self.dg.handle, int(root), ptr(sizes, ctypes.c_int64),
                                       max_levels, byref(st)))
        if st.levels > max_levels:
            raise RuntimeError("more levels than max_levels")
        self.last_bottom_up_levels = int(st.bottom_up_levels)
        self.last_switch_checksum = int(st.switch_checksum)
        return sizes[:st.levels].tolist(), st

    def finish(self):
        st = _lib.RunStatsC()
        check(_lib.load().bfb_rank_finish(self.dg.handle, byref(st)))
        return st

    def levels(self):
        return self.dg.levels()

    def output_parents(self):
        """Output parents of the last device-synchronised BFS (peer HBM min)."""
        out = np.empty(self.dg.num_vertices, dtype=np.int64)
        check(_lib.load().bfb_rank_parents(self.dg.handle, ptr(out, ctypes.c_int64)))
        return out

    def parents_raw(self):
        out = np.empty(self.dg.num_vertices, dtype=np.uint32)
        check(_lib.load().bfb_rank_parents_raw(self.dg.handle, ptr(out, ctypes.c_uint32)))
        return out


class RankEngine:
    """engine.run for one rank of a torch.distributed job: every rank calls
    ``run(root)`` with the same root; each returns the same DistanceArray."""

    def __init__(self, dg, boundaries, fanout=1, strategy="butterfly", parents=False, comm=None,
                 device_sync=True):
        self.comm = comm or Comm()
        self.device_sync = device_sync
        n = len(boundaries) - 1
        if n != self.comm.size:
            raise ValueError("partition must have one part per rank")
        if fanout > n:
            raise ValueError("fanout exceeds num_nodes")
        self.rounds = my_rounds(n, fanout, strategy, self.comm.rank)
        self.node = GpuNode(dg, boundaries, fanout, strategy, parents, self.comm)
        self.parents = parents

    def run(self, root, levels=True, parents=None):
        """engine.run for this rank.  ``parents`` (default:
        as set up) also assembles the output parents."""
        parents = self.parents if parents is None else parents
        if parents and not self.parents:
            raise RuntimeError("engine set up without parents")
        if self.device_sync:
            sizes, st = self.node.bfs(root)
        else:
            sizes = run_levels(self.node, self.rounds, self.comm, root)
            st = self.node.finish()
        stats = aggregate_stats(self.comm, sizes, st)  # collective: every rank is done
        d = self.node.levels() if levels else None
        par = None
        if parents and levels:
            if self.device_sync:
                par = self.node.output_parents()  # min over the peers' parents, read over NVLink
                self.comm.barrier()  # peers' parents stay intact until everyone has read
            else:
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
        sparse_levels=int(getattr(st, "sparse_levels", 0)),
    )
