"""A numpy compute node with the GpuNode step interface (dist.run_levels),
built on the oracle's node (oracle/engine.py).  Peer snapshots are exchanged
through files in a shared directory, read in place by the receivers -- the
CPU stand-in for the CUDA-IPC peer reads -- so the multi-process protocol's
barrier / parity discipline is exercised for real under gloo."""

import os

import numpy as np

from oracle import engine as oe


class OracleRankNode:
    def __init__(self, offsets, adjacency, boundaries, rank, shared_dir):
        self.off = np.asarray(offsets, dtype=np.int64)
        self.adj = adjacency
        self.b = np.asarray(boundaries, dtype=np.int64)
        self.rank = rank
        self.dir = shared_dir
        self.n = self.off.size - 1
        self.deg = np.diff(self.off)
        self.remote_messages = self.remote_vertices = self.high_water = 0
        self.traversed = 0

    def _path(self, g, parity):
        return os.path.join(self.dir, f"node{g}_p{parity}.npy")

    def begin(self, root):
        lo, hi = int(self.b[self.rank]), int(self.b[self.rank + 1])
        self.nd = oe._Node(self.rank, lo, hi, self.n)
        self.nd.d[root] = 0
        if lo <= root < hi:
            self.nd.q_local[0] = root
            self.nd.n_local = 1
        self.level = 0
        self.remote_messages = self.remote_vertices = self.high_water = 0
        self.traversed = 0

    def expand(self):
        nd = self.nd
        nd.n_global_next = 0
        nd.n_local_next = 0
        q = nd.q_local[:nd.n_local]
        if q.size == 0:
            return
        dq = self.deg[q]
        self.traversed += int(dq.sum())
        tot = int(dq.sum())
        if tot:
            pos = np.repeat(self.off[q] - (np.cumsum(dq) - dq), dq) + np.arange(tot, dtype=np.int64)
            nd.claim(self.adj[pos].astype(np.int64), self.level)

    def publish(self, parity):
        snap = self.nd.q_global_next[:self.nd.n_global_next].copy()
        tmp = self._path(self.rank, parity) + ".tmp.npy"
        np.save(tmp, snap)
        os.replace(tmp, self._path(self.rank, parity))
        return int(snap.size)

    def merge(self, parity, srcs, counts):
        incoming = 0
        for s, c in zip(srcs, counts):
            if c <= 0:
                continue
            payload = np.load(self._path(s, parity))
            assert payload.size == c, "snapshot read before its publication completed"
            self.remote_messages += 1
            self.remote_vertices += c
            incoming += c
            self.nd.claim(payload, self.level)
        self.high_water = max(self.high_water, incoming)

    def commit(self):
        nd = self.nd
        nd.q_local, nd.q_local_next = nd.q_local_next, nd.q_local
        nd.n_local = nd.n_local_next
        f = nd.n_global_next
        if f:
            self.level += 1
        return int(f), int(nd.n_local)

    def levels(self):
        return self.nd.d.copy()
