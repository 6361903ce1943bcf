"""Device-resident graph handle over the C ABI (one bfb_ctx per graph).

A ``DeviceGraph`` owns a CSR in HBM (built on device or uploaded) and the
engine buffers of the last ``setup``; nothing here falls back to the CPU.
"""

from __future__ import annotations

import ctypes
import weakref
from ctypes import byref, c_int64, c_void_p

import numpy as np

from . import _lib
from ._lib import check, ptr


class _PinnedPool:
    """Page-locked host buffers handed out as numpy arrays.  A buffer returns
    to the pool when its array is garbage-collected, so repeated engine.run
    calls reuse pinned memory and the levels D2H runs at full PCIe/C2C speed."""

    def __init__(self):
        self._free = {}  # nbytes -> [addr]

    def array(self, count, dtype):
        dtype = np.dtype(dtype)
        nbytes = int(count) * dtype.itemsize
        lst = self._free.setdefault(nbytes, [])
        if not lst:
            # first request of this size: allocate a spare too, so a caller
            # that still holds the previous result never waits on
            # cudaHostAlloc (hundreds of ms for GB-sized buffers)
            for _ in range(2):
                p = c_void_p()
                check(_lib.load().bfb_host_alloc(max(nbytes, 1), byref(p)))
                lst.append(p.value)
        addr = lst.pop()
        buf = (ctypes.c_uint8 * max(nbytes, 1)).from_address(addr)
        weakref.finalize(buf, self._release, nbytes, addr)
        return np.frombuffer(buf, dtype=dtype, count=int(count))

    def _release(self, nbytes, addr):
        lst = self._free.setdefault(nbytes, [])
        if len(lst) < 2:
            lst.append(addr)
        else:
            _lib.load().bfb_host_free(c_void_p(addr))


_POOL = _PinnedPool()


def levels_readout_bytes(num_vertices, num_levels):
    """Bytes the levels read-out moves device -> host for a run with
    num_levels levels (csrc/host_out.cu read_levels): 4 bits per vertex up to
    15 levels, 8 bits up to 255, else 32."""
    if num_levels <= 15:
        return (num_vertices + 1) // 2
    if num_levels <= 255:
        return num_vertices
    return 4 * num_vertices


class DeviceGraph:
    """CSR graph resident on one GPU plus its ButterFly BFS engine state."""

    def __init__(self, device=0):
        lib = _lib.load()
        h = c_void_p()
        check(lib.bfb_create(byref(h), int(device)))
        self._h = h
        self.device = int(device)
        self._engine_key = None
        self._n = self._m = self._maxdeg = None

    # -- lifetime ------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.load().bfb_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("DeviceGraph is closed")
        return self._h

    # -- construction ----------------------------------------------------------
    @classmethod
    def from_rmat(cls, scale, edge_factor, seed, probs=None, device=0):
        """generate_rmat -> symmetrize -> build_csr fused on device."""
        from .graphs import RMAT_PROBS, rmat_device_args

        state, inc, thr = rmat_device_args(scale, edge_factor, seed, probs or RMAT_PROBS)
        dg = cls(device)
        check(_lib.load().bfb_graph_from_rmat(dg.handle, int(scale), int(edge_factor),
                                              ptr(state, ctypes.c_uint64), ptr(inc, ctypes.c_uint64),
                                              ptr(thr, ctypes.c_uint64)))
        dg._refresh()
        return dg

    @classmethod
    def from_rmat_part(cls, scale, edge_factor, seed, num_parts, rank, probs=None, device=0):
        """One rank's share of the generate_rmat -> symmetrize -> build_csr
        graph: every vertex's degree (offsets) plus the adjacency of the
        rank's partition_1d(num_parts) rows only (``boundaries``)."""
        from .graphs import RMAT_PROBS, rmat_device_args

        state, inc, thr = rmat_device_args(scale, edge_factor, seed, probs or RMAT_PROBS)
        dg = cls(device)
        b = np.empty(int(num_parts) + 1, dtype=np.int64)
        check(_lib.load().bfb_graph_from_rmat_part(dg.handle, int(scale), int(edge_factor),
                                                   ptr(state, ctypes.c_uint64),
                                                   ptr(inc, ctypes.c_uint64),
                                                   ptr(thr, ctypes.c_uint64), int(num_parts),
                                                   int(rank), ptr(b, ctypes.c_int64)))
        dg._refresh()
        dg.boundaries = b
        return dg

    @classmethod
    def from_edges(cls, edges, num_vertices, symmetrize, device=0):
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        dg = cls(device)
        check(_lib.load().bfb_graph_from_edges(dg.handle, int(num_vertices),
                                               ptr(e, ctypes.c_uint32), int(e.shape[0]),
                                               1 if symmetrize else 0))
        dg._refresh()
        return dg

    @classmethod
    def from_csr(cls, offsets, adjacency, device=0):
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        adj = np.ascontiguousarray(adjacency, dtype=np.uint32)
        dg = cls(device)
        check(_lib.load().bfb_graph_load_csr(dg.handle, off.size - 1, adj.size,
                                             ptr(off, ctypes.c_int64), ptr(adj, ctypes.c_uint32)))
        dg._refresh()
        return dg

    def _refresh(self):
        n, m, md = c_int64(), c_int64(), c_int64()
        check(_lib.load().bfb_graph_info(self.handle, byref(n), byref(m), byref(md)))
        self._n, self._m, self._maxdeg = n.value, m.value, md.value

    # -- queries ---------------------------------------------------------------
    @property
    def num_vertices(self):
        return self._n

    @property
    def num_edges(self):
        return self._m

    @property
    def max_degree(self):
        return self._maxdeg

    def rows(self):
        """(row_lo, row_hi, adjacency entries) this context holds: all rows,
        or one rank's partition_1d share after from_rmat_part."""
        lo, hi, m = c_int64(), c_int64(), c_int64()
        check(_lib.load().bfb_graph_rows(self.handle, byref(lo), byref(hi), byref(m)))
        return lo.value, hi.value, m.value

    def csr(self):
        off = np.empty(self._n + 1, dtype=np.int64)
        adj = np.empty(self._m, dtype=np.uint32)
        check(_lib.load().bfb_graph_copy_csr(self.handle, ptr(off, ctypes.c_int64),
                                             ptr(adj, ctypes.c_uint32)))
        return off, adj

    def offsets(self):
        off = np.empty(self._n + 1, dtype=np.int64)
        check(_lib.load().bfb_graph_copy_csr(self.handle, ptr(off, ctypes.c_int64), None))
        return off

    def adjacency(self):
        adj = np.empty(self._m, dtype=np.uint32)
        check(_lib.load().bfb_graph_copy_csr(self.handle, None, ptr(adj, ctypes.c_uint32)))
        return adj

    def edges(self):
        out = np.empty((self._m, 2), dtype=np.uint32)
        check(_lib.load().bfb_graph_copy_edges(self.handle, ptr(out, ctypes.c_uint32)))
        return out

    def partition_1d(self, num_parts):
        b = np.empty(int(num_parts) + 1, dtype=np.int64)
        check(_lib.load().bfb_partition_1d(self.handle, int(num_parts), ptr(b, ctypes.c_int64)))
        return b

    def count_nonisolated(self):
        c = c_int64()
        check(_lib.load().bfb_count_nonisolated(self.handle, byref(c)))
        return c.value

    def select_nonisolated(self, ranks):
        r = np.ascontiguousarray(ranks, dtype=np.int64)
        out = np.empty(r.size, dtype=np.int64)
        check(_lib.load().bfb_select_nonisolated(self.handle, ptr(r, ctypes.c_int64), r.size,
                                                 ptr(out, ctypes.c_int64)))
        return out

    # -- engine ----------------------------------------------------------------
    def setup(self, boundaries, fanout=1, strategy="butterfly", parents=False):
        """Allocate the per-node engine buffers once."""
        b = np.ascontiguousarray(boundaries, dtype=np.int64)
        if strategy not in _lib.STRATEGY:
            raise ValueError(f"unknown strategy {strategy!r}")
        key = (tuple(b.tolist()), int(fanout), _lib.STRATEGY[strategy], bool(parents))
        if key == self._engine_key:
            return
        self._engine_key = None
        check(_lib.load().bfb_engine_setup(self.handle, b.size - 1, ptr(b, ctypes.c_int64),
                                           int(fanout), _lib.STRATEGY[strategy],
                                           1 if parents else 0))
        self._engine_key = key

    @property
    def num_parts(self):
        return len(self._engine_key[0]) - 1 if self._engine_key else 0

    def set_direction(self, direction="top-down", alpha=14.0, beta=64.0):
        """Phase-1 direction: "top-down" (Alg. 2), "optimizing" (Beamer
        switch) or "bottom-up"; levels are identical in every mode."""
        if direction not in _lib.DIRECTION:
            raise ValueError(f"unknown direction {direction!r}")
        check(_lib.load().bfb_set_direction(self.handle, _lib.DIRECTION[direction], float(alpha),
                                            float(beta)))

    def timer_start(self):
        check(_lib.load().bfb_timer_start(self.handle))

    def timer_stop(self):
        ms = ctypes.c_double()
        check(_lib.load().bfb_timer_stop(self.handle, byref(ms)))
        return ms.value

    def probe_peak(self, nbytes):
        """Random 4-byte loads per second over an nbytes device buffer (the
        phase-1 probe ceiling; see csrc/probe_peak.cu)."""
        n, ms = c_int64(), ctypes.c_double()
        check(_lib.load().bfb_probe_peak(self.handle, int(nbytes), byref(n), byref(ms)))
        return n.value / (ms.value * 1e-3)

    def set_checks(self, frontier_agreement=True):
        """Instrumented runs (SPEC.md acceptance 8): after every phase 2 all
        nodes' visited bitmaps must be identical, else bfs() raises."""
        check(_lib.load().bfb_set_checks(self.handle, 1 if frontier_agreement else 0))

    def set_small_engine(self, enabled=True):
        """Small graphs (|V| <= 2^15): run top-down BFSs as one single-CTA
        launch (True, default) or force the level-synchronous engine (False)."""
        check(_lib.load().bfb_set_small_engine(self.handle, 1 if enabled else 0))

    def set_sparse_levels(self, enabled=True):
        """One node, top-down: commit levels with few frontier edges from the
        phase-1 claim queue (True, default) or always by bitmap sweeps."""
        check(_lib.load().bfb_set_sparse_levels(self.handle, 1 if enabled else 0))

    @property
    def small_engine_active(self):
        """True if the next top-down bfs() runs on the single-CTA engine."""
        return bool(_lib.load().bfb_small_engine_active(self.handle))

    def set_timing(self, enabled):
        check(_lib.load().bfb_set_timing(self.handle, 1 if enabled else 0))

    def bfs(self, root, levels=True, parents=False, max_levels=4096):
        """One BFS on the configured engine.  Returns (levels|None,
        parents|None, frontier_sizes, RunStatsC, buffer_high_water)."""
        if self._engine_key is None:
            raise RuntimeError("engine not set up")
        lv = _POOL.array(self._n, np.uint32) if levels else None
        pa = np.empty(self._n, dtype=np.int64) if parents else None
        sizes = np.zeros(max_levels, dtype=np.int64)
        hw = np.zeros(self.num_parts, dtype=np.int64)
        st = _lib.RunStatsC()
        check(_lib.load().bfb_bfs(self.handle, int(root), ptr(lv, ctypes.c_uint32),
                                  ptr(pa, ctypes.c_int64), ptr(sizes, ctypes.c_int64), max_levels,
                                  ptr(hw, ctypes.c_int64), byref(st)))
        if st.levels > max_levels:
            sizes = self.frontier_sizes()
        else:
            sizes = sizes[:st.levels].tolist()
        return lv, pa, sizes, st, hw

    def frontier_sizes(self):
        """per_level_frontier_size of the last run, all levels."""
        n = c_int64()
        check(_lib.load().bfb_frontier_sizes(self.handle, None, 0, byref(n)))
        out = np.empty(n.value, dtype=np.int64)
        check(_lib.load().bfb_frontier_sizes(self.handle, ptr(out, ctypes.c_int64), out.size, byref(n)))
        return out.tolist()

    def levels(self):
        out = _POOL.array(self._n, np.uint32)
        check(_lib.load().bfb_copy_levels(self.handle, ptr(out, ctypes.c_uint32)))
        return out

    def parents(self):
        out = np.empty(self._n, dtype=np.int64)
        check(_lib.load().bfb_copy_parents(self.handle, ptr(out, ctypes.c_int64)))
        return out

    def validate(self, root):
        """Device certificate of the last run: 0 = valid."""
        e = c_int64()
        check(_lib.load().bfb_validate(self.handle, int(root), byref(e)))
        return e.value

    def validate_levels(self, root, levels, parents=None):
        """The same certificate for given levels (uint32[n]) and optional
        parents (int64[n], -1 = none): bitmask, 0 = valid (1 root, 2 edge with
        one endpoint unreached, 4 edge spanning > 1 level, 8 reached vertex
        without a predecessor, 16 bad parent)."""
        lv = np.ascontiguousarray(levels, dtype=np.uint32)
        pa = None if parents is None else np.ascontiguousarray(parents, dtype=np.int64)
        if lv.size != self._n or (pa is not None and pa.size != self._n):
            raise ValueError("levels / parents must have num_vertices entries")
        e = c_int64()
        check(_lib.load().bfb_validate_host(self.handle, int(root), ptr(lv, ctypes.c_uint32),
                                            ptr(pa, ctypes.c_int64), byref(e)))
        return e.value
