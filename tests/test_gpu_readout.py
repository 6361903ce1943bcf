"""Result read-out (csrc/host_out.cu): levels cross PCIe packed to 4 or 8 bits
per vertex (by the run's level count) or as uint32, parents as uint32, and
host threads widen each landed chunk into the caller's array.  Every mode,
threaded and single-threaded, aligned and misaligned destinations, against
the oracle BFS."""

import ctypes
import os

import numpy as np
import pytest

from oracle import bfs as ob
from oracle import validate as ov
from paper_2103_13577_b200 import _lib
from paper_2103_13577_b200.device import DeviceGraph
from tests import util

pytestmark = pytest.mark.gpu
U = 0xFFFFFFFF


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def _graph(n, edges):
    off, adj = util.csr_of_undirected(n, edges)
    dg = DeviceGraph.from_csr(off, adj)
    dg.setup(np.array([0, n], dtype=np.int64), parents=True)
    return dg, off, adj


def _check_run(dg, off, adj, root):
    lv, pa, sizes, st, _ = dg.bfs(root, levels=True, parents=True)
    ref = ob.bfs_top_down(off, adj, root)
    assert np.array_equal(lv, ref)
    assert not ov.check_parents(off, adj, root, ref, pa)
    # misaligned destinations: uint32 at 4 mod 16, int64 at 8 mod 16
    lbuf = np.empty(ref.size + 1, dtype=np.uint32)
    lmis = lbuf[1:]
    assert lmis.ctypes.data % 16 != 0
    _lib.check(_lib.load().bfb_copy_levels(dg.handle, _ptr(lmis, ctypes.c_uint32)))
    assert np.array_equal(lmis, ref)
    pbuf = np.empty(ref.size + 1, dtype=np.int64)
    pmis = pbuf[1:]
    _lib.check(_lib.load().bfb_copy_parents(dg.handle, _ptr(pmis, ctypes.c_int64)))
    assert np.array_equal(pmis, pa)
    return ref


@pytest.mark.parametrize("threads", ["1", "3", None])
def test_readout_modes(threads, monkeypatch):
    """Nibble (<= 15 levels), byte (16..255) and uint32 (> 255) read-outs,
    at sizes above the 8 MB threading threshold, with 1, 3 and the default
    number of host threads.  Vertex counts are odd so the last packed
    byte/word is partial."""
    if threads is None:
        monkeypatch.delenv("BFB_HOST_THREADS", raising=False)
    else:
        monkeypatch.setenv("BFB_HOST_THREADS", threads)
    # nibble: a star of stars, 17.3M vertices (8.6 MB packed)
    n = (1 << 24) + 600_001
    edges = [(0, i) for i in range(1, 200)] + [(i, 1000 + i) for i in range(1, 200)]
    edges += [(n - 2, n - 1), (n - 3, n - 2)]  # an unreached component at the end
    dg, off, adj = _graph(n, edges)
    ref = _check_run(dg, off, adj, 0)
    assert ref.max(where=ref != U, initial=0) <= 14
    dg.close()
    # byte: a 120-vertex path at the end of 9M vertices (9 MB packed)
    n = 9_000_001
    edges = [(n - 1 - i, n - 2 - i) for i in range(119)]
    dg, off, adj = _graph(n, edges)
    ref = _check_run(dg, off, adj, n - 1)
    assert 15 <= ref.max(where=ref != U, initial=0) <= 254
    dg.close()
    # uint32: a 400-vertex path in 2.1M vertices (8.4 MB)
    n = 2_100_001
    edges = [(i, i + 1) for i in range(1000, 1399)]
    dg, off, adj = _graph(n, edges)
    ref = _check_run(dg, off, adj, 1000)
    assert ref.max(where=ref != U, initial=0) == 399
    dg.close()


def test_readout_small_and_boundary_level_counts():
    """Single-threaded read-outs at the mode boundaries: exactly 15 levels
    (largest nibble value 14), 16 levels (first byte-mode run), 255 and 256
    levels, and 1..9 vertices."""
    for levels in (15, 16, 255, 256):
        n = levels + 5
        edges = [(i, i + 1) for i in range(levels - 1)]
        dg, off, adj = _graph(n, edges)
        ref = _check_run(dg, off, adj, 0)
        assert ref.max(where=ref != U, initial=0) == levels - 1
        dg.close()
    for n in range(1, 10):
        edges = [(i, i + 1) for i in range(n - 1)][: n // 2]
        dg, off, adj = _graph(n, edges)
        for root in range(n):
            _check_run(dg, off, adj, root)
        dg.close()
