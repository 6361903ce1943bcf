"""ctypes binding of the C/OpenMP BFS oracle (oracle/bfs_omp.c) -- TEST
INFRASTRUCTURE ONLY (and the timed CPU baseline of bench.py).  Restates
SPEC.md:136-163 / Alg. 1 on all host threads."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libbfs_omp.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = ctypes.CDLL(LIB)
        lib.ob_bfs_top_down.restype = ctypes.c_int
        lib.ob_bfs_top_down.argtypes = [
            ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
            ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_int64),
            ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
        lib.ob_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads():
    return int(load().ob_max_threads())


def bfs_top_down(offsets, adjacency, root, time_budget_s=None, threads=0):
    """Same contract as oracle.bfs.bfs_top_down (uint32 levels; with a budget
    returns (d, edges_scanned, seconds, completed))."""
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    adj = np.ascontiguousarray(adjacency, dtype=np.uint32)
    n = off.size - 1
    d = np.empty(n, dtype=np.uint32)
    sc, secs, done = ctypes.c_int64(), ctypes.c_double(), ctypes.c_int()
    rc = load().ob_bfs_top_down(n, off.ctypes.data, adj.ctypes.data, int(root), d.ctypes.data,
                                int(threads), float(time_budget_s or 0.0), ctypes.byref(sc),
                                ctypes.byref(secs), ctypes.byref(done))
    if rc == -1:
        raise ValueError(f"root {root} out of range [0, {n})")
    if rc != 0:
        raise MemoryError("oracle BFS allocation failed")
    if time_budget_s is None:
        return d
    return d, int(sc.value), float(secs.value), bool(done.value)
