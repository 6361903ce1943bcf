"""butterfly-schedule module, computed by libbflybfs.

``make_schedule(CN, f)`` returns ``rounds[i][g]`` = tuple of nodes g pulls from
in round i (receive-oriented); the same tables drive the device
exchange in ``bfb_bfs``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def _decode(flat, num_nodes):
    rounds, k = [], 0
    while k < flat.size:
        rnd = []
        for _ in range(num_nodes):
            c = int(flat[k])
            rnd.append(tuple(int(x) for x in flat[k + 1:k + 1 + c]))
            k += 1 + c
        rounds.append(rnd)
    return rounds


def _schedule(num_nodes, fanout, strategy):
    lib = _lib.load()
    need = ctypes.c_int64()
    _lib.check(lib.bfb_make_schedule(int(num_nodes), int(fanout), strategy, None, 0,
                                     ctypes.byref(need)))
    buf = np.empty(max(need.value, 1), dtype=np.int32)
    _lib.check(lib.bfb_make_schedule(int(num_nodes), int(fanout), strategy,
                                     _lib.ptr(buf, ctypes.c_int32), buf.size, ctypes.byref(need)))
    return _decode(buf[:need.value], int(num_nodes))


def make_schedule(num_nodes, fanout):
    """SPEC.md:193-201.  ValueError if fanout > num_nodes."""
    return _schedule(num_nodes, fanout, 0)


def all_to_all_schedule(num_nodes):
    """The all2all strategy as a one-round schedule."""
    return _schedule(num_nodes, 1, 1)


def num_rounds(num_nodes, fanout):
    """ceil(log_max(f,2) CN); 0 for CN = 1."""
    out = ctypes.c_int()
    _lib.check(_lib.load().bfb_num_rounds(int(num_nodes), int(fanout), ctypes.byref(out)))
    return out.value


def message_count_paper(num_nodes, fanout):
    """CN * f * ceil(log_r CN)."""
    out = ctypes.c_int64()
    _lib.check(_lib.load().bfb_message_count_paper(int(num_nodes), int(fanout), ctypes.byref(out)))
    return out.value


def message_count_remote(schedule):
    """Exact cross-node transfers of a schedule."""
    return sum(len(srcs) for rnd in schedule for srcs in rnd)


def buffer_bound(num_vertices, fanout):
    """f * |V| pre-allocated incoming capacity per node."""
    return int(_lib.load().bfb_buffer_bound(int(num_vertices), int(fanout)))
