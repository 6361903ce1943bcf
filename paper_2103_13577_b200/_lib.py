"""ctypes binding of libbflybfs.so (include/bflybfs.h).

This is the native-kernel slot the reference declares as
``bflybfs._kernels._ext`` (pkg/setup.py:5-15).  Unlike the reference there is
no numpy fallback: if the library is missing, importing the engine fails.
Error codes map to the reference's exception types.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np

LIB_NAME = "libbflybfs.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        os.environ.get("BFB_LIB", LIB_NAME))  # BFB_LIB: tuning-build override

BFB_OK = 0
ERR_INVALID, ERR_ROOT, ERR_PARTITION, ERR_FANOUT = -1, -2, -3, -4
ERR_SELF_EDGE, ERR_DUPLICATE, ERR_NO_REVERSE, ERR_RANGE = -5, -6, -7, -8
ERR_STATE, ERR_CAPACITY, ERR_CUDA, ERR_OOM = -9, -10, -20, -21
ERR_PARSE, ERR_IO = -11, -12

STRATEGY = {"butterfly": 0, "all2all": 1, "all-to-all": 1, "all_to_all": 1}
DIRECTION = {"top-down": 0, "topdown": 0, "optimizing": 1, "direction-optimizing": 1,
             "bottom-up": 2}


class RunStatsC(ctypes.Structure):
    _fields_ = [
        ("levels", c_int64),
        ("rounds_executed", c_int64),
        ("remote_messages", c_int64),
        ("remote_vertices", c_int64),
        ("traversed_edges", c_int64),
        ("reached", c_int64),
        ("buffer_high_water_max", c_int64),
        ("exchange_bytes", c_int64),
        ("elapsed_ms", c_double),
        ("expand_ms", c_double),
        ("exchange_ms", c_double),
        ("commit_ms", c_double),
        ("expand_launches", c_int64),
        ("kernel_launches", c_int64),
        ("edges_examined", c_int64),
        ("bottom_up_levels", c_int64),
        ("expand_max_part_ms", c_double),
        ("switch_checksum", c_int64),
        ("sparse_levels", c_int64),
    ]


class ParseResultC(ctypes.Structure):
    _fields_ = [
        ("num_lines", c_int64),
        ("num_edges", c_int64),
        ("max_id_plus1", c_int64),
        ("err_line", c_int64),
        ("err_code", c_int32),
        ("pad", c_int32),
        ("err_begin", c_int64),
        ("err_end", c_int64),
    ]


_I64P = POINTER(c_int64)
_U32P = POINTER(c_uint32)
_U64P = POINTER(c_uint64)
_I32P = POINTER(c_int32)

# name -> (restype, argtypes)
_SIGNATURES = {
    "bfb_version": (c_char_p, []),
    "bfb_last_error": (c_char_p, []),
    "bfb_device_count": (c_int, [POINTER(c_int)]),
    "bfb_host_alloc": (c_int, [ctypes.c_size_t, POINTER(c_void_p)]),
    "bfb_host_free": (None, [c_void_p]),
    "bfb_num_rounds": (c_int, [c_int, c_int, POINTER(c_int)]),
    "bfb_make_schedule": (c_int, [c_int, c_int, c_int, _I32P, c_int64, _I64P]),
    "bfb_message_count_paper": (c_int, [c_int, c_int, _I64P]),
    "bfb_alloc_count": (c_int64, []),
    "bfb_set_checks": (c_int, [c_void_p, c_int]),
    "bfb_set_small_engine": (c_int, [c_void_p, c_int]),
    "bfb_small_engine_active": (c_int, [c_void_p]),
    "bfb_set_sparse_levels": (c_int, [c_void_p, c_int]),
    "bfb_buffer_bound": (c_int64, [c_int64, c_int]),
    "bfb_create": (c_int, [POINTER(c_void_p), c_int]),
    "bfb_destroy": (None, [c_void_p]),
    "bfb_set_timing": (c_int, [c_void_p, c_int]),
    "bfb_set_direction": (c_int, [c_void_p, c_int, c_double, c_double]),
    "bfb_timer_start": (c_int, [c_void_p]),
    "bfb_timer_stop": (c_int, [c_void_p, POINTER(c_double)]),
    "bfb_rmat_edges": (c_int, [c_void_p, c_int, c_int64, _U64P, _U64P, _U64P, _U32P]),
    "bfb_graph_from_rmat": (c_int, [c_void_p, c_int, c_int64, _U64P, _U64P, _U64P]),
    "bfb_graph_from_rmat_part": (c_int, [c_void_p, c_int, c_int64, _U64P, _U64P, _U64P, c_int,
                                         c_int, _I64P]),
    "bfb_graph_rows": (c_int, [c_void_p, _I64P, _I64P, _I64P]),
    "bfb_graph_from_edges": (c_int, [c_void_p, c_int64, _U32P, c_int64, c_int]),
    "bfb_graph_load_csr": (c_int, [c_void_p, c_int64, c_int64, _I64P, _U32P]),
    "bfb_graph_info": (c_int, [c_void_p, _I64P, _I64P, _I64P]),
    "bfb_graph_copy_csr": (c_int, [c_void_p, _I64P, _U32P]),
    "bfb_graph_copy_edges": (c_int, [c_void_p, _U32P]),
    "bfb_partition_1d": (c_int, [c_void_p, c_int, _I64P]),
    "bfb_count_nonisolated": (c_int, [c_void_p, _I64P]),
    "bfb_select_nonisolated": (c_int, [c_void_p, _I64P, c_int64, _I64P]),
    "bfb_engine_setup": (c_int, [c_void_p, c_int, _I64P, c_int, c_int, c_int]),
    "bfb_bfs": (c_int, [c_void_p, c_int64, _U32P, _I64P, _I64P, c_int64, _I64P,
                        POINTER(RunStatsC)]),
    "bfb_frontier_sizes": (c_int, [c_void_p, _I64P, c_int64, _I64P]),
    "bfb_copy_levels": (c_int, [c_void_p, _U32P]),
    "bfb_copy_parents": (c_int, [c_void_p, _I64P]),
    "bfb_validate": (c_int, [c_void_p, c_int64, _I64P]),
    "bfb_validate_host": (c_int, [c_void_p, c_int64, _U32P, _I64P, _I64P]),
    "bfb_probe_peak": (c_int, [c_void_p, c_int64, _I64P, POINTER(c_double)]),
    "bfb_parse_text": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int64, c_int64,
                               c_int64, POINTER(ParseResultC)]),
    "bfb_parsed_edges": (c_int, [c_void_p, _U32P]),
    "bfb_graph_from_parsed": (c_int, [c_void_p, c_int64, c_int]),
    "bfb_write_edge_list": (c_int, [c_char_p, _U32P, c_int64]),
    "bfb_graph_save": (c_int, [c_void_p, c_char_p]),
    "bfb_graph_load": (c_int, [c_void_p, c_char_p]),
    "bfb_rank_setup": (c_int, [c_void_p, c_int, _I64P, c_int, c_int, c_int, c_int]),
    "bfb_rank_ipc_handles": (c_int, [c_void_p, c_void_p]),
    "bfb_rank_open_peer": (c_int, [c_void_p, c_int, c_void_p]),
    "bfb_rank_begin": (c_int, [c_void_p, c_int64]),
    "bfb_rank_expand": (c_int, [c_void_p]),
    "bfb_rank_publish": (c_int, [c_void_p, c_int, _I64P]),
    "bfb_rank_merge": (c_int, [c_void_p, c_int, _I32P, _I64P, c_int]),
    "bfb_rank_commit": (c_int, [c_void_p, _I64P, _I64P]),
    "bfb_rank_finish": (c_int, [c_void_p, POINTER(RunStatsC)]),
    "bfb_rank_bfs": (c_int, [c_void_p, c_int64, _I64P, c_int64, POINTER(RunStatsC)]),
    "bfb_rank_parents": (c_int, [c_void_p, _I64P]),
    "bfb_rank_parents_raw": (c_int, [c_void_p, _U32P]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load():
    """Load libbflybfs.so (raising ImportError with the build hint if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (or `make -C paper_2103_13577_b200/csrc`); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error():
    return load().bfb_last_error().decode(errors="replace")


def check(rc):
    """Map a C-ABI return code to the reference's exception types."""
    if rc == BFB_OK:
        return
    msg = last_error()
    if rc in (ERR_INVALID, ERR_ROOT, ERR_PARTITION, ERR_FANOUT, ERR_SELF_EDGE, ERR_DUPLICATE,
              ERR_NO_REVERSE, ERR_RANGE):
        raise ValueError(msg)
    if rc == ERR_PARSE:
        raise ValueError(msg)
    if rc == ERR_IO:
        raise OSError(msg)
    if rc == ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def ptr(a, ctype):
    """Pointer to a contiguous numpy array (None for None)."""
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(POINTER(ctype))


def u64_pair(x):
    """128-bit python int -> uint64[2] {hi, lo}."""
    return np.array([(x >> 64) & 0xFFFFFFFFFFFFFFFF, x & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)


def device_count():
    n = c_int(0)
    rc = load().bfb_device_count(ctypes.byref(n))
    return n.value if rc == BFB_OK else 0
