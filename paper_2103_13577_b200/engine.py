"""engine module: ``run(g, p, root, cfg)`` on B200.

Drop-in for the reference's specified entry point: the
graph and partition are the reference's types (or this package's mirrors),
``cfg.fanout`` / ``cfg.strategy`` keep their meaning, and the result is node
0's ``DistanceArray`` (uint32 hops, UNREACHED = 2^32-1) plus ``RunStats``.
All CN = ``p.num_parts`` compute nodes run as device parts of one GPU context
in this process; the multi-process (one rank per GPU) driver is
``paper_2103_13577_b200.dist``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graphs import UNREACHED, device_graph


@dataclass
class EngineConfig:
    """SPEC.md:279-282.  ``worker_mode`` and ``intra_node_parallelism`` are
    accepted for API compatibility: device results are deterministic in both
    modes.  ``parents`` additionally returns BFS parents.  ``direction``
    selects phase 1: "top-down" (Alg. 2, the reference semantics) or
    "optimizing" (top-down/bottom-up switching, the paper's contribution 3,
    PAPER.md:54; SPEC.md:172 keeps the slot) -- levels, frontier sizes and the
    traversed-edge count are identical either way (exchange volumes differ)."""

    fanout: int = 1
    strategy: str = "butterfly"
    worker_mode: str = "lockstep"
    intra_node_parallelism: int = 1
    parents: bool = False
    direction: str = "top-down"

    def __post_init__(self):
        if self.intra_node_parallelism < 1:
            raise ValueError("intra_node_parallelism must be >= 1")
        if self.worker_mode not in ("lockstep", "lockstep-deterministic", "concurrent"):
            raise ValueError(f"unknown worker_mode {self.worker_mode!r}")
        if self.strategy not in _lib.STRATEGY:
            raise ValueError(f"unknown strategy {self.strategy!r}")
        if self.direction not in _lib.DIRECTION:
            raise ValueError(f"unknown direction {self.direction!r}")


@dataclass
class DistanceArray:
    """SPEC.md:127-133 (+ optional parents: int64, -1 unreached, root->root)."""

    d: np.ndarray
    root: int
    parents: np.ndarray | None = None


@dataclass
class RunStats:
    """SPEC.md:283-286, plus device timings (milliseconds)."""

    levels: int = 0
    per_level_frontier_size: list = field(default_factory=list)
    remote_messages: int = 0
    remote_vertices_transferred: int = 0
    rounds_executed: int = 0
    buffer_high_water: list = field(default_factory=list)
    elapsed: float = 0.0
    traversed_edges: int = 0
    reached: int = 0
    exchange_bytes: int = 0
    device_ms: dict = field(default_factory=dict)
    kernel_launches: int = 0
    edges_examined: int = 0
    bottom_up_levels: int = 0
    sparse_levels: int = 0


def _check_partition(g, p):
    b = np.asarray(p.boundaries, dtype=np.int64)
    if (b.size != p.num_parts + 1 or b[0] != 0 or b[-1] != g.num_vertices
            or np.any(np.diff(b) < 0)):
        raise ValueError("partition does not match graph")
    return b


def run(g, p, root, cfg=None):
    """phase 1 -> phase 2 -> swap -> level+1 until the
    synchronized frontier is empty; returns (node 0's DistanceArray, RunStats)."""
    cfg = cfg or EngineConfig()
    root = int(root)
    if not 0 <= root < g.num_vertices:
        raise ValueError(f"root {root} out of range [0, {g.num_vertices})")
    b = _check_partition(g, p)
    if cfg.fanout > p.num_parts:
        raise ValueError("fanout exceeds num_nodes")
    dg = device_graph(g)
    dg.setup(b, cfg.fanout, cfg.strategy, parents=cfg.parents)
    dg.set_direction(cfg.direction)
    lv, pa, sizes, st, hw = dg.bfs(root, levels=True, parents=cfg.parents)
    return DistanceArray(lv, root, pa), stats_of(sizes, st, hw)


def stats_of(sizes, st, hw):
    return RunStats(
        levels=int(st.levels),
        per_level_frontier_size=list(sizes),
        remote_messages=int(st.remote_messages),
        remote_vertices_transferred=int(st.remote_vertices),
        rounds_executed=int(st.rounds_executed),
        buffer_high_water=[int(x) for x in hw],
        elapsed=st.elapsed_ms / 1e3,
        traversed_edges=int(st.traversed_edges),
        reached=int(st.reached),
        exchange_bytes=int(st.exchange_bytes),
        device_ms={"total": st.elapsed_ms, "expand": st.expand_ms,
                   "exchange": st.exchange_ms, "commit": st.commit_ms,
                   "expand_max_part": st.expand_max_part_ms},
        kernel_launches=int(st.kernel_launches),
        edges_examined=int(st.edges_examined),
        bottom_up_levels=int(st.bottom_up_levels),
        sparse_levels=int(st.sparse_levels),
    )


def all_to_all_sync_config(cfg):
    """EngineConfig for the all-to-all strategy."""
    return EngineConfig(fanout=cfg.fanout, strategy="all2all", worker_mode=cfg.worker_mode,
                        intra_node_parallelism=cfg.intra_node_parallelism, parents=cfg.parents,
                        direction=cfg.direction)


__all__ = ["EngineConfig", "DistanceArray", "RunStats", "run", "UNREACHED"]
