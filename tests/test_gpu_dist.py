"""Multi-process mode on a real GPU: 2 (and 3) ranks share cuda:0, each a
compute node whose merge reads its peers' snapshots through CUDA-IPC
mappings -- the same code path as one rank per GPU.  Levels, parents and
aggregated RunStats vs the oracle."""

import json
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import bfs as ob
from oracle import engine as oe
from oracle import graphs as og
from oracle import validate as ov
from tests import util

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, out_dir, scale=14):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_13577_b200 import dist as bd
    from paper_2103_13577_b200 import graphs

    comm = bd.Comm()
    g = graphs.kronecker(scale, 8, 1, device=0)
    dg = g.device
    b = dg.partition_1d(world)
    results = []
    for fanout, strategy, root, device_sync, direction in cases:
        eng = bd.RankEngine(dg, b, fanout, strategy, parents=True, comm=comm,
                            device_sync=device_sync)
        dg.set_direction(direction)
        d, st = eng.run(root)
        np.save(os.path.join(out_dir, f"lv_{rank}_{len(results)}.npy"), d.d)
        np.save(os.path.join(out_dir, f"pa_{rank}_{len(results)}.npy"), d.parents)
        results.append({"sizes": st.per_level_frontier_size, "rm": st.remote_messages,
                        "rv": st.remote_vertices_transferred, "te": st.traversed_edges,
                        "hw": st.buffer_high_water, "rounds": st.rounds_executed})
        comm.barrier()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
        json.dump(results, fh)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_ranks_on_one_gpu(world):
    # (fanout, strategy, root, device-synchronised, phase-1 direction)
    cases = [(1, "butterfly", 0, False, "top-down"), (world, "butterfly", 7, False, "top-down"),
             (1, "all2all", 123, False, "top-down"), (1, "butterfly", 0, True, "top-down"),
             (world, "butterfly", 7, True, "top-down"), (1, "all2all", 123, True, "top-down"),
             (2, "butterfly", 5, True, "optimizing"), (1, "butterfly", 9, True, "bottom-up"),
             (world, "butterfly", 0, True, "optimizing"), (1, "all2all", 123, True, "optimizing")]
    with tempfile.TemporaryDirectory() as out:
        mp.start_processes(_worker, args=(world, _free_port(), cases, out), nprocs=world,
                           join=True, start_method="spawn")
        per_rank = [json.load(open(os.path.join(out, f"rank{r}.json"))) for r in range(world)]
        off, adj = util.rmat_graph(14)
        b = og.partition_1d(off, world)
        for i, (f, strat, root, _, direction) in enumerate(cases):
            ref = ob.bfs_top_down(off, adj, root)
            _, ost = oe.run(off, adj, b, root, fanout=f, strategy=strat)
            for r in range(world):
                res = per_rank[r][i]
                lv = np.load(os.path.join(out, f"lv_{r}_{i}.npy"))
                pa = np.load(os.path.join(out, f"pa_{r}_{i}.npy"))
                assert np.array_equal(lv, ref), (world, f, strat, r)
                assert not ov.check_parents(off, adj, root, lv, pa)
                assert res["sizes"] == ost.per_level_frontier_size
                assert res["te"] == ost.traversed_edges
                assert res["rounds"] == ost.rounds_executed
                if direction == "top-down":
                    # bottom-up phase 1 discovers only owned vertices, so the
                    # snapshot sizes (exchange accounting) legitimately differ
                    assert res["rm"] == ost.remote_messages
                    assert res["rv"] == ost.remote_vertices_transferred
                    assert res["hw"] == ost.buffer_high_water


def test_ipc_ranks_s20_golden(golden):
    """The device-synchronised rank path (one process per node, peers' HBM
    over CUDA IPC) on the s20 golden graph: 2 ranks, fanout 2, top-down and
    direction-optimizing; levels against the golden sha (reference graphs.py
    + scipy BFS), sizes and traversed edges against the golden entry."""
    e = golden["s20_ef8"]
    roots = [0, e["roots64"][0]]
    cases = [(2, "butterfly", r, True, d) for r in roots for d in ("top-down", "optimizing")]
    world = 2
    with tempfile.TemporaryDirectory() as out:
        mp.start_processes(_worker, args=(world, _free_port(), cases, out, 20), nprocs=world,
                           join=True, start_method="spawn")
        per_rank = [json.load(open(os.path.join(out, f"rank{r}.json"))) for r in range(world)]
        for i, (_, _, root, _, direction) in enumerate(cases):
            want = e["bfs"][str(root)]
            for r in range(world):
                lv = np.load(os.path.join(out, f"lv_{r}_{i}.npy"))
                assert util.sha16(lv) == want["levels_sha"], (root, direction, r)
                assert per_rank[r][i]["sizes"] == want["sizes"]
                assert per_rank[r][i]["te"] == want["traversed_edges"]


def _alpha_worker(rank, world, port, alphas, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_13577_b200 import dist as bd
    from paper_2103_13577_b200 import graphs

    comm = bd.Comm()
    g = graphs.kronecker(16, 8, 1, device=0)
    dg = g.device
    b = dg.partition_1d(world)
    eng = bd.RankEngine(dg, b, 2, "butterfly", parents=True, comm=comm)
    one = None
    if rank == 0:  # the same partition as parts of one context, for the reference checksum
        one = graphs.kronecker(16, 8, 1, device=0).device
        one.setup(b, 2, "butterfly", parents=True)
    res = []
    for a in alphas:
        dg.set_direction("optimizing", alpha=a, beta=24.0)
        d, st = eng.run(0)
        np.save(os.path.join(out_dir, f"lv_{rank}_{len(res)}.npy"), d.d)
        res.append({"bu": eng.node.last_bottom_up_levels, "chk": eng.node.last_switch_checksum,
                    "sizes": st.per_level_frontier_size})
        if one is not None:
            one.set_direction("optimizing", alpha=a, beta=24.0)
            _, _, _, st1, _ = one.bfs(0, levels=False)
            res[-1]["chk1"] = int(st1.switch_checksum)
            res[-1]["bu1"] = int(st1.bottom_up_levels)
        comm.barrier()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
        json.dump(res, fh)
    dist.destroy_process_group()


def test_rank_direction_switch_agrees_across_ranks():
    """Direction-optimizing rank mode decides top-down vs bottom-up on each
    rank from global quantities; partition_1d bounds are not 32-aligned, so
    the neighbours' bits of the boundary words must be in every rank's sum.
    A sweep of alpha through the switching range puts some runs right at the
    threshold: every rank must feed the rule the same per-level numbers as the
    one-context engine over the same partition (checksum), take the same
    number of bottom-up levels, and produce the oracle's levels."""
    world = 3
    alphas = [float(a) for a in np.geomspace(0.01, 1e4, 24)]
    with tempfile.TemporaryDirectory() as out:
        mp.start_processes(_alpha_worker, args=(world, _free_port(), alphas, out), nprocs=world,
                           join=True, start_method="spawn")
        per_rank = [json.load(open(os.path.join(out, f"rank{r}.json"))) for r in range(world)]
        off, adj = util.rmat_graph(16)
        ref = ob.bfs_top_down(off, adj, 0)
        b = og.partition_1d(off, world)
        assert any(x % 32 for x in b[1:-1])
        for i, a in enumerate(alphas):
            bus = {per_rank[r][i]["bu"] for r in range(world)}
            assert len(bus) == 1, (a, bus)
            # the rule's input, level by level, is the same global number
            chks = {per_rank[r][i]["chk"] for r in range(world)}
            assert chks == {per_rank[0][i]["chk1"]} and per_rank[0][i]["chk1"] > 0, (a, chks)
            assert bus == {per_rank[0][i]["bu1"]}, a
            for r in range(world):
                assert np.array_equal(np.load(os.path.join(out, f"lv_{r}_{i}.npy")), ref), (a, r)
