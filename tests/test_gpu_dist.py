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
                        "hw": st.buffer_high_water, "rounds": st.rounds_executed,
                        "sl": st.sparse_levels})
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


def _part_worker(rank, world, port, cases, out_dir, scale):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_13577_b200 import dist as bd
    from paper_2103_13577_b200 import graphs

    comm = bd.Comm()
    g, part = graphs.kronecker_part(scale, 8, 1, world, rank, device=0)
    dg = g.device
    lo, hi, held = dg.rows()
    off = g.offsets
    info = {"lo": lo, "hi": hi, "held": held, "m": g.num_edges, "b": part.boundaries.tolist(),
            "span": int(off[hi] - off[lo])}
    try:  # whole-graph calls are refused on a rank's share
        dg.csr()
        info["csr_refused"] = False
    except RuntimeError:
        info["csr_refused"] = True
    results = []
    for fanout, strategy, root, device_sync, direction in cases:
        eng = bd.RankEngine(dg, part.boundaries, fanout, strategy, parents=True, comm=comm,
                            device_sync=device_sync)
        dg.set_direction(direction)
        d, st = eng.run(root)
        np.save(os.path.join(out_dir, f"lv_{rank}_{len(results)}.npy"), d.d)
        np.save(os.path.join(out_dir, f"pa_{rank}_{len(results)}.npy"), d.parents)
        results.append({"sizes": st.per_level_frontier_size, "te": st.traversed_edges,
                        "rm": st.remote_messages, "rv": st.remote_vertices_transferred,
                        "sl": st.sparse_levels})
        comm.barrier()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
        json.dump({"info": info, "results": results}, fh)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_ranks_s20_golden(golden, world):
    """SURVEY §8 e storage: each rank builds only its share of the s20 graph
    (every vertex's degree + its own partition_1d rows' adjacency,
    graphs.kronecker_part) and runs the device-synchronised engine on it.
    The shares are disjoint and cover the graph, the boundaries equal the
    golden partition_1d, whole-graph calls are refused, and the levels match
    the golden sha (reference graphs.py + scipy) for both directions, with
    valid parents and RunStats equal to the lockstep oracle engine."""
    e = golden["s20_ef8"]
    roots = [0, e["roots64"][0]]
    cases = [(min(2, world), "butterfly", r, True, d) for r in roots
             for d in ("top-down", "optimizing")]
    cases.append((1, "butterfly", roots[1], False, "top-down"))  # host-sequenced driver
    with tempfile.TemporaryDirectory() as out:
        mp.start_processes(_part_worker, args=(world, _free_port(), cases, out, 20), nprocs=world,
                           join=True, start_method="spawn")
        per_rank = [json.load(open(os.path.join(out, f"rank{r}.json"))) for r in range(world)]
        want_b = e["partitions"][str(world)]
        spans = 0
        for r in range(world):
            info = per_rank[r]["info"]
            assert info["b"] == want_b
            assert (info["lo"], info["hi"]) == (want_b[r], want_b[r + 1])
            assert info["held"] == info["span"] < info["m"]
            assert info["csr_refused"]
            spans += info["span"]
        assert spans == e["num_edges"]
        off, adj = util.rmat_graph(20)
        for i, (f, strat, root, _, direction) in enumerate(cases):
            want = e["bfs"][str(root)]
            _, ost = oe.run(off, adj, np.asarray(want_b), root, fanout=f, strategy=strat)
            for r in range(world):
                lv = np.load(os.path.join(out, f"lv_{r}_{i}.npy"))
                pa = np.load(os.path.join(out, f"pa_{r}_{i}.npy"))
                res = per_rank[r]["results"][i]
                assert util.sha16(lv) == want["levels_sha"], (world, root, direction, r)
                assert res["sizes"] == want["sizes"] and res["te"] == want["traversed_edges"]
                assert not ov.check_parents(off, adj, root, lv, pa)
                if direction == "top-down":
                    assert (res["rm"], res["rv"]) == (ost.remote_messages,
                                                      ost.remote_vertices_transferred)
                # the device-synchronised driver commits the small levels from
                # the claim queue (no sweeps); the host-sequenced one never does
                assert (res["sl"] > 0) == cases[i][3], (i, res["sl"])
