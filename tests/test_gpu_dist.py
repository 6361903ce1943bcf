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


def _worker(rank, world, port, cases, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_13577_b200 import dist as bd
    from paper_2103_13577_b200 import graphs

    comm = bd.Comm()
    g = graphs.kronecker(14, 8, 1, device=0)
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
