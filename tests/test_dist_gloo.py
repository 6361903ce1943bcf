"""Multi-process ButterFly BFS protocol (paper_2103_13577_b200.dist) on CPU:
world_size 2..4 gloo processes, each a compute node (numpy node with file-
backed peer snapshots).  Levels must equal the oracle BFS on every rank and the
aggregated RunStats must equal the lockstep oracle engine's."""

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
from tests import util


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shared, cases, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_13577_b200 import dist as bd
    from tests.oracle_rank_node import OracleRankNode

    comm = bd.Comm()
    off, adj = util.rmat_graph(11)
    results = []
    for fanout, strategy, root in cases:
        b = og.partition_1d(off, world)
        node = OracleRankNode(off, adj, b, rank, shared)
        rounds = bd.my_rounds(world, fanout, strategy, rank)
        sizes = bd.run_levels(node, rounds, comm, root)
        rm = int(comm.allreduce(node.remote_messages))
        rv = int(comm.allreduce(node.remote_vertices))
        te = int(comm.allreduce(node.traversed))
        hw = comm.allgather_i64(node.high_water)
        results.append({"sizes": sizes, "levels_sha": util.sha16(node.levels()), "rm": rm,
                        "rv": rv, "te": te, "hw": hw})
        comm.barrier()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
        json.dump(results, fh)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_multiprocess_protocol_matches_oracle(world):
    cases = [(1, "butterfly", 0), (min(2, world), "butterfly", 5), (world, "butterfly", 77),
             (1, "all2all", 300)]
    with tempfile.TemporaryDirectory() as shared, tempfile.TemporaryDirectory() as out:
        mp.start_processes(_worker, args=(world, _free_port(), shared, cases, out), nprocs=world,
                           join=True, start_method="fork")
        per_rank = [json.load(open(os.path.join(out, f"rank{r}.json"))) for r in range(world)]
    off, adj = util.rmat_graph(11)
    b = og.partition_1d(off, world)
    for i, (f, strat, root) in enumerate(cases):
        ref = ob.bfs_top_down(off, adj, root)
        _, ost = oe.run(off, adj, b, root, fanout=f, strategy=strat)
        for r in range(world):
            res = per_rank[r][i]
            assert res["levels_sha"] == util.sha16(ref), (world, f, strat, r)
            assert res["sizes"] == ost.per_level_frontier_size
            assert res["rm"] == ost.remote_messages
            assert res["rv"] == ost.remote_vertices_transferred
            assert res["te"] == ost.traversed_edges
            assert res["hw"] == ost.buffer_high_water
