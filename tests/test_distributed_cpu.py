"""The N>1 path on CPU with world-size-2 gloo: tree blocks built by different
ranks (here by the oracle) and broadcast by their owners assemble the exact
single-process index on every rank; query shards cover the batch."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1509_06957_b200.distributed import broadcast_tree_blocks, query_shard, tree_block


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_blocks_partition_trees_and_queries():
    for T in (1, 7, 100, 500, 1000):
        for G in (1, 2, 3, 4, 8):
            blocks = [tree_block(r, G, T) for r in range(G)]
            assert blocks[0][0] == 0 and blocks[-1][1] == T
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(G - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
            shards = [query_shard(r, G, 10_000) for r in range(G)]
            assert sum(b - a for a, b in shards) == 10_000


def _worker(rank, world, port, X, T, depth, seed, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = X.shape[0]
    splits = torch.zeros((T, (1 << depth) - 1), dtype=torch.float32)
    offsets = torch.zeros((T, (1 << depth) + 1), dtype=torch.int64)
    indices = torch.full((T, n), -1, dtype=torch.int32)
    b0, b1 = tree_block(rank, world, T)
    for t in range(b0, b1):  # this rank's trees only
        _, (s, o, i) = O.build_one_tree(X, depth, 1 / np.sqrt(X.shape[1]), seed, t)
        splits[t] = torch.from_numpy(s)
        offsets[t] = torch.from_numpy(o)
        indices[t] = torch.from_numpy(i)
    broadcast_tree_blocks((splits, offsets, indices), T)
    out[rank] = (splits.numpy().copy(), offsets.numpy().copy(), indices.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("T", [5, 8])
def test_gloo_two_ranks_assemble_the_single_process_index(T):
    rng = np.random.default_rng(3)
    X = rng.standard_normal((900, 12)).astype(np.float32)
    depth, seed = 5, 21
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, _free_port(), X, T, depth, seed, out), nprocs=2,
                       join=True, start_method="fork")
    from oracle import oracle as O

    ref = O.grow_trees(X, T, depth, seed=seed)
    for r in range(2):
        s, o, i = out[r]
        assert s.tobytes() == ref["splits"].tobytes()
        assert np.array_equal(o, ref["leaf_offsets"])
        assert np.array_equal(i, ref["leaf_indices"])
