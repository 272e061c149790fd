"""The NCCL path on the one GPU available: a world-size-1 process group runs
grow_trees_distributed (block build + owner broadcasts) and the sharded query
entry point, and must equal the single-process results bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_1509_06957_b200 as mrpt
from conftest import gaussian
from paper_1509_06957_b200.distributed import (
    approximate_knn_batch_sharded,
    grow_trees_distributed,
)

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_world1_distributed_build_and_sharded_query(rng):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        X = gaussian(rng, 6000, 40)
        Q = gaussian(rng, 50, 40)
        a = grow_trees_distributed(X, 9, 7, seed=5)
        b = mrpt.grow_trees(X, 9, 7, seed=5)
        assert a.splits.tobytes() == b.splits.tobytes()
        assert np.array_equal(a.leaf_offsets, b.leaf_offsets)
        assert np.array_equal(a.leaf_indices, b.leaf_indices)
        (s0, s1), ids, dists, counts = approximate_knn_batch_sharded(Q, 5, a, 2)
        rids, rd, rc = mrpt.approximate_knn_batch(Q, 5, b, 2)
        assert (s0, s1) == (0, 50)
        assert np.array_equal(ids, rids) and np.array_equal(counts, rc)
    finally:
        dist.destroy_process_group()


def _world2_worker(rank, world, port, X, Q, T, depth, seed, batch, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_1509_06957_b200.distributed import (
        approximate_knn_batch_sharded,
        grow_trees_distributed,
    )

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        idx = grow_trees_distributed(torch.from_numpy(X).cuda(), T, depth, seed=seed,
                                     batch_trees=batch)
        (s0, s1), ids, dists, counts = approximate_knn_batch_sharded(Q, 7, idx, 2)
        out[rank] = (idx.splits.copy(), idx.leaf_offsets.copy(), idx.leaf_indices.copy(),
                     int(idx.dataset_checksum), (s0, s1), ids, counts)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T,batch", [(9, 2), (5, None)])
def test_world2_distributed_build_on_one_gpu(rng, T, batch):
    """grow_trees_distributed itself at world size 2: two processes share
    cuda:0 over a gloo group (no kernel waits on another rank's kernel -- the
    broadcasts run on the host), each builds its tree block in batches and
    broadcasts every batch as it completes; both ranks end with the
    single-process index bit for bit, and their query shards cover the batch."""
    import torch.multiprocessing as mp

    X = gaussian(rng, 5000, 24)
    Q = gaussian(rng, 64, 24)
    depth, seed = 6, 13
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_world2_worker, args=(2, _port(), X, Q, T, depth, seed, batch, out), nprocs=2,
                       join=True, start_method="spawn")
    ref = mrpt.grow_trees(X, T, depth, seed=seed)
    rids, rd, rc = mrpt.approximate_knn_batch(Q, 7, ref, 2)
    for r in range(2):
        s, o, i, cs, (s0, s1), ids, counts = out[r]
        assert s.tobytes() == ref.splits.tobytes()
        assert np.array_equal(o, ref.leaf_offsets)
        assert np.array_equal(i, ref.leaf_indices)
        assert cs == ref.dataset_checksum
        assert np.array_equal(ids, rids[s0:s1]) and np.array_equal(counts, rc[s0:s1])
    assert out[0][4] == (0, 32) and out[1][4] == (32, 64)
