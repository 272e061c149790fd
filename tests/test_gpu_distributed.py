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
