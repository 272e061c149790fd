"""Multi-GPU execution: one process per GPU (torch.distributed, NCCL over NVLink).

The path partitions naturally:

* build -- trees are independent (trees.py:217-224: tree t depends only on X,
  seed and t), so rank r builds the contiguous block of trees
  [floor(rT/G), floor((r+1)T/G)) on its own GPU, in tree batches; after each
  batch every owner broadcasts that batch's split values, leaf offsets and
  leaf ids to all ranks, asynchronously, so the transfer overlaps the next
  batch's build (the only collectives of the whole path).
  The random matrices are re-drawn on every host (microseconds per tree), so
  they never cross NVLink.
* queries -- every rank holds the full index and answers its own contiguous
  shard of the query batch: no collective on the query path.
"""

from __future__ import annotations

import numpy as np

from . import _device
from .search import approximate_knn_batch
from .trees import (
    _alloc_index,
    _finish_index,
    _grow_block,
    _validate_grow,
    sample_sparse_matrix,
)

__all__ = ["tree_block", "query_shard", "broadcast_tree_blocks", "grow_trees_distributed",
           "approximate_knn_batch_sharded"]


def tree_block(rank, world, n_trees):
    """[begin, end) of the trees rank ``rank`` of ``world`` builds."""
    return (rank * n_trees) // world, ((rank + 1) * n_trees) // world


def query_shard(rank, world, nq):
    """[begin, end) of the query rows rank ``rank`` answers."""
    return (rank * nq) // world, ((rank + 1) * nq) // world


def broadcast_tree_blocks(arrays, n_trees, group=None):
    """Make every rank's (T, ...) ``arrays`` complete: rank r owns rows
    tree_block(r) and broadcasts them to all others.  Device-agnostic (NCCL
    for CUDA tensors, gloo for CPU tensors); arrays are updated in place."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    for owner in range(world):
        b0, b1 = tree_block(owner, world, n_trees)
        if b1 <= b0:
            continue
        src = owner if group is None else dist.get_global_rank(group, owner)
        for a in arrays:
            dist.broadcast(a[b0:b1], src=src, group=group)
    return arrays


def grow_trees_distributed(X, n_trees, depth, sparsity=None, seed=0, fixed_count=False,
                           group=None, batch_trees=None):
    """grow_trees across the ranks of ``group``: same result on every rank as a
    single-GPU grow_trees with the same arguments (bit-identical arrays).

    Rank r builds its tree block in batches of ``tb`` trees (the smallest
    batch any rank's memory allows, agreed by one all-reduce); as soon as the
    kernels of batch j are enqueued, every rank enqueues the asynchronous
    broadcasts of batch j of every owner (same order on all ranks), so the
    transfer of batch j runs on the communication stream under the build of
    batch j+1.  The sources are never rewritten and the
    destinations are other owners' rows, which the local build never touches."""
    import torch.distributed as dist

    from .trees import _batch_trees

    torch = _device.torch_mod()
    X, sparsity, seed = _validate_grow(X, n_trees, depth, sparsity, seed, None)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    checksum = X.checksum_async()
    dev = X.device().device
    splits, offsets, indices = _alloc_index(n_trees, X.n, depth, dev)
    b0, b1 = tree_block(rank, world, n_trees)
    biggest = max(tree_block(r, world, n_trees)[1] - tree_block(r, world, n_trees)[0]
                  for r in range(world))
    tb = batch_trees or _batch_trees(X.n, X.d, depth, max(1, biggest),
                                     torch.cuda.mem_get_info(dev)[0])
    t = torch.tensor([max(1, min(tb, biggest))], dtype=torch.int64,
                     device=dev if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    tb = int(t.item())
    pending = []
    issued = set()

    def send_batch(j):
        # batch j of every owner (owners with fewer batches skip), in rank order
        for owner in range(world):
            o0, o1 = tree_block(owner, world, n_trees)
            lo, hi = o0 + j * tb, min(o1, o0 + (j + 1) * tb)
            if hi <= lo:
                continue
            src = owner if group is None else dist.get_global_rank(group, owner)
            for a in (splits, offsets, indices):
                pending.append(dist.broadcast(a[lo:hi], src=src, group=group, async_op=True))
        issued.add(j)

    mine = []
    if b1 > b0:
        mine = _grow_block(X, b0, b1, depth, sparsity, seed, fixed_count, splits[b0:b1],
                           offsets[b0:b1], indices[b0:b1], tb, after_batch=send_batch)
    for j in range((biggest + tb - 1) // tb):  # batches this rank does not own
        if j not in issued:
            send_batch(j)
    for w in pending:
        w.wait()
    matrices = []
    for t_ in range(n_trees):
        if b0 <= t_ < b1:
            matrices.append(mine[t_ - b0])
        else:
            matrices.append(sample_sparse_matrix(X.d, depth, sparsity, seed=(seed, t_),
                                                 fixed_count=fixed_count))
    return _finish_index(X, n_trees, depth, sparsity, seed, fixed_count, matrices, splits, offsets,
                         indices, checksum)


def approximate_knn_batch_sharded(Q, k, index, votes, group=None):
    """This rank's shard of a query batch against its replica of the index.
    Returns ((begin, end), ids, dists, candidate_count) -- no collective."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    nq = int(Q.shape[0])
    b0, b1 = query_shard(rank, world, nq)
    part = Q[b0:b1]
    if not _device.is_tensor(part):
        part = np.ascontiguousarray(part)
    return (b0, b1), *approximate_knn_batch(part, k, index, votes)
