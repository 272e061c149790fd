"""Ground truth and recall on the GPU (mirrors pkg/src/mrpt/evaluation.py:28-100).

``brute_force_knn`` / ``compute_ground_truth`` keep the reference's
signatures, validation order, errors and results: the exact k nearest
neighbours by a scan of the whole dataset, ascending distance, ties by
ascending id.  The scan is the f3 kernel (``mrpt_brute_force_knn``,
``csrc/gt.cu``): every squared distance is summed in numpy's pairwise order
from float64 differences, exactly like the reference's
``((X - q) ** 2).sum(axis=1)`` (evaluation.py:40-41), so ids and float64
distances are bit-identical to the reference's -- the recall of every
configuration rests on this tested path.  ``recall`` is host bookkeeping
with the reference's semantics (evaluation.py:84-100).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device, _native
from .core import as_dataset
from .exceptions import ParameterError, ShapeError
from .search import NeighborList

__all__ = ["GroundTruth", "brute_force_knn", "compute_ground_truth", "recall"]

_QUERY_CHUNK = 16384


def _knn_device(Xd, Qd64, k):
    """(ids, dists) CUDA tensors (nq, min(k, n)) of the exact k-NN of every
    float64 query row against the float32 rows of Xd."""
    torch = _device.torch_mod()
    n, d = int(Xd.shape[0]), int(Xd.shape[1])
    nq = int(Qd64.shape[0])
    kk = min(int(k), n)
    ids = torch.empty((nq, kk), dtype=torch.int64, device=Xd.device)
    dists = torch.empty((nq, kk), dtype=torch.float64, device=Xd.device)
    for s in range(0, nq, _QUERY_CHUNK):
        e = min(nq, s + _QUERY_CHUNK)
        need = ctypes.c_int64(0)
        _native.call("mrpt_brute_force_workspace_size", n, d, e - s, int(k), ctypes.byref(need))
        ws = torch.empty(max(1, need.value), dtype=torch.uint8, device=Xd.device)
        _native.call("mrpt_brute_force_knn", _native.ptr(Xd), n, d, int(Xd.stride(0)),
                     _native.ptr(Qd64[s:e]), e - s, int(Qd64.stride(0)), int(k),
                     _native.ptr(ids[s:e]), _native.ptr(dists[s:e]), _native.ptr(ws),
                     int(ws.numel()), _native.stream_ptr())
    return ids, dists


def brute_force_knn(q, k, X):
    """Exact k-NN by scanning the whole dataset (evaluation.py:28-47).

    Ascending distance, ties broken by ascending point index; returns
    min(k, n) neighbours.
    """
    if k < 1:
        raise ParameterError(f"k must be >= 1, got {k}")
    X = as_dataset(X)
    qv = np.asarray(q, dtype=np.float64).ravel()
    if qv.shape[0] != X.d:
        raise ShapeError(f"query has length {qv.shape[0]}, expected {X.d}")
    ids, dists = _knn_device(X.device(), _device.h2d(qv.reshape(1, -1)), k)
    return NeighborList(indices=_device.d2h(ids)[0], distances=_device.d2h(dists)[0],
                        requested_k=k, candidate_count=X.n)


@dataclass(frozen=True)
class GroundTruth:
    """Exact k nearest neighbours of each query, from brute force only
    (evaluation.py:50-62)."""

    k: int
    indices: np.ndarray  # int64, (n_queries, k)
    distances: np.ndarray  # float64, (n_queries, k)
    dataset_checksum: int
    query_checksum: int

    @property
    def n_queries(self):
        return self.indices.shape[0]


def compute_ground_truth(X, queries, k):
    """Ground truth of every query row (evaluation.py:65-81), one batched
    device scan instead of one brute-force call per query."""
    X = as_dataset(X)
    queries = as_dataset(queries)
    if X.d != queries.d:
        raise ShapeError(f"queries have d={queries.d} but dataset has d={X.d}")
    if not 1 <= k <= X.n:
        raise ParameterError(f"k must lie in [1, {X.n}], got {k}")
    torch = _device.torch_mod()
    Q64 = queries.device().to(torch.float64)  # float32 -> float64 is exact
    ids, dists = _knn_device(X.device(), Q64, k)
    return GroundTruth(k=k, indices=_device.d2h(ids), distances=_device.d2h(dists),
                       dataset_checksum=X.checksum, query_checksum=queries.checksum)


def recall(result, truth):
    """Fraction of the true k nearest neighbours present in ``result``
    (evaluation.py:84-100): ``truth`` holds exactly k distinct ids (an array
    or a NeighborList); distances are ignored."""
    true_ids = truth.indices if isinstance(truth, NeighborList) else np.asarray(truth)
    true_ids = np.asarray(true_ids, dtype=np.int64).ravel()
    k = true_ids.shape[0]
    if k < 1:
        raise ParameterError("ground truth entry must contain at least one neighbor")
    if np.unique(true_ids).shape[0] != k:
        raise ParameterError("ground truth entry contains duplicate indices")
    got = result.indices if isinstance(result, NeighborList) else np.asarray(result)
    got = np.asarray(got, dtype=np.int64).ravel()
    return float(np.intersect1d(got, true_ids).shape[0] / k)


def recall_batch(ids, truth_ids):
    """Mean recall of a batch: row i of ``ids`` (padded with -1) against row i
    of ``truth_ids``; the batched form of ``recall``."""
    ids = np.asarray(ids, dtype=np.int64)
    truth_ids = np.asarray(truth_ids, dtype=np.int64)
    if ids.shape[0] != truth_ids.shape[0]:
        raise ShapeError(f"{ids.shape[0]} results for {truth_ids.shape[0]} ground-truth rows")
    if ids.shape[0] == 0:
        return 0.0
    return float(np.mean([recall(a[a >= 0], b) for a, b in zip(ids, truth_ids)]))
