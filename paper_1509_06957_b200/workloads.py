"""Seeded synthetic stand-ins for the five BASELINE.json configurations.

The reference measures nothing at these sizes and ships no data; these
generators pin the interpretation of BASELINE.json's config text that
SURVEY.md section 8(d) describes (all fp32, ``numpy.random.default_rng(seed)``,
data and queries drawn from the same distribution, data first).  Configs
3-5 are generated in 65,536-row chunks, chunk i from its own stream
``default_rng([seed, config, i])`` on a thread pool, so 10M rows take seconds
and the rows do not depend on the thread count.  ``scale``
shrinks n and the query count proportionally for tests; T, depth, a, k and v
are the configuration's own (depth is clamped so 2^depth <= n).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    nq: int
    d: int
    n_trees: int
    depth: int
    sparsity: float
    k: int
    votes: tuple
    headline_votes: int
    generator: str
    notes: str = ""
    extra: dict = field(default_factory=dict)


CONFIGS = {
    1: Workload("config1-gaussian-mixture", 10_000, 1_000, 128, 16, 7, 1 / math.sqrt(128), 10,
                (1, 2, 3, 4), 2,
                "32 clusters, centres 4*N(0,1) (i.e. N(0,16 I)), points centre+N(0,1)"),
    2: Workload("config2-image-pixels", 60_000, 10_000, 784, 100, 8, 1 / math.sqrt(784), 10,
                (1, 2, 4, 8), 1,
                "28x28; per point Gaussian blob centre (13.5,13.5)+N(0,2^2), sigma~U(4,8); "
                "nonzero prob ~ blob scaled to mean 0.2, clipped to 1; nonzero ~ U(0,1)"),
    3: Workload("config3-local-descriptors", 1_000_000, 10_000, 128, 200, 11, 1 / math.sqrt(128),
                10, (1, 2, 3, 4, 5, 6, 7, 8), 1,
                "min(255, floor(Exp(mean 20))) iid, exactly 13 = ceil(0.1*128) coords per "
                "vector zeroed"),
    4: Workload("config4-global-descriptors", 1_000_000, 1_000, 960, 500, 10, 1 / math.sqrt(960),
                10, (2, 5, 10), 10,
                "256 centres U[0,0.5]^960, sigma 0.05, clipped to [0,1]"),
    5: Workload("config5-scale-out", 10_000_000, 100_000, 256, 1000, 13, 1 / 16, 100, (10,), 10,
                "1024 centres 3*N(0,1) (N(0,9 I)), sigma 1"),
}

_CHUNK = 65_536


def _parallel_rows(count, d, seed, tag, fill):
    """(count, d) float32 rows made chunk by chunk, chunk i from its own stream
    default_rng([seed, tag, i]), on a thread pool (numpy's generators release
    the GIL while filling): the result does not depend on the thread count."""
    out = np.empty((count, d), dtype=np.float32)
    bounds = [(i, s, min(count, s + _CHUNK)) for i, s in enumerate(range(0, count, _CHUNK))]

    def job(b):
        i, s, e = b
        out[s:e] = fill(np.random.default_rng([seed, tag, i]), e - s)

    workers = max(1, min(32, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
                         else (os.cpu_count() or 1)))
    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(job, bounds))
    return out


def _mixture_fill(centres, sigma):
    c32 = centres.astype(np.float32)

    def fill(rng, m):
        lab = rng.integers(0, c32.shape[0], size=m)
        noise = rng.standard_normal((m, c32.shape[1]), dtype=np.float32)
        noise *= np.float32(sigma)
        noise += c32[lab]
        return noise

    return fill


def _descriptor_fill(d, zeros):
    def fill(rng, m):
        x = np.minimum(255.0, np.floor(rng.exponential(20.0, size=(m, d))))
        kill = np.argsort(rng.random((m, d)), axis=1)[:, :zeros]
        np.put_along_axis(x, kill, 0.0, axis=1)
        return x

    return fill


def _gaussian_mixture(rng, count, centres, sigma):
    out = np.empty((count, centres.shape[1]), dtype=np.float32)
    for s in range(0, count, _CHUNK):
        e = min(count, s + _CHUNK)
        lab = rng.integers(0, centres.shape[0], size=e - s)
        out[s:e] = centres[lab] + sigma * rng.standard_normal((e - s, centres.shape[1]))
    return out


def _blobs(rng, count):
    yy, xx = np.mgrid[0:28, 0:28].astype(np.float64)
    out = np.empty((count, 784), dtype=np.float32)
    for s in range(0, count, 8192):
        e = min(count, s + 8192)
        m = e - s
        c = 13.5 + 2.0 * rng.standard_normal((m, 2))
        sig = rng.uniform(4.0, 8.0, size=m)
        blob = np.exp(-((yy[None] - c[:, 0, None, None]) ** 2 + (xx[None] - c[:, 1, None, None]) ** 2)
                      / (2 * sig[:, None, None] ** 2)).reshape(m, 784)
        p = np.minimum(1.0, blob * (0.2 / blob.mean(axis=1, keepdims=True)))
        nz = rng.random((m, 784)) < p
        out[s:e] = np.where(nz, rng.random((m, 784)), 0.0)
    return out


def generate(config, scale=1.0, seed=0):
    """(X, Q, params) for a configuration; params mirrors grow_trees/query args."""
    w = CONFIGS[config]
    n = max(2, int(round(w.n * scale)))
    nq = max(1, int(round(w.nq * scale)))
    depth = min(w.depth, int(math.floor(math.log2(n))))
    rng = np.random.default_rng(seed)
    total = n + nq
    if config == 1:
        centres = 4.0 * rng.standard_normal((32, w.d))
        allx = _gaussian_mixture(rng, total, centres, 1.0)
    elif config == 2:
        allx = _blobs(rng, total)
    elif config == 3:
        allx = _parallel_rows(total, w.d, seed, 3, _descriptor_fill(w.d, math.ceil(0.1 * w.d)))
    elif config == 4:
        centres = rng.uniform(0.0, 0.5, size=(256, w.d))
        allx = _parallel_rows(total, w.d, seed, 4, _mixture_fill(centres, 0.05))
        np.clip(allx, 0.0, 1.0, out=allx)
    elif config == 5:
        centres = 3.0 * rng.standard_normal((1024, w.d))
        allx = _parallel_rows(total, w.d, seed, 5, _mixture_fill(centres, 1.0))
    else:
        raise KeyError(config)
    X = np.ascontiguousarray(allx[:n])
    Q = np.ascontiguousarray(allx[n:])
    params = dict(n_trees=w.n_trees, depth=depth, sparsity=w.sparsity, k=w.k, votes=w.votes,
                  headline_votes=w.headline_votes, seed=0, name=w.name, n=n, nq=nq, d=w.d,
                  generator=w.generator)
    return X, Q, params
