"""Deterministic Lloyd k-means (mirrors Q/clustering.py:1-168) on the GPU.

Same RNG (numpy Philox seeded with ``seed``), same float64 operation order,
so centroids, assignments, objective and iteration count are bit-identical
to the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .. import device as _d
from . import _dev
from .errors import DimensionMismatch, EmptyInput


@dataclass(frozen=True)
class KMeansResult:
    centroids: np.ndarray
    assignments: np.ndarray
    objective: float
    iterations_used: int


def _rows(rows) -> np.ndarray:
    r = np.asarray(rows, dtype=np.float64)
    if r.ndim != 2 or r.shape[0] == 0:
        raise EmptyInput("need at least one row")
    return r


def _draws(seed: int, k: int) -> np.ndarray:
    return np.random.Generator(np.random.Philox(seed)).random(k)


def kmeans_pp_init(rows, k: int, seed: int) -> np.ndarray:
    r = _rows(rows)
    if k < 1:
        raise ValueError("k must be >= 1")
    cent = _d.kmeans_pp(_dev.to_dev(r)[None], k, _dev.to_dev(_draws(seed, k))[None])
    return _dev.to_host(cent[0])


def _assign(rows, centroids) -> np.ndarray:
    r = _rows(rows)
    c = np.asarray(centroids, dtype=np.float64)
    return _dev.to_host(_d.assign(_dev.to_dev(r)[None], _dev.to_dev(c)[None])[0]).astype(np.int64)


def lloyd_step(rows, centroids):
    r = _rows(rows)
    c = np.asarray(centroids, dtype=np.float64)
    if r.shape[1] != c.shape[1]:
        raise DimensionMismatch("rows and centroids disagree on d")
    cent, asg, obj = _d.lloyd_step(_dev.to_dev(r)[None], _dev.to_dev(c)[None])
    return _dev.to_host(cent[0]), _dev.to_host(asg[0]).astype(np.int64), float(obj[0].item())


def kmeans(rows, k: int, max_iters: int = 10, tol: float = 1e-4, seed: int = 0,
           init=None) -> KMeansResult:
    r = _rows(rows)
    if not 1 <= k <= 256:
        raise ValueError("k must be in [1, 256] (one-byte assignments)")
    init_t = draws_t = None
    if init is not None:
        c = np.asarray(init, dtype=np.float64)
        if c.ndim != 2 or c.shape != (k, r.shape[1]):
            raise DimensionMismatch(f"init must be ({k}, {r.shape[1]}), got {c.shape}")
        init_t = _dev.to_dev(c)[None]
    else:
        draws_t = _dev.to_dev(_draws(seed, k))[None]
    cent, asg, obj, it = _d.kmeans(_dev.to_dev(r)[None], k, max_iters, tol, draws=draws_t,
                                   init=init_t)
    return KMeansResult(centroids=_dev.to_host(cent[0]), assignments=_dev.to_host(asg[0]),
                        objective=float(obj[0].item()), iterations_used=int(it[0].item()))


def warm_start_from_prev(prev: KMeansResult) -> np.ndarray:
    c = np.asarray(prev.centroids, dtype=np.float64)
    if c.ndim != 2:
        raise DimensionMismatch("previous centroids must be a k x d matrix")
    return c.copy()
