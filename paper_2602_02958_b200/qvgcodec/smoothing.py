"""Semantic-Aware Smoothing (mirrors Q/smoothing.py:1-54) on the GPU."""

from __future__ import annotations

import numpy as np
import torch

from .. import device as _d
from . import _dev
from .errors import DimensionMismatch
from .types import StageMeta


def sa_smoothing(x, k: int, seed: int, warm_init=None, max_iters: int = 10, tol: float = 1e-4):
    """-> (float64 residual x - C_bf16[pi], StageMeta)."""
    xs = np.asarray(x, dtype=np.float64)
    xt = _dev.to_dev(xs)[None]
    if warm_init is not None:
        w = np.asarray(warm_init, dtype=np.float64)
        if w.ndim != 2 or w.shape != (k, xs.shape[1]):
            raise DimensionMismatch(f"init must be ({k}, {xs.shape[1]}), got {w.shape}")
        res, cb, asg, _, _ = _d.sa_smoothing(xt, k, warm_init=_dev.to_dev(w)[None],
                                              max_iters=max_iters, tol=tol)
    else:
        if not 1 <= k <= 256:
            raise ValueError("k must be in [1, 256] (one-byte assignments)")
        draws = np.random.Generator(np.random.Philox(seed)).random(k)
        res, cb, asg, _, _ = _d.sa_smoothing(xt, k, draws=_dev.to_dev(draws)[None],
                                              max_iters=max_iters, tol=tol)
    cent = _dev.to_host(cb[0].float())
    return _dev.to_host(res[0]), StageMeta(centroids=cent, assignments=_dev.to_host(asg[0]))


def add_back(residual, meta: StageMeta) -> np.ndarray:
    r = np.asarray(residual, dtype=np.float64)
    if r.ndim != 2:
        raise DimensionMismatch("residual must be an N x d matrix")
    if meta.assignments.shape[0] != r.shape[0]:
        raise DimensionMismatch("assignment count != residual rows")
    if meta.centroids.shape[1] != r.shape[1]:
        raise DimensionMismatch("centroid width != residual width")
    out = _d.add_back(_dev.to_dev(r)[None], _dev.to_dev(meta.centroids, torch.bfloat16)[None],
                      _dev.to_dev(meta.assignments)[None])
    return _dev.to_host(out[0])
