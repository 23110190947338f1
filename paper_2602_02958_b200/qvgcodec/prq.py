"""Progressive Residual Quantization (mirrors Q/prq.py:1-172) on the GPU.

``prq_compress`` is one ``qvg_compress`` call: S stages of SAS (k-means++,
Lloyd, bf16 centroid subtraction) and the per-group quantizer, all in HBM.
Both decoders are one ``qvg_dequantize`` call (the fused one-pass kernel);
they are bit-identical, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .. import device as _d
from . import _dev
from .quant import quantize_matrix
from .smoothing import sa_smoothing
from .types import CompressedChunk, KVPlane, QuantConfig, StageMeta, validate_plane

stage_seed = _d.stage_seed


def _chunk_from_device(spec, config, dc: "_d.DeviceChunks") -> CompressedChunk:
    cent = _dev.to_host(dc.centroids[0].float())
    asg = _dev.to_host(dc.assignments[0])
    metas = tuple(StageMeta(centroids=cent[t], assignments=asg[t]) for t in range(config.stages))
    return CompressedChunk(spec=spec, config=config, payload=_dev.to_host(dc.payload[0]).tobytes(),
                           scales=_dev.to_host(dc.scales[0]).tobytes(), stages=metas)


def prq_compress(plane: KVPlane, config: QuantConfig, warm_init=None) -> CompressedChunk:
    validate_plane(plane, config)
    if warm_init is not None and len(warm_init) != config.stages:
        raise ValueError("warm_init must provide one centroid matrix per stage")
    x = _dev.to_dev(plane.data)[None]
    warm = None
    if warm_init is not None and config.stages:
        warm = _dev.to_dev(np.stack([np.asarray(w, dtype=np.float64) for w in warm_init]))[None]
    dc = _d.compress(x, config, chunk_index=plane.spec.chunk_index, warm_init=warm)
    return _chunk_from_device(plane.spec, config, dc)


def _smoothing_chain(plane: KVPlane, config: QuantConfig, n_stages: int):
    residual = plane.data.astype(np.float64)
    metas = []
    for t in range(1, n_stages + 1):
        residual, meta = sa_smoothing(residual, config.centroids,
                                      seed=stage_seed(config.seed, plane.spec.chunk_index, t),
                                      max_iters=config.kmeans_max_iters, tol=config.kmeans_tol)
        metas.append(meta)
    return residual, metas


def final_residual(plane: KVPlane, config: QuantConfig) -> np.ndarray:
    validate_plane(plane, config)
    return _smoothing_chain(plane, config, config.stages)[0]


def _to_device_chunks(chunk: CompressedChunk) -> "_d.DeviceChunks":
    cfg, n, d = chunk.config, chunk.spec.n_tokens, chunk.spec.head_dim
    dev = _dev.device()
    if cfg.stages:
        cent = np.stack([m.centroids for m in chunk.stages])[None]
        asg = np.stack([m.assignments for m in chunk.stages])[None]
        cent_t = _dev.to_dev(cent, torch.bfloat16)
        asg_t = _dev.to_dev(asg)
    else:
        cent_t = torch.empty((1, 0, cfg.centroids, d), dtype=torch.bfloat16, device=dev)
        asg_t = torch.empty((1, 0, n), dtype=torch.uint8, device=dev)
    return _d.DeviceChunks(cfg, n, d,
                           payload=_dev.to_dev(np.frombuffer(chunk.payload, np.uint8))[None],
                           scales=_dev.to_dev(np.frombuffer(chunk.scales, np.uint8))[None],
                           centroids=cent_t, assignments=asg_t)


def prq_decompress(chunk: CompressedChunk) -> KVPlane:
    out = _d.dequantize(_to_device_chunks(chunk), torch.float32)
    return KVPlane(spec=chunk.spec, data=_dev.to_host(out[0]))


@dataclass
class DecodeCounters:
    payload_reads: int = 0
    centroid_lookups_per_token: int = 0
    tokens: int = 0


def prq_decompress_onepass(chunk: CompressedChunk, counters: DecodeCounters = None) -> KVPlane:
    plane = prq_decompress(chunk)           # the device decoder is already one pass
    if counters is not None:
        counters.payload_reads = 1
        counters.centroid_lookups_per_token = len(chunk.stages)
        counters.tokens = chunk.spec.n_tokens
    return plane


def stage_mse_curve(plane: KVPlane, config: QuantConfig, max_stages: int) -> list:
    """MSE of compress->decompress for S = 0..max_stages, extending one chain."""
    validate_plane(plane, config)
    original = plane.data.astype(np.float64)
    residual = plane.data.astype(np.float64)
    metas = []
    curve = []
    for s in range(max_stages + 1):
        if s:
            residual, meta = sa_smoothing(residual, config.centroids,
                                          seed=stage_seed(config.seed, plane.spec.chunk_index, s),
                                          max_iters=config.kmeans_max_iters, tol=config.kmeans_tol)
            metas.append(meta)
        cfg_s = config.with_stages(s)
        payload, scales = quantize_matrix(residual, cfg_s)
        chunk = CompressedChunk(spec=plane.spec, config=cfg_s, payload=payload, scales=scales,
                                stages=tuple(metas))
        recon = prq_decompress(chunk).data.astype(np.float64)
        curve.append(float(np.mean((original - recon) ** 2)))
    return curve
