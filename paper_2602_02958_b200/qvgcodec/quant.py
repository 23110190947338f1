"""Per-group quantizer, packing, dequantizer (mirrors Q/quant.py:1-168).

Every transform runs on the GPU through libqvg_b200.so; the functions here
check arguments the way the reference does and move bytes in and out.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .. import _lib, device as _d
from . import _dev
from .errors import DimensionMismatch, NonFiniteInput, RangeOverflow, Truncated
from .lowprec import fp8_e4m3_decode_array
from .types import KVPlane, QuantConfig, validate_plane

FP8_ONE = 0x38  # E4M3 1.0, the scale of an all-zero group


@dataclass(frozen=True)
class QuantizedGroup:
    q: np.ndarray
    scale_fp8: int
    bits: int


def _quantize_f64(x: np.ndarray, bits: int, group_size: int):
    """(n, d) float64/float32 matrix -> (payload u8, scales u8) on device."""
    n, d = x.shape
    cfg = QuantConfig(bits=bits, group_size=group_size, stages=0, centroids=1)
    dtype = torch.float32 if x.dtype == np.float32 else torch.float64
    xt = _dev.to_dev(x, dtype).reshape(1, n, d)
    payload, scales = _d.quantize(xt, cfg)
    return _dev.to_host(payload[0]), _dev.to_host(scales[0])


def quantize_group(values, bits: int) -> QuantizedGroup:
    v = np.asarray(values, dtype=np.float64).reshape(1, -1)
    if not np.isfinite(v).all():
        raise NonFiniteInput("group contains NaN or Inf")
    payload, scales = _quantize_f64(v, bits, v.shape[1])
    return QuantizedGroup(q=unpack_payload(payload.tobytes(), v.shape[1], bits),
                          scale_fp8=int(scales[0]), bits=bits)


def dequantize_group(g: QuantizedGroup) -> np.ndarray:
    payload = pack_payload(g.q, g.bits)
    return dequantize_plane(payload, bytes([g.scale_fp8]), 1, len(g.q), g.bits, len(g.q))[0]


def pack_payload(q, bits: int) -> bytes:
    codes = np.asarray(q, dtype=np.int64).ravel()
    qmax = (1 << (bits - 1)) - 1
    if codes.size and (codes.min() < -qmax or codes.max() > qmax):
        raise RangeOverflow(f"code outside symmetric {bits}-bit range")
    if codes.size == 0:
        return b""
    qt = _dev.to_dev(codes.astype(np.int8))
    out = torch.empty((codes.size * bits + 7) // 8, dtype=torch.uint8, device=qt.device)
    st = torch.zeros(1, dtype=torch.int32, device=qt.device)
    lib = _lib.load()
    _lib.check(lib.qvg_pack_codes(_d._ptr(qt), codes.size, bits, _d._ptr(out), _d._ptr(st),
                                  _d._stream(qt.device)))
    _d.check_status(st)
    return _dev.to_host(out).tobytes()


def unpack_payload(data: bytes, count: int, bits: int) -> np.ndarray:
    need = (count * bits + 7) // 8
    if len(data) < need:
        raise Truncated(f"payload has {len(data)} bytes, need {need}")
    if count == 0:
        return np.zeros(0, np.int8)
    raw = _dev.to_dev(np.frombuffer(data, dtype=np.uint8, count=need))
    out = torch.empty(count, dtype=torch.int8, device=raw.device)
    _lib.check(_lib.load().qvg_unpack_codes(_d._ptr(raw), count, bits, _d._ptr(out),
                                            _d._stream(raw.device)))
    return _dev.to_host(out)


def quantize_plane(plane: KVPlane, config: QuantConfig):
    validate_plane(plane, config)
    return quantize_matrix(plane.data, config)


def quantize_matrix(x, config: QuantConfig):
    x = np.asarray(x)
    if x.ndim != 2:
        raise DimensionMismatch("expected an N x d matrix")
    if x.shape[1] % config.group_size:
        raise DimensionMismatch(f"group_size {config.group_size} does not divide width {x.shape[1]}")
    if not np.isfinite(x).all():
        raise NonFiniteInput("matrix contains NaN or Inf")
    if x.dtype != np.float32:
        x = x.astype(np.float64)
    payload, scales = _quantize_f64(x, config.bits, config.group_size)
    return payload.tobytes(), scales.tobytes()


def dequantize_plane(payload: bytes, scales: bytes, n_tokens: int, head_dim: int, bits: int,
                     group_size: int) -> np.ndarray:
    count = n_tokens * head_dim
    need = (count * bits + 7) // 8
    if len(payload) < need:
        raise Truncated(f"payload has {len(payload)} bytes, need {need}")
    n_groups = count // group_size
    if len(scales) < n_groups:
        raise Truncated(f"scales has {len(scales)} bytes, need {n_groups}")
    if count % group_size or head_dim % group_size:
        # layouts the device decoder does not cover: decode the scales on host
        # only to raise the reference's error for NaN patterns, then fail loudly
        fp8_e4m3_decode_array(np.frombuffer(scales, np.uint8, count=n_groups))
        raise DimensionMismatch("group_size must divide head_dim")
    cfg = QuantConfig(bits=bits, group_size=group_size, stages=0, centroids=1)
    dev = _dev.device()
    chunks = _d.DeviceChunks(
        cfg, n_tokens, head_dim,
        payload=_dev.to_dev(np.frombuffer(payload, np.uint8, count=need)).reshape(1, need),
        scales=_dev.to_dev(np.frombuffer(scales, np.uint8, count=n_groups)).reshape(1, n_groups),
        centroids=torch.empty((1, 0, 1, head_dim), dtype=torch.bfloat16, device=dev),
        assignments=torch.empty((1, 0, n_tokens), dtype=torch.uint8, device=dev))
    return _dev.to_host(_d.dequantize(chunks, torch.float32)[0])
