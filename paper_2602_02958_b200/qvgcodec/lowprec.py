"""FP8 E4M3 and bf16 format helpers (mirrors Q/lowprec.py:1-132).

Host-side format utilities (the in-kernel versions live in csrc/); the
encoder works by position on the monotone table of non-negative E4M3
values: "up" = first grid value >= x, "nearest" = closer neighbour with
ties to the even code (even code == even mantissa).
"""

from __future__ import annotations

import numpy as np

from .errors import NaNPattern, NonFiniteScale

E4M3_MAX = 448.0
E4M3_MIN_SUBNORMAL = 2.0 ** -9
E4M3_NAN_BYTES = (0x7F, 0xFF)


def _value_of(code: int) -> float:
    e, m = (code >> 3) & 0xF, code & 7
    if e == 0xF and m == 7:
        return float("nan")
    mag = m * E4M3_MIN_SUBNORMAL if e == 0 else (8 + m) * 2.0 ** (e - 10)
    return -mag if code & 0x80 else mag


_TABLE = np.array([_value_of(c) for c in range(256)], dtype=np.float64)
_GRID = _TABLE[:0x7F]          # codes 0x00..0x7E, strictly increasing values


def fp8_e4m3_encode_array(x, rounding: str = "nearest") -> np.ndarray:
    if rounding not in ("nearest", "up"):
        raise ValueError(f"unknown rounding mode {rounding!r}")
    x = np.asarray(x, dtype=np.float64)
    if not np.isfinite(x).all():
        raise NonFiniteScale("scale must be finite")
    if (x < 0).any():
        raise ValueError("scale must be non-negative")
    x = np.minimum(x, E4M3_MAX)
    if rounding == "up":
        code = np.searchsorted(_GRID, x, side="left")
    else:
        lo = np.searchsorted(_GRID, x, side="right") - 1
        hi = np.minimum(lo + 1, 0x7E)
        mid = (_GRID[lo] + _GRID[hi]) / 2.0          # exact: few significant bits
        code = np.where(x < mid, lo, np.where(x > mid, hi, np.where(lo % 2 == 0, lo, hi)))
        code = np.where(x == _GRID[lo], lo, code)
    return np.minimum(code, 0x7E).astype(np.uint8)


def fp8_e4m3_decode_array(codes) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.uint8)
    if np.isin(codes, E4M3_NAN_BYTES).any():
        raise NaNPattern("byte is the E4M3 NaN pattern")
    return _TABLE[codes]


def fp8_e4m3_encode(x: float, rounding: str = "nearest") -> int:
    return int(fp8_e4m3_encode_array(np.array([x]), rounding)[0])


def fp8_e4m3_decode(byte: int) -> float:
    if not 0 <= byte <= 255:
        raise ValueError("byte out of range")
    return float(fp8_e4m3_decode_array(np.array([byte], dtype=np.uint8))[0])


def round_to_bf16(a) -> np.ndarray:
    """float32 -> nearest bf16 (ties to even), kept in float32 storage."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    bias = np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    return ((u + bias) & np.uint32(0xFFFF0000)).astype(np.uint32).view(np.float32)


def bf16_pack(a) -> np.ndarray:
    return (np.ascontiguousarray(a, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def bf16_unpack(u) -> np.ndarray:
    return (np.asarray(u, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)
