"""ctypes binding of libqvg_b200.so (the C ABI in include/qvg.h).

The product path has no CPU fallback: if the shared library is missing or
cannot be loaded, every entry point raises ``NativeLibraryError``.  Build it
with ``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_2602_02958_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os

from .qvgcodec import errors as _errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QVG_LIB_PATH") or os.path.join(_HERE, "libqvg_b200.so")

# status bits (QVG_STATUS_*)
STATUS_NONFINITE = 1
STATUS_NAN_SCALE = 2
STATUS_BAD_ASSIGN = 4
STATUS_RANGE = 8

DTYPE_F32, DTYPE_BF16, DTYPE_F64 = 0, 1, 2


class NativeLibraryError(RuntimeError):
    """libqvg_b200.so is missing or failed to load (no CPU fallback exists)."""


class QvgConfig(ctypes.Structure):
    _fields_ = [
        ("bits", ctypes.c_int32),
        ("group_size", ctypes.c_int32),
        ("stages", ctypes.c_int32),
        ("centroids", ctypes.c_int32),
        ("kmeans_max_iters", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("kmeans_tol", ctypes.c_double),
        ("seed", ctypes.c_uint64),
    ]

    @classmethod
    def from_config(cls, cfg) -> "QvgConfig":
        return cls(cfg.bits, cfg.group_size, cfg.stages, cfg.centroids, cfg.kmeans_max_iters, 0,
                   float(cfg.kmeans_tol), int(cfg.seed))


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_SZ = ctypes.c_size_t
_D = ctypes.c_double
_CFG = ctypes.POINTER(QvgConfig)

_SIGS = {
    "qvg_abi_version": (_I32, []),
    "qvg_last_error": (ctypes.c_char_p, []),
    "qvg_compress_workspace_size": (_SZ, [_I64, _I64, _I32, _CFG]),
    "qvg_compress": (_I32, [_P, _I32, _I64, _I64, _I32, _CFG, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                            _P, _SZ, _P]),
    "qvg_quantize": (_I32, [_P, _I32, _I64, _I64, _I32, _CFG, _P, _P, _P, _P, _P, _P]),
    "qvg_dequantize": (_I32, [_P, _P, _P, _P, _I64, _I64, _I32, _CFG, _P, _I32, _P, _P]),
    "qvg_pack_codes": (_I32, [_P, _I64, _I32, _P, _P, _P]),
    "qvg_unpack_codes": (_I32, [_P, _I64, _I32, _P, _P]),
    "qvg_kmeans_workspace_size": (_SZ, [_I64, _I64, _I32, _I32]),
    "qvg_kmeanspp": (_I32, [_P, _I64, _I64, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "qvg_assign": (_I32, [_P, _P, _I64, _I64, _I32, _I32, _P, _P]),
    "qvg_lloyd_step": (_I32, [_P, _P, _I64, _I64, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "qvg_kmeans": (_I32, [_P, _I64, _I64, _I32, _I32, _I32, _D, _P, _P, _P, _P, _P, _P, _P, _SZ,
                          _P]),
    "qvg_sa_smoothing_workspace_size": (_SZ, [_I64, _I64, _I32, _I32]),
    "qvg_sa_smoothing": (_I32, [_P, _I64, _I64, _I32, _I32, _I32, _D, _P, _P, _P, _P, _P, _P, _P,
                                _P, _SZ, _P]),
    "qvg_add_back": (_I32, [_P, _P, _P, _I64, _I64, _I32, _I32, _P, _P]),
    "qvg_attention_workspace_size": (_SZ, [_I64, _I64, _I64, _I32, _I32, _CFG]),
    "qvg_attention": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _CFG,
                             ctypes.c_float, _P, _P, _SZ, _P, _P]),
    "qvg_attention_rope": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _CFG,
                                  ctypes.c_float, _P, _P, _I32, _P, _P, _SZ, _P, _P]),
    "qvg_hadamard": (_I32, [_P, _I32, _I64, _I32, _P, _D, _I32, _P, _I32, _P]),
    "qvg_token_transpose": (_I32, [_P, _I32, _I64, _I64, _I64, _I32, _I32, _P, _P]),
    "qvg_record_bytes": (_SZ, [_I64, _I32, _CFG]),
    "qvg_pack_records": (_I32, [_P, _P, _P, _P, _I64, _I64, _I32, _CFG, ctypes.c_uint32, _P, _P]),
    "qvg_unpack_records": (_I32, [_P, _I64, _I64, _I32, _CFG, _P, _P, _P, _P, _P, _P]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and return the native library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not found: build it with `make -C {os.path.join(_HERE, 'csrc')}` "
            "(there is no CPU fallback)")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - depends on the box
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.qvg_abi_version() != 2:
        raise NativeLibraryError("libqvg_b200.so ABI version mismatch")
    _lib = lib
    return lib


_CODE_TO_EXC = {
    1: _errors.DimensionMismatch,
    2: _errors.NonFiniteInput,
    3: _errors.EmptyPlane,
    4: _errors.EmptyInput,
    5: ValueError,
    6: _errors.RangeOverflow,
    7: _errors.Truncated,
    8: _errors.NaNPattern,
    9: RuntimeError,
    10: RuntimeError,
    11: _errors.UnsupportedShape,
}


def check(rc: int) -> None:
    """Map a QVG_ERR_* return code to the reference's exception class."""
    if rc == 0:
        return
    msg = load().qvg_last_error().decode(errors="replace")
    raise _CODE_TO_EXC.get(rc, RuntimeError)(msg or f"qvg error {rc}")


def raise_for_status(word: int) -> None:
    """Map the device status word (after a sync) to exceptions."""
    if word & STATUS_NONFINITE:
        raise _errors.NonFiniteInput("plane contains NaN or Inf")
    if word & STATUS_NAN_SCALE:
        raise _errors.NaNPattern("byte is the E4M3 NaN pattern")
    if word & STATUS_RANGE:
        raise _errors.RangeOverflow("code outside symmetric range")
    if word & STATUS_BAD_ASSIGN:
        raise _errors.DimensionMismatch("assignment index out of centroid range")


def cfg_ptr(cfg) -> ctypes.POINTER(QvgConfig):
    return ctypes.pointer(QvgConfig.from_config(cfg))
