"""The C-ABI library loads, exports every symbol include/qvg.h declares, and
rejects bad arguments with the right codes before touching a GPU."""
import ctypes
import os
import re

import pytest

from paper_2602_02958_b200 import _lib
from paper_2602_02958_b200.qvgcodec import errors
from paper_2602_02958_b200.qvgcodec.types import QuantConfig

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "qvg.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"QVG_API\s+[\w\s\*]*?\b(qvg_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared_symbols()
    for want in ("qvg_compress", "qvg_quantize", "qvg_dequantize", "qvg_attention",
                 "qvg_kmeans", "qvg_sa_smoothing", "qvg_last_error", "qvg_abi_version"):
        assert want in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_lib.EXPORTED)
    assert lib.qvg_abi_version() == 2


def _cfg(**kw):
    base = dict(bits=2, group_size=64, stages=1, centroids=16)
    base.update(kw)
    return _lib.QvgConfig(base["bits"], base["group_size"], base["stages"], base["centroids"],
                          base.get("kmeans_max_iters", 10), 0, base.get("kmeans_tol", 1e-4), 0)


@pytest.mark.parametrize("kw,N,d,code,exc", [
    (dict(bits=3), 16, 128, 5, ValueError),
    (dict(group_size=48), 16, 128, 1, errors.DimensionMismatch),
    (dict(centroids=300), 16, 128, 5, ValueError),
    (dict(), 0, 128, 3, errors.EmptyPlane),
    (dict(stages=1), 16, 256, 11, errors.UnsupportedShape),
])
def test_compress_argument_errors(kw, N, d, code, exc):
    lib = _lib.load()
    cfg = _cfg(**kw)
    rc = lib.qvg_compress(None, 1, 1, N, d, ctypes.byref(cfg), None, None, None, None, None, None,
                          None, None, None, None, 0, None)
    assert rc == code
    assert lib.qvg_last_error()
    with pytest.raises(exc):
        _lib.check(rc)


def test_dequantize_and_quantize_argument_errors():
    lib = _lib.load()
    cfg = _cfg(group_size=48)
    assert lib.qvg_dequantize(None, None, None, None, 1, 4, 128, ctypes.byref(cfg), None, 1, None,
                              None) == 1
    assert lib.qvg_quantize(None, 7, 1, 4, 128, ctypes.byref(_cfg()), None, None, None, None, None,
                            None) == 5
    assert lib.qvg_pack_codes(None, 4, 3, None, None, None) == 5


def test_workspace_sizes_are_positive_and_monotone():
    lib = _lib.load()
    cfg = _cfg(centroids=64, stages=2)
    small = lib.qvg_compress_workspace_size(1, 4680, 128, ctypes.byref(cfg))
    big = lib.qvg_compress_workspace_size(24, 4680, 128, ctypes.byref(cfg))
    assert 0 < small < big
    assert lib.qvg_kmeans_workspace_size(2, 1000, 64, 32) > 0


def test_config_struct_layout_matches_header():
    assert ctypes.sizeof(_lib.QvgConfig) == 40
    c = _lib.QvgConfig.from_config(QuantConfig(bits=4, group_size=16, stages=3, centroids=7, seed=9))
    assert (c.bits, c.group_size, c.stages, c.centroids, c.seed) == (4, 16, 3, 7, 9)
