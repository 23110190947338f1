"""Host-side pieces of the drop-in API that run without a GPU: FP8/bf16
format helpers (against the reference's own known answers and the
reference-generated fixtures), value types, error classes, accounting."""
import math

import numpy as np
import pytest

from golden_io import load_kat
from paper_2602_02958_b200.qvgcodec import errors, lowprec, metrics
from paper_2602_02958_b200.qvgcodec.types import (ChunkSpec, CompressedChunk, KVPlane,
                                                  QuantConfig, StageMeta, validate_plane)


@pytest.mark.parametrize("value,byte", [(0.0, 0x00), (1.0, 0x38), (448.0, 0x7E),
                                        (2.0 ** -9, 0x01), (0.015625, 0x08), (3.0, 0x44)])
def test_fp8_exact_values(value, byte):
    assert lowprec.fp8_e4m3_encode(value, "nearest") == byte
    assert lowprec.fp8_e4m3_encode(value, "up") == byte


def test_fp8_rounding_cases():
    assert lowprec.fp8_e4m3_decode(lowprec.fp8_e4m3_encode(1 / 7, "nearest")) == 0.140625
    assert lowprec.fp8_e4m3_decode(lowprec.fp8_e4m3_encode(1 / 7, "up")) == 0.15625
    assert lowprec.fp8_e4m3_encode(1000.0, "up") == 0x7E
    assert lowprec.fp8_e4m3_encode(1e-9, "up") == 0x01
    assert lowprec.fp8_e4m3_encode(2.0 ** -10, "nearest") == 0x00
    assert lowprec.fp8_e4m3_decode(0xB8) == -1.0
    for bad in (0x7F, 0xFF):
        with pytest.raises(errors.NaNPattern):
            lowprec.fp8_e4m3_decode(bad)
    with pytest.raises(errors.NonFiniteScale):
        lowprec.fp8_e4m3_encode(float("nan"))
    with pytest.raises(ValueError):
        lowprec.fp8_e4m3_encode(-1.0)


def test_fp8_encode_matches_reference_fixture():
    kat = load_kat()
    assert np.array_equal(lowprec.fp8_e4m3_encode_array(kat["fp8_x"], "up"), kat["fp8_up"])
    assert np.array_equal(lowprec.fp8_e4m3_encode_array(kat["fp8_x"], "nearest"), kat["fp8_nearest"])


def test_fp8_identity_on_all_codes():
    for code in range(0x7F):
        v = lowprec.fp8_e4m3_decode(code)
        assert lowprec.fp8_e4m3_encode(v, "nearest") == code == lowprec.fp8_e4m3_encode(v, "up")


def test_bf16_helpers_match_reference_fixture():
    kat = load_kat()
    assert np.array_equal(lowprec.round_to_bf16(kat["bf16_in"]).view(np.uint32),
                          kat["bf16_out"].view(np.uint32))
    a = lowprec.round_to_bf16(np.random.default_rng(4).normal(scale=100.0, size=4096).astype(np.float32))
    assert np.array_equal(lowprec.bf16_unpack(lowprec.bf16_pack(a)), a)
    assert lowprec.round_to_bf16(np.float32(1.0 + 2.0 ** -8))[()] == np.float32(1.0)


def test_config_validation():
    for bad in (dict(bits=3), dict(group_size=0), dict(stages=-1), dict(centroids=0),
                dict(centroids=257), dict(kmeans_max_iters=0), dict(kmeans_tol=-1.0), dict(seed=-1)):
        with pytest.raises(ValueError):
            QuantConfig(**bad)
    assert QuantConfig(bits=4).qmax == 7
    assert QuantConfig().with_stages(3).stages == 3


def test_types_and_validate_plane():
    with pytest.raises(errors.EmptyPlane):
        ChunkSpec(n_tokens=0, head_dim=4)
    with pytest.raises(errors.DimensionMismatch):
        KVPlane(spec=ChunkSpec(4, 8), data=np.zeros((4, 9)))
    p = KVPlane.from_array(np.zeros((4, 100), np.float32))
    with pytest.raises(errors.DimensionMismatch):
        validate_plane(p, QuantConfig(group_size=64))
    d = np.zeros((4, 64), np.float32)
    d[2, 3] = np.nan
    with pytest.raises(errors.NonFiniteInput):
        validate_plane(KVPlane.from_array(d), QuantConfig())
    assert not p.data.flags.writeable
    m = StageMeta(centroids=np.zeros((4, 8)), assignments=np.array([0, 3, 1]))
    with pytest.raises(errors.DimensionMismatch):
        StageMeta(centroids=np.zeros((4, 8)), assignments=np.array([4]))
    cfg = QuantConfig(bits=2, group_size=8, stages=1, centroids=4)
    ok = CompressedChunk(ChunkSpec(3, 8), cfg, bytes(6), bytes(3), (m,))
    assert len(ok.stages) == 1
    with pytest.raises(errors.DimensionMismatch):
        CompressedChunk(ChunkSpec(3, 8), cfg, bytes(5), bytes(3), (m,))


def test_error_class_tree():
    assert issubclass(errors.DimensionMismatch, errors.CodecError)
    assert issubclass(errors.DimensionMismatch, ValueError)
    assert issubclass(errors.OutOfRange, IndexError)


def test_memory_breakdown_matches_paper_accounting():
    # config 1 (N 4680, b2 B64 S2 K64) 5.953x; QVG INT2 / QVG-Pro at N=38400
    r = metrics.memory_breakdown(QuantConfig(bits=2, group_size=64, stages=2, centroids=64),
                                 ChunkSpec(4680, 128)).ratio_vs_bf16
    assert round(r, 3) == 5.953
    r = metrics.memory_breakdown(QuantConfig(bits=2, group_size=64, stages=1, centroids=256),
                                 ChunkSpec(38400, 128)).ratio_vs_bf16
    assert round(r, 3) == 6.974
    r = metrics.memory_breakdown(QuantConfig(bits=2, group_size=16, stages=0, centroids=1),
                                 ChunkSpec(38400, 128)).ratio_vs_bf16
    assert r == 6.4
    fr = metrics.breakdown_fractions(metrics.memory_breakdown(QuantConfig(), ChunkSpec(100, 128)))
    assert math.isclose(sum(fr.values()), 1.0)
    assert metrics.psnr(np.zeros(3), np.zeros(3)) == metrics.PSNR_INF


def test_nvtx_wrappers_opt_in():
    """QVG_NVTX=1 wraps the device entry points in NVTX ranges (tracing hook);
    without it the functions are the plain ones."""
    import subprocess
    import sys
    code = ("import paper_2602_02958_b200.device as D; "
            "print(int(all(hasattr(getattr(D, n), '__wrapped__') for n in "
            "('compress', 'quantize', 'dequantize', 'attention'))))")
    env = dict(__import__("os").environ, QVG_NVTX="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert out.stdout.strip() == "1", out.stderr
    env.pop("QVG_NVTX")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert out.stdout.strip() == "0", out.stderr
