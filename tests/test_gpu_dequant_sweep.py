"""K6 (prq_decompress_onepass, Q/prq.py:113-132) over synthetic compressed
caches, bit-exact against the CPU oracle across the kernel-selection space:
head_dim 128 / 256 (the 32-channel ring kernel), 64 (the 16-channel ring
kernel), odd token counts (the tile kernels),
bits 2 / 4 / 8, S = 1..4 stages, K = 16 / 256 centroids, groups of 32 / 64 /
128, bf16 and f32 outputs, token counts that are not a multiple of a ring
stage.  Inputs are arbitrary valid caches (random code bytes, every non-NaN
E4M3 scale code, centroid rows whose magnitudes span 2^-24..2^12 with zero and
tiny entries), which drives the per-half exactness certificates, the S = 2
swapped-order certificate and the per-element float64 fallback."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.lowprec import round_to_bf16  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402


def _cache(P, N, d, bits, B, S, K, seed):
    rng = np.random.default_rng(seed)
    payload = rng.integers(0, 256, size=(P, N * d * bits // 8), dtype=np.uint8)
    scales = rng.integers(0, 0x7F, size=(P, N * d // B), dtype=np.uint8)          # 0x00..0x7E
    mag = 2.0 ** rng.integers(-24, 13, size=(P, S, K, 1))
    cent = rng.normal(0.0, 1.0, size=(P, S, K, d)) * mag
    cent[rng.random(cent.shape) < 0.02] = 0.0
    cent[rng.random(cent.shape) < 0.01] *= 2.0 ** -30                              # tiny entries
    cent = round_to_bf16(cent.astype(np.float32)).astype(np.float32)
    asg = rng.integers(0, K, size=(P, S, N), dtype=np.uint8)
    return payload, scales, cent, asg


@pytest.mark.parametrize("d", [128, 256, 64])
@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("S", [1, 2, 3, 4])
def test_dequant_sweep_vs_oracle(oracle_lib, d, bits, S):
    for K, B, N in ((16, 32, 1004), (256, 64, 1004), (64, 128, 1004), (16, 64, 1003)):
        if B > d:
            continue
        P = 3
        payload, scales, cent, asg = _cache(P, N, d, bits, B, S, K, seed=d * 1000 + bits * 100 + S * 10 + K % 7)
        cfg = QuantConfig(bits=bits, group_size=B, stages=S, centroids=K)
        cb = torch.from_numpy(cent).to(torch.bfloat16)
        dc = D.DeviceChunks(cfg, N, d, torch.from_numpy(payload).cuda(), torch.from_numpy(scales).cuda(),
                            cb.cuda(), torch.from_numpy(asg).cuda())
        ref = oracle_lib.prq_decompress_batch(payload, scales, cent, asg, N, d, bits, B, 16)
        out32 = D.dequantize(dc, torch.float32).cpu().numpy()
        assert np.array_equal(out32.view(np.uint32), ref.view(np.uint32)), (K, B)
        out16 = D.dequantize(dc, torch.bfloat16).cpu()
        assert torch.equal(out16, torch.from_numpy(ref).to(torch.bfloat16)), (K, B)


@pytest.mark.parametrize("S,K", [(1, 256), (2, 256), (2, 64)])
def test_longcat_tables_codec_vs_oracle(oracle_lib, S, K):
    """LongCat-sized planes (38 400 tokens) with large centroid tables: the
    ring kernels' shared-memory plans at the budget edge (K = 256 tables leave
    few ring stages) -- quantize given the metadata and dequantize, bit-exact."""
    P, N, d, bits, B = 2, 38400, 128, 2, 64
    payload, scales, cent, asg = _cache(P, N, d, bits, B, S, K, seed=77 + S + K)
    cfg = QuantConfig(bits=bits, group_size=B, stages=S, centroids=K)
    cb = torch.from_numpy(cent).to(torch.bfloat16).cuda()
    ag = torch.from_numpy(asg).cuda()
    dc = D.DeviceChunks(cfg, N, d, torch.from_numpy(payload).cuda(), torch.from_numpy(scales).cuda(), cb, ag)
    ref = oracle_lib.prq_decompress_batch(payload, scales, cent, asg, N, d, bits, B, 16)
    out = D.dequantize(dc, torch.float32)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    x = out.to(torch.bfloat16)                                   # any bf16 planes: quantize given the metadata
    pay, sc = D.quantize(x, cfg, cb, ag)
    rp, rs = oracle_lib.quantize_given_metas_batch(x.float().cpu().numpy(), cent, asg, bits, B, 16)
    assert np.array_equal(pay.cpu().numpy(), rp) and np.array_equal(sc.cpu().numpy(), rs)


@pytest.mark.parametrize("d", [128, 256, 64])
@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("S", [0, 1, 2, 3])
def test_quantize_sweep_vs_oracle(oracle_lib, d, bits, S):
    """K5 (quantize given the stage metadata, Q/quant.py:124-148 after
    Q/smoothing.py:40) over every kernel the dispatcher can pick: the
    32-channel ring (S >= 2), the 16-channel ring (S = 1, d = 64), the tile
    kernels (S = 0, odd N), on bf16 planes with outlier channels and tiny
    entries (uncertified lanes, window and exact-scale fallbacks)."""
    rng = np.random.default_rng(d * 100 + bits * 10 + S)
    for K, B, N in ((16, 64, 1004), (64, 32, 1003)):
        if B > d:
            continue
        P = 3
        x = rng.normal(0.0, 2.5, size=(P, N, d))
        x[:, :, ::16] *= 40.0                                          # outlier channels
        x[rng.random(x.shape) < 0.003] *= 2.0 ** -20                   # tiny entries
        x = round_to_bf16(x.astype(np.float32)).astype(np.float32)
        Sc = max(S, 1)
        cent = round_to_bf16((rng.normal(0.0, 2.0, size=(P, Sc, K, d)) *
                              np.where(np.arange(d) % 16 == 0, 30.0, 1.0)).astype(np.float32)).astype(np.float32)
        asg = rng.integers(0, K, size=(P, Sc, N), dtype=np.uint8)
        cent, asg = cent[:, :S], asg[:, :S]
        cfg = QuantConfig(bits=bits, group_size=B, stages=S, centroids=K)
        xd = torch.from_numpy(x).to(torch.bfloat16).cuda()
        pay, sc = D.quantize(xd, cfg, torch.from_numpy(np.ascontiguousarray(cent)).to(torch.bfloat16).cuda(),
                             torch.from_numpy(np.ascontiguousarray(asg)).cuda())
        rp, rs = oracle_lib.quantize_given_metas_batch(x, np.ascontiguousarray(cent), np.ascontiguousarray(asg),
                                                       bits, B, 16)
        assert np.array_equal(sc.cpu().numpy(), rs), (K, B, N)
        assert np.array_equal(pay.cpu().numpy(), rp), (K, B, N)
