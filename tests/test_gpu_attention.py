"""Attention over the quantized cache vs the fp64 CPU oracle
(oracle/qvg_oracle.c:qo_attention over the oracle's own dequantized cache).

Tolerance: max-abs <= 2e-2 * max|O_ref| and rel-L2 <= 1e-2
(bf16 operands / P, fp32 accumulation)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402
from paper_2602_02958_b200.synth import clustered_planes  # noqa: E402

ATOL_REL, RL2 = 2e-2, 1e-2


def _check(out, ref):
    out = out.float().cpu().numpy().astype(np.float64)
    err = np.abs(out - ref)
    scale = np.abs(ref).max()
    rel_l2 = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    assert err.max() <= ATOL_REL * scale, (err.max(), scale)
    assert rel_l2 <= RL2, rel_l2
    return err.max() / scale, rel_l2


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("H,nq,nc,ncur,cfg", [
    (2, 200, 300, 150, dict(bits=2, group_size=64, stages=2, centroids=16)),
    (1, 128, 256, 128, dict(bits=4, group_size=16, stages=1, centroids=32)),
    (3, 70, 129, 0, dict(bits=2, group_size=64, stages=1, centroids=8)),
    (2, 130, 0, 200, dict(bits=2, group_size=64, stages=2, centroids=8)),
])
def test_quantized_attention_vs_oracle(oracle_lib, H, nq, nc, ncur, cfg, fused):
    torch.manual_seed(0)
    cfg = QuantConfig(**cfg)
    d = 128
    q = (torch.randn(nq, H, d, device="cuda") * 0.5).to(torch.bfloat16)
    kc = torch.randn(ncur, H, d, device="cuda").to(torch.bfloat16)
    vc = torch.randn(ncur, H, d, device="cuda").to(torch.bfloat16)
    scale = d ** -0.5
    if nc:
        planes = clustered_planes(2 * H, nc, d, n_clusters=16, outlier_scale=4.0, seed=1)
        chunks = D.compress(planes, cfg)
        out = D.attention(q, chunks, kc, vc, scale, fused=fused)
        deq = oracle_lib.prq_decompress_batch(chunks.payload.cpu().numpy(), chunks.scales.cpu().numpy(),
                                              chunks.centroids.float().cpu().numpy(),
                                              chunks.assignments.cpu().numpy(), nc, d, cfg.bits,
                                              cfg.group_size, 8)
        kcache, vcache = deq[0::2], deq[1::2]
    else:
        out = D.attention(q, None, kc, vc, scale)
        kcache = vcache = np.zeros((H, 0, d), np.float32)
    torch.cuda.synchronize()
    ref = oracle_lib.attention(q.float().cpu().numpy(), kcache, vcache, kc.float().cpu().numpy(),
                               vc.float().cpu().numpy(), scale, 8)
    _check(out, ref)


def test_bf16_cache_mode_vs_oracle(oracle_lib):
    torch.manual_seed(1)
    H, nq, nc, ncur, d = 2, 256, 384, 128, 128
    q = torch.randn(nq, H, d, device="cuda").to(torch.bfloat16)
    kv = torch.randn(2 * H, nc, d, device="cuda").to(torch.bfloat16)
    kc = torch.randn(ncur, H, d, device="cuda").to(torch.bfloat16)
    vc = torch.randn(ncur, H, d, device="cuda").to(torch.bfloat16)
    out = D.attention(q, None, kc, vc, d ** -0.5, kv_bf16=kv)
    torch.cuda.synchronize()
    kvf = kv.float().cpu().numpy()
    ref = oracle_lib.attention(q.float().cpu().numpy(), kvf[0::2], kvf[1::2], kc.float().cpu().numpy(),
                               vc.float().cpu().numpy(), d ** -0.5, 8)
    _check(out, ref)
    # and against torch SDPA on the same bf16 data (library comparator)
    k_all = torch.cat([kv[0::2].permute(1, 0, 2), kc], 0)      # [nkv, H, d]
    v_all = torch.cat([kv[1::2].permute(1, 0, 2), vc], 0)
    sd = torch.nn.functional.scaled_dot_product_attention(
        q.permute(1, 0, 2)[None].float(), k_all.permute(1, 0, 2)[None].float(),
        v_all.permute(1, 0, 2)[None].float())[0].permute(1, 0, 2)
    assert torch.allclose(out.float(), sd, atol=2e-2 * sd.abs().max().item())


def test_attention_long_cache_online_softmax(oracle_lib):
    """Many KV blocks with a growing score range: exercises the lazy rescale."""
    torch.manual_seed(2)
    H, nq, nc, ncur, d = 1, 128, 2048, 64, 128
    q = torch.randn(nq, H, d, device="cuda").to(torch.bfloat16)
    kv = torch.randn(2 * H, nc, d, device="cuda")
    kv[0] *= torch.linspace(0.2, 3.0, nc, device="cuda")[:, None]      # scores grow along the cache
    kv = kv.to(torch.bfloat16)
    kc = torch.randn(ncur, H, d, device="cuda").to(torch.bfloat16)
    vc = torch.randn(ncur, H, d, device="cuda").to(torch.bfloat16)
    out = D.attention(q, None, kc, vc, d ** -0.5, kv_bf16=kv)
    torch.cuda.synchronize()
    kvf = kv.float().cpu().numpy()
    ref = oracle_lib.attention(q.float().cpu().numpy(), kvf[0::2], kvf[1::2], kc.float().cpu().numpy(),
                               vc.float().cpu().numpy(), d ** -0.5, 8)
    _check(out, ref)


def test_head_sharding_is_bit_identical():
    """A rank computing only its heads (shard.head_range) reproduces the
    1-GPU output for those heads byte for byte (no cross-head coupling)."""
    from paper_2602_02958_b200.shard import head_range
    torch.manual_seed(3)
    H, nq, nc, ncur, d = 4, 130, 260, 70, 128
    cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=8)
    planes = clustered_planes(2 * H, nc, d, n_clusters=8, outlier_scale=4.0, seed=5)
    chunks = D.compress(planes, cfg)
    q = torch.randn(nq, H, d, device="cuda").to(torch.bfloat16)
    kc = torch.randn(ncur, H, d, device="cuda").to(torch.bfloat16)
    vc = torch.randn(ncur, H, d, device="cuda").to(torch.bfloat16)
    full = D.attention(q, chunks, kc, vc)
    for world in (2, 3):
        for r in range(world):
            h0, h1 = head_range(H, world, r)
            sl = lambda t: t[:, h0:h1].contiguous()
            local_cache = D.compress(planes[2 * h0:2 * h1].contiguous(), cfg)
            assert torch.equal(local_cache.payload, chunks.payload[2 * h0:2 * h1])
            local = D.attention(sl(q), local_cache, sl(kc), sl(vc))
            assert torch.equal(local, full[:, h0:h1])


def _rope_np(k, cos, sin, mode):
    """k [H, n, d] float64 rotated per position (the kernel's rule, bf16 store)."""
    import torch as _t
    half = k.shape[-1] // 2
    if mode == "rotate_half":
        a, b = k[..., :half], k[..., half:]
    else:
        a, b = k[..., 0::2], k[..., 1::2]
    ra = a * cos - b * sin
    rb = a * sin + b * cos
    out = np.empty_like(k)
    if mode == "rotate_half":
        out[..., :half], out[..., half:] = ra, rb
    else:
        out[..., 0::2], out[..., 1::2] = ra, rb
    return _t.from_numpy(out.astype(np.float32)).to(_t.bfloat16).float().numpy()


@pytest.mark.parametrize("mode", ["rotate_half", "interleaved"])
@pytest.mark.parametrize("quant", [True, False])
def test_pre_rope_cached_keys_vs_oracle(oracle_lib, mode, quant):
    """keys cached before RoPE, rotated after the decode."""
    torch.manual_seed(3)
    H, nq, nc, ncur, d = 2, 160, 320, 96, 128
    cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=16)
    pos = np.arange(nc, dtype=np.float64)[:, None]
    freq = 10000.0 ** (-np.arange(d // 2, dtype=np.float64) / (d // 2))
    cos = np.cos(pos * freq).astype(np.float32)
    sin = np.sin(pos * freq).astype(np.float32)
    q = (torch.randn(nq, H, d, device="cuda") * 0.5).to(torch.bfloat16)
    kc = torch.randn(ncur, H, d, device="cuda").to(torch.bfloat16)
    vc = torch.randn(ncur, H, d, device="cuda").to(torch.bfloat16)
    planes = clustered_planes(2 * H, nc, d, n_clusters=16, outlier_scale=4.0, seed=2)
    rope = (torch.from_numpy(cos).cuda(), torch.from_numpy(sin).cuda(), mode)
    if quant:
        chunks = D.compress(planes, cfg)
        out = D.attention(q, chunks, kc, vc, d ** -0.5, rope=rope)
        deq = oracle_lib.prq_decompress_batch(chunks.payload.cpu().numpy(), chunks.scales.cpu().numpy(),
                                              chunks.centroids.float().cpu().numpy(),
                                              chunks.assignments.cpu().numpy(), nc, d, cfg.bits,
                                              cfg.group_size, 8)
        kcache = torch.from_numpy(deq[0::2]).to(torch.bfloat16).double().numpy()
        vcache = deq[1::2]
    else:
        out = D.attention(q, None, kc, vc, d ** -0.5, kv_bf16=planes, rope=rope)
        pf = planes.float().cpu().numpy()
        kcache, vcache = pf[0::2].astype(np.float64), pf[1::2]
    torch.cuda.synchronize()
    kr = _rope_np(kcache, cos.astype(np.float64), sin.astype(np.float64), mode)
    ref = oracle_lib.attention(q.float().cpu().numpy(), kr, vcache, kc.float().cpu().numpy(),
                               vc.float().cpu().numpy(), d ** -0.5, 8)
    _check(out, ref)


@pytest.mark.parametrize("fused", [False, True])
def test_attention_reports_corrupt_cache(fused):
    """a NaN-pattern scale or an assignment >= K in the cache is
    reported (NaNPattern / DimensionMismatch) like dequantize does, and the
    corrupt assignment decodes with centroid 0 instead of reading past the
    centroid table."""
    from paper_2602_02958_b200.qvgcodec.errors import DimensionMismatch, NaNPattern

    H, nc, nq, d = 1, 256, 64, 128
    g = torch.Generator(device="cuda").manual_seed(5)
    x = (torch.randn((2 * H, nc, d), generator=g, device="cuda") * 2).to(torch.bfloat16)
    cfg = QuantConfig(bits=2, group_size=64, stages=1, centroids=8)
    chunks = D.compress(x, cfg, chunk_index=0)
    q, kc, vc = (torch.randn((nq, H, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    D.attention(q, chunks, kc, vc, fused=fused)                       # clean cache: no error
    bad = D.DeviceChunks(cfg, nc, d, chunks.payload, chunks.scales, chunks.centroids,
                         chunks.assignments.clone())
    bad.assignments[0, 0, 5] = 200
    with pytest.raises(DimensionMismatch):
        D.attention(q, bad, kc, vc, fused=fused)
    bad2 = D.DeviceChunks(cfg, nc, d, chunks.payload, chunks.scales.clone(), chunks.centroids,
                          chunks.assignments)
    bad2.scales[1, 7] = 0x7F
    with pytest.raises(NaNPattern):
        D.attention(q, bad2, kc, vc, fused=fused)


def test_attention_validates_inputs():
    H, nc, nq, d = 2, 128, 32, 128
    kv = torch.zeros((2 * H, nc, d), dtype=torch.bfloat16, device="cuda")
    q = torch.zeros((nq, H, d), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        D.attention(q.float(), None, q, q, kv_bf16=kv)                 # fp32 q
    with pytest.raises(ValueError):
        D.attention(q, None, q[:, :1], q[:, :1], kv_bf16=kv)            # k_cur heads != q heads
    with pytest.raises(ValueError):
        D.attention(q, None, q, q, kv_bf16=kv[:, :, :64])                # head_dim mismatch
