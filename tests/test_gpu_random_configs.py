"""Randomised configurations through the codec dispatcher (quantize given the
stage metadata, then dequantize), bit-exact against the CPU oracle.

Each case draws P, N, head_dim, bits, group size, stages and centroid count
from the ranges the kernels plan for (and their fallbacks: N not a multiple
of 4, head_dims other than 128 / 256, K up to 256 with tables at the shared-
memory budget edge), and bf16 planes with outlier channels, tiny entries,
exact zeros and exactly representable ties (values on a coarse grid), so the
certificates, the window tests, the exact-scale and exact-code fallbacks and
the Fast2Sum add-back checks all run.  Seeds are fixed: failures reproduce.
QVG_RANDOM_SCALE=k multiplies the case counts (soak runs)."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.lowprec import round_to_bf16  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402

SCALE = int(os.environ.get("QVG_RANDOM_SCALE", "1"))
N_CASES = 150 * SCALE


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.choice([64, 128, 128, 256]))
    bits = int(rng.choice([2, 2, 4, 8]))
    B = int(rng.choice([b for b in (16, 32, 64, 128) if b <= d]))
    S = int(rng.integers(0, 5))
    K = int(rng.choice([8, 16, 64, 256]))
    P = int(rng.integers(1, 6))
    N = int(rng.integers(1, 40)) * 64 + int(rng.choice([0, 0, 0, 1, 3]))
    x = rng.normal(0.0, float(rng.choice([0.01, 1.0, 2.5])), size=(P, N, d))
    x[:, :, :: int(rng.choice([8, 16, 32]))] *= float(rng.choice([1.0, 40.0, 300.0]))
    x[rng.random(x.shape) < 0.002] *= 2.0 ** -30
    x[rng.random(x.shape) < 0.002] = 0.0
    grid = rng.random(x.shape) < 0.05
    x[grid] = np.round(x[grid] * 4.0) / 4.0                     # coarse values: exact ties
    x = round_to_bf16(x.astype(np.float32)).astype(np.float32)
    Sc = max(S, 1)
    cent = rng.normal(0.0, 1.5, size=(P, Sc, K, d)) * (2.0 ** rng.integers(-6, 4, size=(P, Sc, K, 1)))
    cent = round_to_bf16(cent.astype(np.float32)).astype(np.float32)[:, :S]
    asg = rng.integers(0, K, size=(P, Sc, N), dtype=np.uint8)[:, :S]
    return dict(P=P, N=N, d=d, bits=bits, B=B, S=S, K=K), x, np.ascontiguousarray(cent), np.ascontiguousarray(asg)


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_config_codec_vs_oracle(oracle_lib, seed):
    c, x, cent, asg = _case(seed)
    cfg = QuantConfig(bits=c["bits"], group_size=c["B"], stages=c["S"], centroids=c["K"])
    cb = torch.from_numpy(cent).to(torch.bfloat16).cuda()
    ag = torch.from_numpy(asg).cuda()
    pay, sc = D.quantize(torch.from_numpy(x).to(torch.bfloat16).cuda(), cfg, cb, ag)
    rp, rs = oracle_lib.quantize_given_metas_batch(x, cent, asg, c["bits"], c["B"], 16)
    assert np.array_equal(sc.cpu().numpy(), rs), c
    assert np.array_equal(pay.cpu().numpy(), rp), c
    dc = D.DeviceChunks(cfg, c["N"], c["d"], pay, sc, cb, ag)
    out = D.dequantize(dc, torch.float32).cpu().numpy()
    ref = oracle_lib.prq_decompress_batch(rp, rs, cent, asg, c["N"], c["d"], c["bits"], c["B"], 16)
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32)), c


def _compress_case(seed):
    rng = np.random.default_rng(5000 + seed)
    d = int(rng.choice([24, 64, 128, 128]))
    bits = int(rng.choice([2, 2, 4, 8]))
    B = int(rng.choice([b for b in (8, 16, 32, 64) if d % b == 0]))
    S = int(rng.integers(1, 4))
    K = int(rng.choice([4, 8, 16, 64]))
    P = int(rng.integers(1, 4))
    N = int(rng.integers(max(K, 40), 1200))
    centers = rng.normal(0.0, 3.0, size=(P, 12, d))
    x = centers[:, rng.integers(0, 12, size=N)] + rng.normal(0.0, 0.7, size=(P, N, d))
    x[:, :, :: int(rng.choice([8, 16]))] *= float(rng.choice([1.0, 20.0]))
    x = round_to_bf16(x.astype(np.float32)).astype(np.float32)
    chunks = [int(v) for v in rng.integers(0, 50, size=P)]
    return dict(P=P, N=N, d=d, bits=bits, B=B, S=S, K=K, chunks=chunks), x


@pytest.mark.parametrize("seed", range(80 * SCALE))
def test_random_config_compress_vs_oracle(oracle_lib, seed):
    """prq_compress (k-means++ / Lloyd / smoothing / quantize) over random
    shapes, bits, groups, stages, K and per-plane chunk indices: assignments,
    bf16 centroids, iteration counts, payload and scales bit-exact."""
    c, x = _compress_case(seed)
    cfg = QuantConfig(bits=c["bits"], group_size=c["B"], stages=c["S"], centroids=c["K"])
    dc = D.compress(torch.from_numpy(x).to(torch.bfloat16).cuda(), cfg, chunk_index=c["chunks"])
    draws = np.stack([oracle_lib.pp_draws(0, ch, c["S"], c["K"]) for ch in c["chunks"]])
    pay, sc, cent, asg, iters = oracle_lib.prq_compress_batch(x, c["bits"], c["B"], c["S"], c["K"], 10, 1e-4,
                                                              draws, 16)
    assert np.array_equal(dc.assignments.cpu().numpy(), asg), c
    assert np.array_equal(dc.centroids.float().cpu().numpy().view(np.uint32), cent.view(np.uint32)), c
    assert np.array_equal(dc.iters.cpu().numpy(), iters), c
    assert np.array_equal(dc.scales.cpu().numpy(), sc), c
    assert np.array_equal(dc.payload.cpu().numpy(), pay), c


@pytest.mark.parametrize("seed", range(60 * SCALE))
def test_random_attention_vs_oracle(oracle_lib, seed):
    """Attention over a quantized cache at random head counts, query / cache /
    current-chunk lengths (partial tiles, empty cache or empty current chunk),
    codec configs and softmax scales, both the two-pass (decode + tcgen05
    pipeline) and the in-tile decoder.  Both attend over the bf16 rounding of
    the reconstruction (the operand precision of the tensor-core path), so the
    fp64 oracle over that rounding is the tight reference (max-abs <= 1e-2
    max|O|, rel-L2 <= 5e-3: bf16 P and output); at the model's softmax scale
    d^-1/2 the result is also held to SURVEY 8(c)'s tolerance against the
    oracle over the f32 reconstruction (max-abs <= 2e-2 max|O|, rel-L2 <=
    1e-2).  At the sharper scale 0.3 the bf16 rounding of the cached keys moves
    the logits by up to 3.4x more and that second bound is not the kernel's
    to meet (soak: 3 of 3 600 cases at 1.7-2.5e-2 max-abs, all <= 3.2e-3
    against the bf16 reconstruction; tests/diag_attn_seed.py)."""
    from paper_2602_02958_b200.synth import clustered_planes
    rng = np.random.default_rng(9000 + seed)
    H, d = int(rng.integers(1, 4)), 128
    nq = int(rng.integers(1, 300))
    nc = int(rng.choice([0, int(rng.integers(1, 700))]))
    ncur = int(rng.integers(0 if nc else 1, 260))
    cfg = QuantConfig(bits=int(rng.choice([2, 4])), group_size=int(rng.choice([32, 64])),
                      stages=int(rng.integers(1, 3)), centroids=int(rng.choice([8, 16])))
    fused = bool(rng.integers(0, 2))
    scale = float(rng.choice([d ** -0.5, 0.3]))
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = (torch.randn((nq, H, d), generator=g, device="cuda") * 0.5).to(torch.bfloat16)
    kc = torch.randn((ncur, H, d), generator=g, device="cuda").to(torch.bfloat16)
    vc = torch.randn((ncur, H, d), generator=g, device="cuda").to(torch.bfloat16)
    if nc:
        planes = clustered_planes(2 * H, nc, d, n_clusters=8, outlier_scale=4.0, seed=seed)
        chunks = D.compress(planes, cfg)
        out = D.attention(q, chunks, kc, vc, scale, fused=fused)
        deq = oracle_lib.prq_decompress_batch(chunks.payload.cpu().numpy(), chunks.scales.cpu().numpy(),
                                              chunks.centroids.float().cpu().numpy(),
                                              chunks.assignments.cpu().numpy(), nc, d, cfg.bits,
                                              cfg.group_size, 8)
    else:
        out = D.attention(q, None, kc, vc, scale)
        deq = np.zeros((2 * H, 0, d), np.float32)
    o = out.float().cpu().numpy().astype(np.float64)
    args = (q.float().cpu().numpy(), kc.float().cpu().numpy(), vc.float().cpu().numpy())
    case = dict(H=H, nq=nq, nc=nc, ncur=ncur, fused=fused, scale=scale)
    for dq, tol, rtol in ((round_to_bf16(deq).astype(np.float32), 1e-2, 5e-3),
                          (deq, 2e-2, 1e-2) if scale == d ** -0.5 else (None, 0, 0)):
        if dq is None:
            continue
        ref = oracle_lib.attention(args[0], dq[0::2], dq[1::2], args[1], args[2], scale, 8)
        err = np.abs(o - ref).max() / np.abs(ref).max()
        rl2 = np.linalg.norm(o - ref) / np.linalg.norm(ref)
        assert err <= tol and rl2 <= rtol, (case, tol, err, rl2)
