"""GPU parity at the shapes the benchmark runs (VERDICT r1 "Next round" 1).

Inputs are the reference generator's planes (paper_2602_02958_b200/datagen.py,
bit-identical to Q/datagen.py, pinned by tests/golden/datagen.npz) with the
SURVEY §8(d) K/V parameters:

* LongCat compress — N 38 400, K 256, S 1, b2/B64, one K and one V plane:
  assignments, float64 centroids, iterations, payload, scales and the f32
  reconstruction bit-exact against the oracle (Q/prq.py:58-80,113-132).
* Self-Forcing compress of 456 C1-shaped planes (4680 x 128, S2 K64) in one
  call: the final quantize takes the ring kernel with ~3 planes
  per CTA and 49 row passes per plane, i.e. the mbarrier flow across plane
  boundaries (buffer reuse j >= 2, mid-plane widening) the bench exercises.
* C5 N 65 536, K 256: the full k-means trajectory (k-means++ picks, every
  Lloyd step, iteration count) against the oracle, not a self-check.
* Generic float32 input that is not bf16-exact (datagen without the bf16
  rounding), through both the few-plane and the >= 148-plane kernels.
* LongCat-layer attention (32 heads, 38 400 cached + 7 800 current tokens,
  7 800 queries) against the float64 oracle on sampled query rows.
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2602_02958_b200 import datagen as G  # noqa: E402
from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402

THREADS = max(2, len(os.sched_getaffinity(0)))


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def _planes(refs, n_heads, n_tokens, drift=0.0, bf16=True):
    """Host float32 planes of the listed (layer, head, K|V, chunk) streams."""
    out = []
    for r in refs:
        x = G.stream_chunk(G.kv_seed(r.layer, r.head, n_heads, r.value), r.chunk,
                           G.kv_params(n_tokens, r.value, drift))
        out.append(G.bf16_bits_to_f32(G.round_bf16_bits(x)) if bf16 else x)
    return np.stack(out)


def _oracle_compress_planes(oracle_lib, x, cfg, chunk, threads=None):
    """oracle.prq_compress per plane on a thread pool (ctypes releases the GIL)."""
    draws = oracle_lib.pp_draws(cfg.seed, chunk, cfg.stages, cfg.centroids)

    def one(p):
        return oracle_lib.prq_compress(x[p], cfg.bits, cfg.group_size, cfg.stages, cfg.centroids,
                                       cfg.kmeans_max_iters, cfg.kmeans_tol, draws=draws)

    with cf.ThreadPoolExecutor(threads or len(x)) as ex:
        return list(ex.map(one, range(len(x))))


def _check_against(dc, refs, x, cfg, oracle_lib):
    P, N, d = x.shape
    for p, r in enumerate(refs):
        assert np.array_equal(dc.iters[p].cpu().numpy(), r["iters"]), ("iters", p)
        assert np.array_equal(dc.assignments[p].cpu().numpy(), r["assignments"]), ("assignments", p)
        assert np.array_equal(dc.centroids_f64[p].cpu().numpy().view(np.uint64),
                              r["centroids_f64"].view(np.uint64)), ("f64 centroids", p)
        assert np.array_equal(_u32(dc.centroids[p].float().cpu().numpy()), _u32(r["centroids"])), p
        assert np.array_equal(dc.payload[p].cpu().numpy(), r["payload"]), ("payload", p)
        assert np.array_equal(dc.scales[p].cpu().numpy(), r["scales"]), ("scales", p)
    out = D.dequantize(dc, torch.float32).cpu().numpy()
    for p, r in enumerate(refs):
        ref = oracle_lib.prq_decompress(r["payload"], r["scales"], r["centroids"], r["assignments"], N, d,
                                        cfg.bits, cfg.group_size)
        assert np.array_equal(_u32(out[p]), _u32(ref)), ("decoded", p)


def test_longcat_compress_vs_oracle(oracle_lib):
    cfg = QuantConfig(bits=2, group_size=64, stages=1, centroids=256)
    refs = [G.PlaneRef(0, 3, False, 0), G.PlaneRef(0, 3, True, 0)]
    x = _planes(refs, 32, 38400)
    dc = D.compress(torch.from_numpy(x).to(torch.bfloat16).cuda(), cfg, chunk_index=0, keep_f64=True)
    torch.cuda.synchronize()
    _check_against(dc, _oracle_compress_planes(oracle_lib, x, cfg, 0), x, cfg, oracle_lib)


def test_self_forcing_456_planes_vs_oracle(oracle_lib):
    cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=64)
    refs = G.cache_layout(19, 12, [2])                                   # 456 planes of chunk 2
    u = G.kv_cache_bf16(refs, 12, 4680, drift=0.0125)
    x = torch.from_numpy(u.view(np.int16)).view(torch.bfloat16)
    dc = D.compress(x.cuda(), cfg, chunk_index=2)
    P = x.shape[0]
    draws = np.stack([oracle_lib.pp_draws(0, 2, 2, 64)] * P)
    xf = G.bf16_bits_to_f32(u)
    pay, sc, cent, asg, iters = oracle_lib.prq_compress_batch(xf, 2, 64, 2, 64, 10, 1e-4, draws, THREADS)
    assert np.array_equal(dc.assignments.cpu().numpy(), asg)
    assert np.array_equal(dc.iters.cpu().numpy(), iters)
    assert np.array_equal(_u32(dc.centroids.float().cpu().numpy()), _u32(cent))
    assert np.array_equal(dc.scales.cpu().numpy(), sc)
    assert np.array_equal(dc.payload.cpu().numpy(), pay)
    # the decode of the same 456 planes (persistent stream kernel), f32 and bf16
    sel = np.arange(0, P, 37)
    ref = oracle_lib.prq_decompress_batch(pay[sel], sc[sel], cent[sel], asg[sel], 4680, 128, 2, 64, THREADS)
    out = D.dequantize(dc, torch.float32)[torch.from_numpy(sel).cuda()].cpu().numpy()
    assert np.array_equal(_u32(out), _u32(ref))
    outb = D.dequantize(dc, torch.bfloat16)[torch.from_numpy(sel).cuda()].cpu()
    assert torch.equal(outb.view(torch.int16), torch.from_numpy(ref).to(torch.bfloat16).view(torch.int16))


def test_c5_full_trajectory_n65536_k256(oracle_lib):
    cfg = QuantConfig(bits=2, group_size=64, stages=1, centroids=256)
    refs = [G.PlaneRef(0, 0, False, 0), G.PlaneRef(0, 0, True, 0)]
    x = _planes(refs, 1, 65536)
    dc = D.compress(torch.from_numpy(x).to(torch.bfloat16).cuda(), cfg, chunk_index=0, keep_f64=True)
    torch.cuda.synchronize()
    _check_against(dc, _oracle_compress_planes(oracle_lib, x, cfg, 0), x, cfg, oracle_lib)


@pytest.mark.parametrize("P,N", [(4, 4680), (160, 1560)])
def test_generic_f32_compress_vs_oracle(oracle_lib, P, N):
    """float32 planes that are not bf16-exact (the reference's KVPlane dtype,
    Q/types.py:57-64): the uncertified residual paths and the float32 ring kernel."""
    cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=64)
    refs = G.cache_layout(P // 24 or 1, 12, [1])[:P]
    x = _planes(refs, 12, N, drift=0.0125, bf16=False)
    assert not np.array_equal(x, G.bf16_bits_to_f32(G.round_bf16_bits(x)))
    dc = D.compress(torch.from_numpy(x).cuda(), cfg, chunk_index=1, keep_f64=True)
    if P <= 8:
        _check_against(dc, _oracle_compress_planes(oracle_lib, x, cfg, 1), x, cfg, oracle_lib)
        return
    draws = np.stack([oracle_lib.pp_draws(0, 1, 2, 64)] * P)
    pay, sc, cent, asg, iters = oracle_lib.prq_compress_batch(x, 2, 64, 2, 64, 10, 1e-4, draws, THREADS)
    assert np.array_equal(dc.assignments.cpu().numpy(), asg)
    assert np.array_equal(dc.iters.cpu().numpy(), iters)
    assert np.array_equal(dc.scales.cpu().numpy(), sc)
    assert np.array_equal(dc.payload.cpu().numpy(), pay)


# Attention over the quantized LongCat layer, two references:
# (a) SURVEY §8(c): float64 attention over the oracle's float32 reconstruction
#     (includes the bf16 rounding of the reconstructed K/V, inherent to a bf16
#     attention: |K| ~ 1e2 makes score errors of ~0.1 possible);
# (b) float64 attention over the same reconstruction rounded to bf16 (the
#     kernel's actual operands): the kernel's own error (P in bf16, fp32
#     accumulation, exp2 polynomial).
# Measured on B200 (r02, pipelined and fused kernels alike):
#   (a) max-abs/max|O| 1.717e-2, rel-L2 6.87e-3  -> SURVEY §8(c) bounds kept;
#   (b) max-abs/max|O| 2.52e-3,  rel-L2 2.03e-3  -> bounds ~2.5x the measurement.
ATTN_A = (2e-2, 1e-2)        # (max-abs / max|O|, rel-L2) — SURVEY §8(c)
ATTN_B = (6e-3, 5e-3)


def test_longcat_layer_attention_vs_oracle(oracle_lib):
    H, nc, nq, d = 32, 38400, 7800, 128
    cfg = QuantConfig(bits=2, group_size=64, stages=1, centroids=256)
    refs = G.cache_layout(1, H, [0])
    u = G.kv_cache_bf16(refs, H, nc)
    planes = torch.from_numpy(u.view(np.int16)).view(torch.bfloat16).cuda()
    chunks = D.compress(planes, cfg, chunk_index=0)
    g = torch.Generator(device="cuda")
    g.manual_seed(12345)
    q = torch.randn((nq, H, d), generator=g, device="cuda").to(torch.bfloat16)
    kc = torch.randn((nq, H, d), generator=g, device="cuda").to(torch.bfloat16)
    vc = torch.randn((nq, H, d), generator=g, device="cuda").to(torch.bfloat16)
    out = D.attention(q, chunks, kc, vc)
    outf = D.attention(q, chunks, kc, vc, fused=True)
    torch.cuda.synchronize()
    deq = oracle_lib.prq_decompress_batch(chunks.payload.cpu().numpy(), chunks.scales.cpu().numpy(),
                                          chunks.centroids.float().cpu().numpy(),
                                          chunks.assignments.cpu().numpy(), nc, d, 2, 64, THREADS)
    deq16 = G.bf16_bits_to_f32(G.round_bf16_bits(deq))
    rows = np.sort(np.random.default_rng(7).choice(nq, 96, replace=False))
    qs, kn, vn = q[rows].float().cpu().numpy(), kc.float().cpu().numpy(), vc.float().cpu().numpy()
    refa = oracle_lib.attention(qs, deq[0::2], deq[1::2], kn, vn, d ** -0.5, THREADS)
    refb = oracle_lib.attention(qs, deq16[0::2], deq16[1::2], kn, vn, d ** -0.5, THREADS)
    for o, name in ((out, "pipelined"), (outf, "fused")):
        got = o[torch.from_numpy(rows).cuda()].float().cpu().numpy().astype(np.float64)
        for ref, (tm, tl), tag in ((refa, ATTN_A, "f32 reconstruction"), (refb, ATTN_B, "bf16 operands")):
            maxabs = np.abs(got - ref).max() / np.abs(ref).max()
            rel_l2 = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            print(f"longcat attention {name} vs {tag}: max-abs/max|O| {maxabs:.3e}, rel-L2 {rel_l2:.3e}")
            assert maxabs <= tm and rel_l2 <= tl, (name, tag, maxabs, rel_l2)
