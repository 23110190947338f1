"""BASELINE configs 4 and 5 as parity cases.

C4 (HY-WorldPlay long horizon): PRQ stage sweep S = 1..4 with group sizes 16
and 64 on streaming chunks — bit-exact against the CPU oracle on identical
clustered planes, and the reconstruction MSE decreasing with S.
C5 (microbench grid N 4K..256K x K 16..256 x b 2/4): full-size planes are
checked through size-independent properties — every sampled row's assignment
is the exact float64 argmin for the device's own final centroids (the
reference's FMA-chain distance, recomputed by the oracle on those rows), and
quantize/dequantize of sampled rows given the device's stage metadata equals
the oracle bit for bit (rows are independent given the metadata)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402
from paper_2602_02958_b200.synth import kv_cache_planes  # noqa: E402


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("S", [1, 2, 3, 4])
@pytest.mark.parametrize("B", [16, 64])
def test_c4_prq_stage_sweep_vs_oracle(oracle_lib, S, B):
    cfg = QuantConfig(bits=2, group_size=B, stages=S, centroids=64)
    x = kv_cache_planes(1, 2, 1560, 128, seed=40 + S, device="cuda")     # 4 planes, one latent frame each
    P, N, d = x.shape
    chunk = 7
    dc = D.compress(x, cfg, chunk_index=chunk)
    draws = np.stack([oracle_lib.pp_draws(0, chunk, S, 64)] * P)
    pay, sc, cent, asg, iters = oracle_lib.prq_compress_batch(x.float().cpu().numpy(), 2, B, S, 64, 10, 1e-4,
                                                              draws, 16)
    assert np.array_equal(dc.assignments.cpu().numpy(), asg)
    assert np.array_equal(dc.payload.cpu().numpy(), pay)
    assert np.array_equal(dc.scales.cpu().numpy(), sc)
    out = D.dequantize(dc, torch.float32).cpu().numpy()
    ref = oracle_lib.prq_decompress_batch(pay, sc, cent, asg, N, d, 2, B, 16)
    assert np.array_equal(_u32(out), _u32(ref))


def test_c4_mse_decreases_with_stages():
    x = kv_cache_planes(1, 1, 1560, 128, seed=3, device="cuda")
    mse = []
    for S in range(0, 5):
        cfg = QuantConfig(bits=2, group_size=64, stages=S, centroids=64)
        dc = D.compress(x, cfg, chunk_index=0)
        rec = D.dequantize(dc, torch.float32)
        mse.append(float(((rec - x.float()) ** 2).mean()))
    assert all(b < a for a, b in zip(mse, mse[1:])), mse


@pytest.mark.parametrize("N,K,bits", [(4096, 16, 2), (32768, 128, 4), (65536, 256, 2), (262144, 64, 2)])
def test_c5_full_size_properties(oracle_lib, N, K, bits):
    cfg = QuantConfig(bits=bits, group_size=64, stages=1, centroids=K)
    x = kv_cache_planes(1, 1, N, 128, seed=N % 1000 + K, device="cuda")[:1]   # one K plane
    dc = D.compress(x, cfg, chunk_index=0)
    rng = np.random.default_rng(N + K)
    rows = np.sort(rng.choice(N, size=min(N, 2048), replace=False))
    xs = x[0, rows].float().cpu().numpy().astype(np.float64)
    cent64 = D.compress(x, cfg, chunk_index=0, keep_f64=True).centroids_f64[0, 0].cpu().numpy()
    # assignment = exact argmin (reference distance) for the final centroids
    a_ref = oracle_lib.assign(xs, cent64)
    assert np.array_equal(dc.assignments[0, 0, rows].cpu().numpy(), a_ref.astype(np.uint8))
    # quantize / dequantize of the sampled rows given the device metadata
    cb = dc.centroids[0:1].float().cpu().numpy()
    asg = dc.assignments[0:1, :, rows].cpu().numpy()
    rp, rs = oracle_lib.quantize_given_metas_batch(x[0:1, rows].float().cpu().numpy(), cb, asg, bits, 64, 8)
    pay = dc.payload[0].cpu().numpy().reshape(N, -1)[rows]
    sc = dc.scales[0].cpu().numpy().reshape(N, -1)[rows]
    assert np.array_equal(pay.reshape(1, -1), rp)
    assert np.array_equal(sc.reshape(1, -1), rs)
    out = D.dequantize(dc, torch.float32)[0, rows].cpu().numpy()
    ref = oracle_lib.prq_decompress_batch(rp, rs, cb, asg, len(rows), 128, bits, 64, 8)[0]
    assert np.array_equal(_u32(out), _u32(ref))
