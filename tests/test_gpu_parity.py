"""GPU parity: the sm_100a path (through the C ABI) against the reference's
own outputs (tests/golden) and the CPU oracle on seeded inputs.

Bar: bit-exact payload / scale bytes, assignments, bf16 centroids, f64
centroids, k-means iteration counts; dequantized float32 bit-exact; bf16
output = RNE(oracle float32)."""
import numpy as np
import pytest
import torch

from conftest import golden_planes
from golden_io import load_plane

pytestmark = pytest.mark.gpu

from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402


def cfg_of(rec, **kw):
    return QuantConfig(bits=rec["bits"], group_size=rec["group_size"], stages=rec["stages"],
                       centroids=rec["centroids"], **kw)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("name", golden_planes())
@pytest.mark.parametrize("xdtype", [torch.bfloat16, torch.float32])
def test_compress_matches_reference_fixture(name, xdtype):
    rec = load_plane(name)
    cfg = cfg_of(rec)
    x = torch.from_numpy(rec["x"]).to(xdtype).cuda()[None]
    warm = None
    if "warm" in rec:
        warm = torch.from_numpy(rec["warm"]).cuda()[None]
    dc = D.compress(x, cfg, chunk_index=rec["chunk_index"], warm_init=warm, keep_f64=True)
    torch.cuda.synchronize()
    S = rec["stages"]
    if S:
        assert np.array_equal(dc.iters[0].cpu().numpy(), rec["iters"]), "iterations"
        assert np.array_equal(dc.assignments[0].cpu().numpy(), rec["assignments"]), "assignments"
        assert np.array_equal(dc.centroids_f64[0].cpu().numpy().view(np.uint64),
                              rec["cent_f64"].view(np.uint64)), "f64 centroids"
        assert np.array_equal(_u32(dc.centroids[0].float().cpu().numpy()),
                              _u32(rec["centroids_bf16"])), "bf16 centroids"
    assert np.array_equal(dc.payload[0].cpu().numpy(), rec["payload"]), "payload"
    assert np.array_equal(dc.scales[0].cpu().numpy(), rec["scales"]), "scales"
    out = D.dequantize(dc, torch.float32)
    assert np.array_equal(_u32(out[0].cpu().numpy()), _u32(rec["decoded"])), "decoded f32"
    outb = D.dequantize(dc, torch.bfloat16)
    ref_b = torch.from_numpy(rec["decoded"]).to(torch.bfloat16)
    assert torch.equal(outb[0].cpu().view(torch.int16), ref_b.view(torch.int16)), "decoded bf16"


def _rand_planes(rng, P, N, d, scale_outlier):
    x = rng.normal(0, 2.5, size=(P, N, d)) + rng.normal(0, 0.125, size=(P, N, d))
    x[:, :, ::16] *= scale_outlier
    return torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)


@pytest.mark.parametrize("bits,B,S,K,d", [
    (2, 64, 2, 64, 128), (4, 16, 1, 32, 128), (8, 32, 3, 8, 64), (2, 16, 4, 16, 128),
    (2, 128, 1, 256, 128), (4, 8, 2, 5, 24), (2, 4, 1, 7, 20), (4, 128, 0, 1, 128)])
def test_quantize_dequantize_given_metas_vs_oracle(oracle_lib, bits, B, S, K, d):
    rng = np.random.default_rng(bits * 1000 + B * 10 + S)
    P, N = 3, 517
    x = _rand_planes(rng, P, N, d, 40.0)
    # metas: centroids drawn near the data, random assignments
    cent = torch.from_numpy(rng.normal(0, 2.0, size=(P, S, K, d)).astype(np.float32)).to(torch.bfloat16)
    asg = torch.from_numpy(rng.integers(0, K, size=(P, S, N)).astype(np.uint8))
    cfg = QuantConfig(bits=bits, group_size=B, stages=S, centroids=K)
    pay, sc = D.quantize(x.cuda(), cfg, cent.cuda(), asg.cuda())
    rp, rs = oracle_lib.quantize_given_metas_batch(x.float().numpy(), cent.float().numpy(),
                                                   asg.numpy(), bits, B, 4)
    assert np.array_equal(pay.cpu().numpy(), rp)
    assert np.array_equal(sc.cpu().numpy(), rs)
    dc = D.DeviceChunks(cfg, N, d, pay, sc, cent.cuda(), asg.cuda())
    out = D.dequantize(dc, torch.float32).cpu().numpy()
    ref = oracle_lib.prq_decompress_batch(rp, rs, cent.float().numpy(), asg.numpy(), N, d, bits, B, 4)
    assert np.array_equal(_u32(out), _u32(ref))


def test_quantize_boundary_cases(oracle_lib):
    """Residuals placed exactly on / one ulp around rounding boundaries, zero
    groups, saturating groups (s > 448) and sub-2^-9 scales exercise the
    certified fallback paths of the fast kernel."""
    rng = np.random.default_rng(7)
    P, N, d, B = 2, 256, 128, 64
    x = rng.normal(size=(P, N, d)).astype(np.float32)
    s = np.float32(0.15625)
    x[0, 0, :B] = 0.0                                  # zero group -> 0x38
    x[0, 1, :B] = 0.0
    x[0, 1, 0] = 1e-7                                  # tiny scale -> 0x01
    x[0, 2, :B] = 3000.0                               # saturating scale
    x[0, 3, :B] = s / 2                                # exact half -> ties
    x[0, 3, 0] = s
    x[0, 4, :B] = np.nextafter(s / 2, np.float32(1))   # just above the tie
    x[0, 4, 0] = s
    x[0, 5, :B] = np.nextafter(s / 2, np.float32(0))
    x[0, 5, 0] = s
    for bits in (2, 4, 8):
        cfg = QuantConfig(bits=bits, group_size=B, stages=0, centroids=1)
        xt = torch.from_numpy(x).cuda()
        pay, sc = D.quantize(xt, cfg)
        rp, rs = oracle_lib.quantize_given_metas_batch(x, np.zeros((P, 0, 1, d), np.float32),
                                                       np.zeros((P, 0, N), np.uint8), bits, B, 4)
        assert np.array_equal(sc.cpu().numpy(), rs), bits
        assert np.array_equal(pay.cpu().numpy(), rp), bits


def test_kmeans_primitives_vs_oracle(oracle_lib):
    rec = load_plane("s4_pro")
    rows = rec["x"].astype(np.float64)
    K = 16
    draws = oracle_lib.pp_draws(0, 0, 1, K)[0]
    cent_o, _ = oracle_lib.kmeans_pp(rows, K, draws)
    rt = torch.from_numpy(rows).cuda()[None]
    cent_g = D.kmeans_pp(rt, K, torch.from_numpy(draws).cuda()[None])
    assert np.array_equal(cent_g[0].cpu().numpy(), cent_o)
    a_o = oracle_lib.assign(rows, cent_o)
    a_g = D.assign(rt, cent_g)[0].cpu().numpy()
    assert np.array_equal(a_g, a_o)
    c_o, asg_o, obj_o, it_o = oracle_lib.kmeans(rows, K, 10, 1e-4, draws=draws)
    c_g, asg_g, obj_g, it_g = D.kmeans(rt, K, 10, 1e-4, draws=torch.from_numpy(draws).cuda()[None])
    assert np.array_equal(c_g[0].cpu().numpy().view(np.uint64), c_o.view(np.uint64))
    assert np.array_equal(asg_g[0].cpu().numpy(), asg_o.astype(np.uint8))
    assert obj_g[0].item() == obj_o and it_g[0].item() == it_o


def test_batched_planes_independent(oracle_lib):
    """P planes in one launch == each plane alone (and == the oracle)."""
    rng = np.random.default_rng(3)
    P, N, d = 5, 700, 128
    x = _rand_planes(rng, P, N, d, 10.0)
    cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=16)
    dc = D.compress(x.cuda(), cfg, chunk_index=[0, 1, 2, 3, 4])
    draws = np.stack([oracle_lib.pp_draws(0, c, 2, 16) for c in range(P)])
    pay, sc, cent, asg, iters = oracle_lib.prq_compress_batch(x.float().numpy(), 2, 64, 2, 16, 10,
                                                              1e-4, draws, 4)
    assert np.array_equal(dc.assignments.cpu().numpy(), asg)
    assert np.array_equal(dc.payload.cpu().numpy(), pay)
    assert np.array_equal(dc.scales.cpu().numpy(), sc)
    assert np.array_equal(dc.iters.cpu().numpy(), iters)
    one = D.compress(x[2:3].cuda(), cfg, chunk_index=2)
    assert torch.equal(one.payload[0], dc.payload[2])


def test_nonfinite_input_raises():
    from paper_2602_02958_b200.qvgcodec.errors import NonFiniteInput
    x = torch.zeros((1, 16, 128), dtype=torch.float32, device="cuda")
    x[0, 3, 5] = float("nan")
    with pytest.raises(NonFiniteInput):
        D.compress(x, QuantConfig(stages=1, centroids=4))
    with pytest.raises(NonFiniteInput):
        D.quantize(x, QuantConfig(stages=0))


@pytest.mark.parametrize("bits,B,S,K", [(2, 64, 2, 64), (4, 16, 1, 32), (2, 16, 3, 16), (8, 32, 2, 8)])
def test_many_planes_tma_path_vs_oracle(oracle_lib, bits, B, S, K):
    """>= 2*148 planes select the persistent TMA-staged kernels (k_*_v5)."""
    rng = np.random.default_rng(bits + 10 * S)
    P, N, d = 320, 97, 128
    x = _rand_planes(rng, P, N, d, 30.0)
    cent = torch.from_numpy(rng.normal(0, 2.0, size=(P, S, K, d)).astype(np.float32)).to(torch.bfloat16)
    asg = torch.from_numpy(rng.integers(0, K, size=(P, S, N)).astype(np.uint8))
    cfg = QuantConfig(bits=bits, group_size=B, stages=S, centroids=K)
    pay, sc = D.quantize(x.cuda(), cfg, cent.cuda(), asg.cuda())
    rp, rs = oracle_lib.quantize_given_metas_batch(x.float().numpy(), cent.float().numpy(),
                                                   asg.numpy(), bits, B, 8)
    assert np.array_equal(sc.cpu().numpy(), rs)
    assert np.array_equal(pay.cpu().numpy(), rp)
    dc = D.DeviceChunks(cfg, N, d, pay, sc, cent.cuda(), asg.cuda())
    out = D.dequantize(dc, torch.float32).cpu().numpy()
    ref = oracle_lib.prq_decompress_batch(rp, rs, cent.float().numpy(), asg.numpy(), N, d, bits, B, 8)
    assert np.array_equal(_u32(out), _u32(ref))
    outb = D.dequantize(dc, torch.bfloat16).cpu()
    assert torch.equal(outb.view(torch.int16), torch.from_numpy(ref).to(torch.bfloat16).view(torch.int16))


def test_quantize_boundary_cases_with_stages(oracle_lib):
    """The same boundary residuals reached through a centroid subtraction
    (S >= 1 selects the f32-table kernels): exact ties at s/2 and at the
    half-integers of the 4/8-bit grids, zero / tiny / saturating groups."""
    rng = np.random.default_rng(11)
    P, N, d, B = 2, 300, 128, 64
    x = rng.normal(size=(P, N, d)).astype(np.float32)
    s = np.float32(0.15625)
    x[0, 0, :B] = 0.0
    x[0, 1, :B] = 0.0
    x[0, 1, 0] = 1e-7
    x[0, 2, :B] = 3000.0
    x[0, 3, :B] = s / 2
    x[0, 3, 0] = s
    x[0, 4, :B] = np.nextafter(s / 2, np.float32(1))
    x[0, 4, 0] = s
    x[1, 5, :B] = np.float32(7.0) * np.arange(B, dtype=np.float32) / 8   # many grid half-points
    x[1, 5, 0] = 7.0
    xb = torch.from_numpy(x).to(torch.bfloat16)
    for S in (1, 2):
        cent = np.zeros((P, S, 3, d), np.float32)
        cent[:, :, 1, :] = 0.5
        cent[:, :, 2, ::3] = -0.25
        asg = rng.integers(0, 3, size=(P, S, N)).astype(np.uint8)
        asg[:, :, :6] = 0                               # boundary rows keep their exact values
        ct = torch.from_numpy(cent).to(torch.bfloat16)
        for bits in (2, 4, 8):
            cfg = QuantConfig(bits=bits, group_size=B, stages=S, centroids=3)
            for xt in (torch.from_numpy(x), xb):
                pay, sc = D.quantize(xt.cuda(), cfg, ct.cuda(), torch.from_numpy(asg).cuda())
                rp, rs = oracle_lib.quantize_given_metas_batch(xt.float().numpy(), ct.float().numpy(), asg,
                                                               bits, B, 4)
                assert np.array_equal(sc.cpu().numpy(), rs), (S, bits, xt.dtype)
                assert np.array_equal(pay.cpu().numpy(), rp), (S, bits, xt.dtype)


@pytest.mark.parametrize("bits,S", [(2, 2), (2, 3), (4, 2), (8, 4)])
def test_dequant_exactness_certificate_stress(oracle_lib, bits, S):
    """Centroid tables mixing magnitudes 1e-30 .. 1e4 (and zeros) make the
    non-final f32 partial sums inexact for many rows: those rows must take
    the float64 chain and still match the oracle bit for bit."""
    rng = np.random.default_rng(bits * 7 + S)
    P, N, d, K, B = 4, 400, 128, 8, 64
    mags = np.array([0.0, 1e-30, 1e-8, 3e-3, 0.7, 1.0, 55.0, 1e4], np.float32)
    cent = (rng.choice(mags, size=(P, S, K, d)) * rng.choice([-1, 1], size=(P, S, K, d))).astype(np.float32)
    ct = torch.from_numpy(cent).to(torch.bfloat16)
    asg = rng.integers(0, K, size=(P, S, N)).astype(np.uint8)
    x = _rand_planes(rng, P, N, d, 30.0)
    cfg = QuantConfig(bits=bits, group_size=B, stages=S, centroids=K)
    pay, sc = D.quantize(x.cuda(), cfg, ct.cuda(), torch.from_numpy(asg).cuda())
    rp, rs = oracle_lib.quantize_given_metas_batch(x.float().numpy(), ct.float().numpy(), asg, bits, B, 4)
    assert np.array_equal(sc.cpu().numpy(), rs)
    assert np.array_equal(pay.cpu().numpy(), rp)
    dc = D.DeviceChunks(cfg, N, d, pay, sc, ct.cuda(), torch.from_numpy(asg).cuda())
    ref = oracle_lib.prq_decompress_batch(rp, rs, ct.float().numpy(), asg, N, d, bits, B, 4)
    out = D.dequantize(dc, torch.float32).cpu().numpy()
    assert np.array_equal(_u32(out), _u32(ref))
    outb = D.dequantize(dc, torch.bfloat16).cpu()
    assert torch.equal(outb.view(torch.int16), torch.from_numpy(ref).to(torch.bfloat16).view(torch.int16))


@pytest.mark.parametrize("P,N", [(1, 9001), (3, 6000), (2, 40000)])
def test_planes_split_into_row_ranges(oracle_lib, P, N):
    """Few long planes: the kernels split each plane into row ranges (work
    items) spread over the CTAs; results equal the oracle."""
    rng = np.random.default_rng(P * N)
    d, K, S, B, bits = 128, 64, 2, 64, 2
    x = _rand_planes(rng, P, N, d, 20.0)
    cent = torch.from_numpy(rng.normal(0, 2.0, size=(P, S, K, d)).astype(np.float32)).to(torch.bfloat16)
    asg = rng.integers(0, K, size=(P, S, N)).astype(np.uint8)
    cfg = QuantConfig(bits=bits, group_size=B, stages=S, centroids=K)
    pay, sc = D.quantize(x.cuda(), cfg, cent.cuda(), torch.from_numpy(asg).cuda())
    rp, rs = oracle_lib.quantize_given_metas_batch(x.float().numpy(), cent.float().numpy(), asg, bits, B, 8)
    assert np.array_equal(sc.cpu().numpy(), rs)
    assert np.array_equal(pay.cpu().numpy(), rp)
    dc = D.DeviceChunks(cfg, N, d, pay, sc, cent.cuda(), torch.from_numpy(asg).cuda())
    ref = oracle_lib.prq_decompress_batch(rp, rs, cent.float().numpy(), asg, N, d, bits, B, 8)
    outb = D.dequantize(dc, torch.bfloat16).cpu()
    assert torch.equal(outb.view(torch.int16), torch.from_numpy(ref).to(torch.bfloat16).view(torch.int16))


def test_compress_clustered_many_planes_vs_oracle(oracle_lib):
    """Bench-like clustered K/V planes (outlier channels x10 / x100) through the
    full compress: the tensor-core assignment filter with its exact recheck
    must reproduce the reference's assignments, iterations and bytes."""
    from paper_2602_02958_b200.synth import kv_cache_planes

    cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=64)
    x = kv_cache_planes(2, 6, 1024, 128, seed=5, device="cuda")        # 24 planes
    P = x.shape[0]
    dc = D.compress(x, cfg, chunk_index=3)
    draws = np.stack([oracle_lib.pp_draws(0, 3, 2, 64)] * P)
    pay, sc, cent, asg, iters = oracle_lib.prq_compress_batch(x.float().cpu().numpy(), 2, 64, 2, 64, 10, 1e-4,
                                                              draws, 16)
    assert np.array_equal(dc.assignments.cpu().numpy(), asg)
    assert np.array_equal(dc.iters.cpu().numpy(), iters)
    assert np.array_equal(dc.payload.cpu().numpy(), pay)
    assert np.array_equal(dc.scales.cpu().numpy(), sc)


def test_compress_longcat_k256_vs_oracle(oracle_lib):
    """K = 256 centroids (two 128-centroid blocks in the tensor-core filter)."""
    from paper_2602_02958_b200.synth import kv_cache_planes

    cfg = QuantConfig(bits=2, group_size=64, stages=1, centroids=256)
    x = kv_cache_planes(1, 2, 2048, 128, seed=9, device="cuda")        # 4 planes
    P = x.shape[0]
    dc = D.compress(x, cfg, chunk_index=0)
    draws = np.stack([oracle_lib.pp_draws(0, 0, 1, 256)] * P)
    pay, sc, cent, asg, iters = oracle_lib.prq_compress_batch(x.float().cpu().numpy(), 2, 64, 1, 256, 10, 1e-4,
                                                              draws, 16)
    assert np.array_equal(dc.assignments.cpu().numpy(), asg)
    assert np.array_equal(dc.payload.cpu().numpy(), pay)


@pytest.mark.parametrize("scale_exp", [-112, -60, 90])
def test_compress_tiny_and_huge_scale_planes_vs_oracle(oracle_lib, scale_exp):
    """planes scaled far from 1 (bf16 near its underflow / large
    range): the tensor-core filter must not certify rows whose split products
    underflow -- assignments, centroids and codes stay bit-exact."""
    from paper_2602_02958_b200.synth import kv_cache_planes

    cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=16)
    x = (kv_cache_planes(1, 1, 1024, 128, seed=21, device="cuda").float() * 2.0 ** scale_exp).to(torch.bfloat16)
    P = x.shape[0]
    dc = D.compress(x, cfg, chunk_index=0)
    draws = np.stack([oracle_lib.pp_draws(0, 0, 2, 16)] * P)
    pay, sc, cent, asg, iters = oracle_lib.prq_compress_batch(x.float().cpu().numpy(), 2, 64, 2, 16, 10, 1e-4,
                                                              draws, 4)
    assert np.array_equal(dc.assignments.cpu().numpy(), asg)
    assert np.array_equal(dc.payload.cpu().numpy(), pay)
    assert np.array_equal(dc.scales.cpu().numpy(), sc)
    ref = oracle_lib.prq_decompress_batch(pay, sc, cent, asg, 1024, 128, 2, 64, 4)
    out = D.dequantize(dc, torch.float32).cpu().numpy()
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("bits,B,S", [(2, 64, 2), (2, 16, 1), (4, 32, 3), (8, 64, 2), (2, 128, 4)])
def test_many_planes_bf16_certificate_stress(oracle_lib, bits, B, S):
    """>= 148 bf16 planes through the certified ring quantize (qvg_stream.cu):
    coarse dyadic inputs and centroids put residuals exactly on code
    boundaries and group maxima exactly on the E4M3 grid (exact ties resolved
    from registers), while zeros, subnormals and 1e-30 .. 1e4 magnitude mixes
    make the exactness certificate fail for many rows (the float64 path)."""
    rng = np.random.default_rng(bits * 13 + B + S)
    P, N, d, K = 160, 70, 128, 6
    coarse = rng.integers(-24, 25, size=(P, N, d)).astype(np.float32) / 16
    x = np.where(rng.random((P, N, d)) < 0.5, coarse, rng.normal(0, 1.5, size=(P, N, d)).astype(np.float32))
    x[:8] = coarse[:8]                                          # whole planes on the grid
    x[8, :, ::5] = 0.0
    x[9, :, ::7] = 1e-39                                        # subnormal (bf16 keeps some)
    x[10] *= np.float32(1e-30)
    x[11, :, ::3] *= np.float32(1e4)
    mags = np.array([0.0, 1e-30, 1e-8, 0.125, 0.5, 1.0, 0.75, 3.0], np.float32)
    cent = (rng.choice(mags, size=(P, S, K, d)) * rng.choice([-1, 1], size=(P, S, K, d))).astype(np.float32)
    cent[:P // 2] = np.round(cent[:P // 2] * 8) / 8                # half the planes: dyadic centroids only
    xt = torch.from_numpy(x).to(torch.bfloat16)
    ct = torch.from_numpy(cent).to(torch.bfloat16)
    asg = rng.integers(0, K, size=(P, S, N)).astype(np.uint8)
    cfg = QuantConfig(bits=bits, group_size=B, stages=S, centroids=K)
    pay, sc = D.quantize(xt.cuda(), cfg, ct.cuda(), torch.from_numpy(asg).cuda())
    rp, rs = oracle_lib.quantize_given_metas_batch(xt.float().numpy(), ct.float().numpy(), asg, bits, B, 8)
    assert np.array_equal(sc.cpu().numpy(), rs)
    assert np.array_equal(pay.cpu().numpy(), rp)


@pytest.mark.parametrize("c1mag", [1e-30, 1e-12, 3e-8, 0.0])
def test_dequant_two_stage_add_order_certificate(oracle_lib, c1mag):
    """S = 2 rows whose stage-2 centroid block holds tiny entries: the
    reversed-order add-back (C_2 last) is certified only when the reference's
    float64 chain is exact too.  Dyadic stage-1 centroids equal to -q*s
    cancel exactly, so a wrong order would surface the tiny term."""
    rng = np.random.default_rng(int(abs(np.log10(c1mag))) if c1mag else 7)
    P, N, d, K, bits, B = 160, 64, 128, 4, 2, 64
    pay = rng.integers(0, 256, size=(P, N * d * bits // 8)).astype(np.uint8)
    codes = np.array([0x28, 0x30, 0x38, 0x2C], np.uint8)           # 0.25, 0.5, 1.0, 0.375
    sc = rng.choice(codes, size=(P, N * d // B)).astype(np.uint8)
    c0 = rng.choice(np.array([0.0, 0.25, -0.25, 0.5, -0.5, 0.75, 1.0, -1.5], np.float32), size=(P, 1, K, d))
    c1 = (rng.choice(np.array([0.0, 1.0, 3.0], np.float32), size=(P, 1, K, d)) * np.float32(c1mag)
          + rng.choice(np.array([0.0, 0.0, 0.125, -0.0625], np.float32), size=(P, 1, K, d)))
    c1[:, :, ::2] = np.float32(c1mag) * rng.choice([-1.0, 1.0], size=c1[:, :, ::2].shape)
    cent = torch.from_numpy(np.concatenate([c0, c1], axis=1).astype(np.float32)).to(torch.bfloat16)
    asg = rng.integers(0, K, size=(P, 2, N)).astype(np.uint8)
    cfg = QuantConfig(bits=bits, group_size=B, stages=2, centroids=K)
    dc = D.DeviceChunks(cfg, N, d, torch.from_numpy(pay).cuda(), torch.from_numpy(sc).cuda(), cent.cuda(),
                        torch.from_numpy(asg).cuda())
    ref = oracle_lib.prq_decompress_batch(pay, sc, cent.float().numpy(), asg, N, d, bits, B, 8)
    out = D.dequantize(dc, torch.float32).cpu().numpy()
    assert np.array_equal(_u32(out), _u32(ref))
    outb = D.dequantize(dc, torch.bfloat16).cpu()
    assert torch.equal(outb.view(torch.int16), torch.from_numpy(ref).to(torch.bfloat16).view(torch.int16))


@pytest.mark.parametrize("d,K,S,bits,B", [(64, 64, 2, 2, 64), (256, 32, 2, 4, 64), (128, 256, 1, 2, 64),
                                          (128, 256, 2, 2, 32), (128, 16, 3, 8, 16)])
def test_many_planes_shapes_vs_oracle(oracle_lib, d, K, S, bits, B):
    """>= 148 planes at other head dims / table sizes: d 64 and 256, K 256
    (one f32 table buffer: the per-plane barrier path), 16-channel groups."""
    rng = np.random.default_rng(d + K + S)
    P, N = 150, 40
    x = _rand_planes(rng, P, N, d, 10.0)
    cent = torch.from_numpy(rng.normal(0, 1.5, size=(P, S, K, d)).astype(np.float32)).to(torch.bfloat16)
    asg = torch.from_numpy(rng.integers(0, K, size=(P, S, N)).astype(np.uint8))
    cfg = QuantConfig(bits=bits, group_size=B, stages=S, centroids=K)
    pay, sc = D.quantize(x.cuda(), cfg, cent.cuda(), asg.cuda())
    rp, rs = oracle_lib.quantize_given_metas_batch(x.float().numpy(), cent.float().numpy(), asg.numpy(), bits, B, 8)
    assert np.array_equal(sc.cpu().numpy(), rs)
    assert np.array_equal(pay.cpu().numpy(), rp)
    dc = D.DeviceChunks(cfg, N, d, pay, sc, cent.cuda(), asg.cuda())
    out = D.dequantize(dc, torch.float32).cpu().numpy()
    ref = oracle_lib.prq_decompress_batch(rp, rs, cent.float().numpy(), asg.numpy(), N, d, bits, B, 8)
    assert np.array_equal(_u32(out), _u32(ref))
