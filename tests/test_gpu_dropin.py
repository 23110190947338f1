"""The drop-in mirror (paper_2602_02958_b200.qvgcodec) against the
reference's outputs: same functions, same arguments, same results."""
import numpy as np
import pytest

from conftest import golden_planes
from golden_io import load_kat, load_plane

pytestmark = pytest.mark.gpu

from paper_2602_02958_b200.qvgcodec import clustering, errors, prq, quant, smoothing  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import ChunkSpec, KVPlane, QuantConfig  # noqa: E402


def _plane(rec):
    return KVPlane.from_array(rec["x"], chunk_index=rec["chunk_index"])


@pytest.mark.parametrize("name", ["c1_key", "s4_pro", "k1", "ties", "n_lt_k", "d24", "zero",
                                  "s0_rtn_saturate"])
def test_prq_compress_decompress(name):
    rec = load_plane(name)
    cfg = QuantConfig(bits=rec["bits"], group_size=rec["group_size"], stages=rec["stages"],
                      centroids=rec["centroids"])
    chunk = prq.prq_compress(_plane(rec), cfg)
    assert chunk.payload == rec["payload"].tobytes()
    assert chunk.scales == rec["scales"].tobytes()
    for t, meta in enumerate(chunk.stages):
        assert np.array_equal(meta.assignments, rec["assignments"][t])
        assert np.array_equal(meta.centroids.view(np.uint32), rec["centroids_bf16"][t].view(np.uint32))
    counters = prq.DecodeCounters()
    out = prq.prq_decompress_onepass(chunk, counters)
    assert np.array_equal(out.data.view(np.uint32), rec["decoded"].view(np.uint32))
    assert np.array_equal(prq.prq_decompress(chunk).data, out.data)
    assert counters.centroid_lookups_per_token == cfg.stages and counters.tokens == rec["x"].shape[0]


def test_warm_start_via_dropin():
    rec = load_plane("warm1")
    cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=32)
    chunk = prq.prq_compress(_plane(rec), cfg, warm_init=list(rec["warm"]))
    assert chunk.payload == rec["payload"].tobytes()
    with pytest.raises(ValueError):
        prq.prq_compress(_plane(rec), cfg, warm_init=[rec["warm"][0]])


def test_kmeans_and_smoothing_dropin(oracle_lib):
    rec = load_plane("s4_pro")
    rows = rec["x"].astype(np.float64)
    seed = prq.stage_seed(0, 2, 1)
    res = clustering.kmeans(rows, 16, 10, 1e-4, seed=seed)
    draws = np.random.Generator(np.random.Philox(seed)).random(16)
    c_o, a_o, obj_o, it_o = oracle_lib.kmeans(rows, 16, 10, 1e-4, draws=draws)
    assert np.array_equal(res.centroids.view(np.uint64), c_o.view(np.uint64))
    assert res.iterations_used == it_o and res.objective == obj_o
    resid, meta = smoothing.sa_smoothing(rows, 16, seed)
    assert np.array_equal(meta.assignments, rec["assignments"][0])
    back = smoothing.add_back(resid, meta)
    assert np.array_equal(back, rows)                          # exact inverse
    init = clustering.kmeans_pp_init(rows, 16, seed)
    assert np.array_equal(init, oracle_lib.kmeans_pp(rows, 16, draws)[0])
    new_c, asg, obj = clustering.lloyd_step(rows, init)
    c_o, a_o, obj_o = oracle_lib.lloyd_step(rows, init)
    assert np.array_equal(new_c.view(np.uint64), c_o.view(np.uint64))
    assert np.array_equal(asg, a_o) and obj == obj_o
    with pytest.raises(errors.EmptyInput):
        clustering.kmeans(np.zeros((0, 4)), 2)
    with pytest.raises(errors.DimensionMismatch):
        clustering.kmeans(rows, 16, init=np.zeros((3, 3)))


def _curve_planes():
    from paper_2602_02958_b200 import datagen as G

    out = {}
    for name, seed, value in (("key", 10, False), ("value", 11, True)):
        p = G.StreamParams(n_tokens=1560, drift=0.0125, outlier_scale=100.0 if value else 10.0)
        out[name] = G.bf16_bits_to_f32(G.round_bf16_bits(G.stream_chunk(seed, 3, p)))
    return out


def test_stage_mse_curve_vs_reference():
    """C4 stage sweep (S 0..4, B 16/64): the drop-in curve equals the
    reference's own stage_mse_curve values (tests/golden/curves.npz) exactly;
    the batched device curve matches them to float64 reduction-order noise."""
    import os
    import torch
    from paper_2602_02958_b200 import device as D

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "curves.npz"))
    xs = _curve_planes()
    for B in (16, 64):
        cfg = QuantConfig(bits=2, group_size=B, stages=1, centroids=64)
        for name, x in xs.items():
            plane = KVPlane(spec=ChunkSpec(n_tokens=1560, head_dim=128, chunk_index=3), data=x)
            assert prq.stage_mse_curve(plane, cfg, 4) == list(z[f"{name}_curve_b{B}"]), (name, B)
        xd = torch.from_numpy(np.stack([xs["key"], xs["value"]])).to(torch.bfloat16).cuda()
        dev = D.stage_mse_curve(xd, cfg, 4, chunk_index=3).cpu().numpy()
        ref = np.stack([z[f"key_curve_b{B}"], z[f"value_curve_b{B}"]])
        assert np.allclose(dev, ref, rtol=1e-12, atol=0), (dev, ref)


def test_lloyd_step_vs_reference_with_empty_clusters():
    import os
    import torch
    from paper_2602_02958_b200 import device as D

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "curves.npz"))
    rows = _curve_planes()["value"].astype(np.float64)[:700]
    init = rows[z["lloyd_pick"]].copy()
    init[z["lloyd_far"]] = 1e4
    c, a, obj = clustering.lloyd_step(rows, init)
    assert np.array_equal(c.view(np.uint64), z["lloyd_cent"].view(np.uint64))
    assert np.array_equal(a, z["lloyd_asg"]) and obj == float(z["lloyd_obj"])
    cd, ad, od = D.lloyd_step(torch.from_numpy(rows).cuda()[None], torch.from_numpy(init).cuda()[None])
    assert np.array_equal(cd[0].cpu().numpy().view(np.uint64), z["lloyd_cent"].view(np.uint64))
    assert np.array_equal(ad[0].cpu().numpy(), z["lloyd_asg"].astype(np.uint8))
    assert od[0].item() == float(z["lloyd_obj"])


def test_final_residual_inverse():
    rec = load_plane("s4_pro")
    cfg = QuantConfig(bits=2, group_size=16, stages=2, centroids=16)
    plane = _plane(rec)
    r = prq.final_residual(plane, cfg)
    back = r.copy()
    # residual + stage centroids == x (exact in f64)
    chunk = prq.prq_compress(plane, cfg)
    for meta in reversed(chunk.stages):
        back = smoothing.add_back(back, meta)
    assert np.array_equal(back, rec["x"].astype(np.float64))


def test_quantizer_known_answers():
    g = quant.quantize_group(np.zeros(8), bits=2)
    assert not g.q.any() and g.scale_fp8 == 0x38
    g = quant.quantize_group([3.0, -3.0, 1.4, 0.0], bits=2)
    assert list(g.q) == [1, -1, 0, 0]
    g = quant.quantize_group(np.concatenate([[1.0, -0.5, 0.25, 0.0], np.zeros(12)]), bits=4)
    assert list(g.q[:4]) == [6, -3, 2, 0]
    assert np.allclose(quant.dequantize_group(g)[:4], 0.15625 * np.array([6, -3, 2, 0]), atol=0)
    assert quant.pack_payload([1, -1, 0, 1], 2) == bytes([0x4D])
    assert quant.pack_payload([7, -4], 4) == bytes([0xC7])
    assert quant.pack_payload([], 2) == b""
    assert list(quant.unpack_payload(bytes([0x4D]), 4, 2)) == [1, -1, 0, 1]
    assert list(quant.unpack_payload(bytes([0xC7]), 2, 4)) == [7, -4]
    with pytest.raises(errors.RangeOverflow):
        quant.pack_payload([-2], 2)
    with pytest.raises(errors.Truncated):
        quant.unpack_payload(b"\x00", 5, 2)
    with pytest.raises(errors.NonFiniteInput):
        quant.quantize_group([1.0, np.nan], bits=4)


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("g", [8, 16, 64, 128])
def test_quantize_matrix_f64_matches_reference(bits, g):
    kat = load_kat()
    pre = f"qm_b{bits}_g{g}_"
    p, s = quant.quantize_matrix(kat[pre + "x"], QuantConfig(bits=bits, group_size=g))
    assert p == kat[pre + "payload"].tobytes() and s == kat[pre + "scales"].tobytes()
    deq = quant.dequantize_plane(p, s, 37, 128, bits, g)
    assert np.array_equal(deq.view(np.uint32), kat[pre + "deq"].view(np.uint32))


def test_random_pack_roundtrip_and_errors():
    rng = np.random.default_rng(51)
    for bits in (2, 4, 8):
        qmax = 2 ** (bits - 1) - 1
        for n in (1, 2, 3, 7, 8, 64, 1000):
            q = rng.integers(-qmax, qmax + 1, size=n)
            packed = quant.pack_payload(q, bits)
            assert np.array_equal(quant.unpack_payload(packed, n, bits), q)
    plane = KVPlane.from_array(np.zeros((4, 32), np.float32))
    payload, scales = quant.quantize_plane(plane, QuantConfig(bits=2, group_size=16))
    assert payload == bytes(len(payload)) and set(scales) == {0x38}
    with pytest.raises(errors.DimensionMismatch):
        quant.quantize_matrix(np.zeros((4, 100)), QuantConfig(group_size=64))
