"""Baseline competitors (Q/baselines.py) and the QVGC container on the device,
bit-exact against outputs of the REFERENCE itself (tests/golden/baselines.npz,
container_*.npz, made by tests/golden/make_golden_baselines.py)."""
import io
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2602_02958_b200.qvgcodec import baselines as Bq  # noqa: E402
from paper_2602_02958_b200.qvgcodec import container as C  # noqa: E402
from paper_2602_02958_b200.qvgcodec.prq import prq_compress, prq_decompress_onepass  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import KVPlane, QuantConfig  # noqa: E402

HERE = os.path.join(os.path.dirname(__file__), "golden")
G = np.load(os.path.join(HERE, "baselines.npz"))
CASES = sorted({k.split("_")[0] for k in G.files})


def _b(a):
    return np.asarray(a, np.uint8).tobytes()


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("c", CASES)
def test_rtn(c):
    n, d, bits, gs = (int(v) for v in G[f"{c}_cfg"])
    p, s = Bq.rtn_compress(KVPlane.from_array(G[f"{c}_x"]), bits, gs)
    assert p == _b(G[f"{c}_rtn_payload"]) and s == _b(G[f"{c}_rtn_scales"])
    assert _same(Bq.rtn_decompress(p, s, n, d, bits, gs), G[f"{c}_rtn_dec"])


@pytest.mark.parametrize("c", CASES)
def test_kivi(c):
    n, d, bits, gs = (int(v) for v in G[f"{c}_cfg"])
    kc = Bq.kivi_compress(KVPlane.from_array(G[f"{c}_x"]), KVPlane.from_array(G[f"{c}_v"]), bits, gs)
    assert kc.padded_tokens == int(G[f"{c}_kivi_pad"][0])
    assert kc.keys_payload == _b(G[f"{c}_kivi_kp"]) and kc.keys_scales == _b(G[f"{c}_kivi_ks"])
    assert kc.values_payload == _b(G[f"{c}_kivi_vp"]) and kc.values_scales == _b(G[f"{c}_kivi_vs"])
    k, v = Bq.kivi_decompress(kc)
    assert _same(k, G[f"{c}_kivi_kdec"]) and _same(v, G[f"{c}_kivi_vdec"])


@pytest.mark.parametrize("c", CASES)
def test_quarot_and_hadamard(c):
    n, d, bits, gs = (int(v) for v in G[f"{c}_cfg"])
    seed = int(G[f"{c}_quarot_seed"][0])
    signs = Bq.random_signs(d, seed)
    assert np.array_equal(signs, G[f"{c}_signs"])
    x8 = G[f"{c}_x"][:8]
    assert _same(Bq.hadamard_transform(x8, signs), G[f"{c}_had_fwd"])
    assert _same(Bq.inverse_hadamard(x8, signs), G[f"{c}_had_inv"])
    qc = Bq.quarot_compress(KVPlane.from_array(G[f"{c}_x"]), bits, gs, seed)
    assert qc.payload == _b(G[f"{c}_quarot_payload"]) and qc.scales == _b(G[f"{c}_quarot_scales"])
    assert _same(Bq.quarot_decompress(qc), G[f"{c}_quarot_dec"])


@pytest.mark.parametrize("tag", ["s2", "s1b4"])
def test_container_written_on_device_matches_reference_file(tag):
    z = np.load(os.path.join(HERE, f"container_{tag}.npz"))
    bits, gs, S, K, seed, n = (int(v) for v in z["cfg"])
    cfg = QuantConfig(bits=bits, group_size=gs, stages=S, centroids=K, seed=seed)
    buf = io.BytesIO()
    w = C.ChunkWriter(buf, C.QvgcHeader.for_config(cfg, 128))
    chunks = []
    for c, x in enumerate(z["planes"]):
        ch = prq_compress(KVPlane.from_array(x, chunk_index=c), cfg)
        chunks.append(ch)
        w.append_chunk(ch)
    assert buf.getvalue() == z["qvgc"].tobytes()
    r = C.ChunkReader(io.BytesIO(buf.getvalue()))
    planes = C.dequantize_range(r, 0, r.count - 1)
    for ch, pl in zip(chunks, planes):
        assert _same(pl.data, prq_decompress_onepass(ch).data)
    assert C.dequantize_range(r, 1, 0) == []


def test_container_baseline_tags_decode():
    c = CASES[0]
    n, d, bits, gs = (int(v) for v in G[f"{c}_cfg"])
    for tag in (C.MethodTag.RTN, C.MethodTag.QUAROT):
        cfg = QuantConfig(bits=bits, group_size=gs, stages=0, centroids=1, seed=int(G[f"{c}_quarot_seed"][0]))
        hdr = C.QvgcHeader.for_config(cfg, d, method_tag=tag)
        from paper_2602_02958_b200.qvgcodec.types import ChunkSpec, CompressedChunk
        pay = G[f"{c}_rtn_payload"] if tag == C.MethodTag.RTN else G[f"{c}_quarot_payload"]
        sc = G[f"{c}_rtn_scales"] if tag == C.MethodTag.RTN else G[f"{c}_quarot_scales"]
        ch = CompressedChunk(spec=ChunkSpec(n, d), config=cfg, payload=_b(pay), scales=_b(sc))
        buf = io.BytesIO()
        C.ChunkWriter(buf, hdr).append_chunk(ch)
        out = C.dequantize_range(C.ChunkReader(io.BytesIO(buf.getvalue())), 0, 0)[0].data
        want = G[f"{c}_rtn_dec"] if tag == C.MethodTag.RTN else G[f"{c}_quarot_dec"]
        assert _same(out, want)
