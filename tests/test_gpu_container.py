"""QVGC records built and verified on the device (SURVEY §8(f) row 2,
Q/container.py:158-387): byte-identical to files the reference wrote, CRC32
computed on the GPU equals zlib's, corrupt / torn records isolated as the
reference reader does, and a whole device batch written / read / decoded in
one launch each."""
import io
import os
import zlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2602_02958_b200 import datagen as G  # noqa: E402
from paper_2602_02958_b200 import device as D  # noqa: E402
from paper_2602_02958_b200.qvgcodec import container as C  # noqa: E402
from paper_2602_02958_b200.qvgcodec.errors import ConfigMismatch, CorruptChunk  # noqa: E402
from paper_2602_02958_b200.qvgcodec.types import QuantConfig  # noqa: E402

HERE = os.path.join(os.path.dirname(__file__), "golden")


def _ref_file(tag):
    z = np.load(os.path.join(HERE, f"container_{tag}.npz"))
    return z["qvgc"].tobytes(), z


@pytest.mark.parametrize("tag", ["s2", "s1b4"])
def test_reference_file_reread_on_device_and_rewritten_byte_identical(tag):
    raw, z = _ref_file(tag)
    r = C.ChunkReader(io.BytesIO(raw))
    dc = r.read_device(0, r.count - 1)
    out = io.BytesIO()
    w = C.ChunkWriter(out, r.header)
    assert list(w.append_planes(dc)) == [0, 1]
    assert out.getvalue() == raw
    # per-record host API through the same device path
    out2 = io.BytesIO()
    w2 = C.ChunkWriter(out2, r.header)
    for i in range(r.count):
        w2.append_chunk(r.read_chunk(i))
    assert out2.getvalue() == raw


def test_device_crc_matches_zlib_on_odd_lengths():
    # records whose body length is not a multiple of the 256-way segmentation
    for n, S, K in ((4, 1, 1), (36, 2, 3), (1000, 3, 5), (4680, 2, 64)):
        cfg = QuantConfig(bits=2, group_size=32, stages=S, centroids=K)
        g = torch.Generator(device="cuda").manual_seed(n)
        P = 3
        dc = D.DeviceChunks(
            cfg, n, 128,
            torch.randint(0, 256, (P, n * 128 * 2 // 8), generator=g, device="cuda", dtype=torch.uint8),
            torch.randint(0, 120, (P, n * 128 // 32), generator=g, device="cuda", dtype=torch.uint8),
            torch.randn((P, S, K, 128), generator=g, device="cuda").to(torch.bfloat16),
            torch.randint(0, K, (P, S, n), generator=g, device="cuda", dtype=torch.uint8))
        h = C.QvgcHeader.for_config(cfg, 128)
        recs = C.pack_records(dc, h, 7).cpu().numpy()
        for p in range(P):
            b = recs[p].tobytes()
            body = b[20:-4]
            assert int.from_bytes(b[-4:], "little") == zlib.crc32(body)
            assert int.from_bytes(b[:4], "little") == 7 + p
        back, ok = C.unpack_records(torch.from_numpy(recs).cuda(), h, n)
        assert torch.all(ok == 1)
        for f in ("payload", "scales", "assignments"):
            assert torch.equal(getattr(back, f), getattr(dc, f))
        assert torch.equal(back.centroids.view(torch.int16), dc.centroids.view(torch.int16))


def test_corrupt_and_torn_records_are_isolated():
    raw, _ = _ref_file("s2")
    r = C.ChunkReader(io.BytesIO(raw))
    bad = bytearray(raw)
    bad[r._index[0][0] + C.RECORD_HEADER_SIZE + 3] ^= 0xFF          # a body byte of chunk 0
    r2 = C.ChunkReader(io.BytesIO(bytes(bad)))
    with pytest.raises(CorruptChunk):
        r2.read_chunk(0)
    r2.read_chunk(1)                                                # neighbour still readable
    with pytest.raises(CorruptChunk):
        C.dequantize_range(r2, 0, 1)
    assert len(C.dequantize_range(r2, 1, 1)) == 1
    r3 = C.ChunkReader(io.BytesIO(raw[:-7]))                        # last record cut short
    r3.read_chunk(0)
    with pytest.raises(CorruptChunk):
        r3.read_chunk(1)


def test_device_batch_write_read_decode(tmp_path):
    """One chunk of 24 C1-shaped planes: written as one batch, read back as one
    batch, decoded in one launch; equals the device decode of the compressed
    batch and the per-record files."""
    cfg = QuantConfig(bits=2, group_size=64, stages=2, centroids=64)
    refs = G.cache_layout(1, 12, [0])
    x = torch.from_numpy(G.kv_cache_bf16(refs, 12, 1024, workers=4).view(np.int16)).cuda().view(torch.bfloat16)
    dc = D.compress(x, cfg, chunk_index=0)
    h = C.QvgcHeader.for_config(cfg, 128)
    path = tmp_path / "cache.qvgc"
    with C.ChunkWriter(str(path), h) as w:
        w.append_planes(dc.select(slice(0, 10)))
        w.append_planes(dc.select(slice(10, 24)))
    with C.ChunkReader(str(path)) as r:
        assert r.count == 24
        back = r.read_device(0, 23)
        for f in ("payload", "scales", "assignments"):
            assert torch.equal(getattr(back, f), getattr(dc, f))
        planes = C.dequantize_range(r, 3, 20)
        ref = D.dequantize(dc, torch.float32).cpu().numpy()
        for k, pl in enumerate(planes):
            assert pl.spec.chunk_index == 3 + k
            assert np.array_equal(pl.data.view(np.uint32), ref[3 + k].view(np.uint32))
    with pytest.raises(ConfigMismatch):
        C.ChunkWriter(io.BytesIO(), C.QvgcHeader.for_config(cfg.with_stages(1), 128)).append_planes(dc)
