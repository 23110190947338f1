"""QVGC container (Q/container.py mirror) on the host: files written by the
REFERENCE (tests/golden/container_*.npz) parse with our reader and re-write
byte-identically; torn / corrupt records are isolated as the reference does."""
import io
import os

import numpy as np
import pytest

from paper_2602_02958_b200.qvgcodec import container as C
from paper_2602_02958_b200.qvgcodec.errors import BadMagic, CorruptChunk, OutOfRange, Truncated

HERE = os.path.join(os.path.dirname(__file__), "golden")


def _ref_file(tag):
    z = np.load(os.path.join(HERE, f"container_{tag}.npz"))
    return z["qvgc"].tobytes(), z


@pytest.mark.parametrize("tag", ["s2", "s1b4"])
def test_reference_file_roundtrips_byte_identical(tag):
    raw, z = _ref_file(tag)
    r = C.ChunkReader(io.BytesIO(raw))
    bits, gs, S, K, seed, n = (int(v) for v in z["cfg"])
    assert (r.header.bits, r.header.group_size, r.header.stages, r.header.centroids, r.header.seed) == \
        (bits, gs, S, K, seed)
    assert r.count == 2
    out = io.BytesIO()
    w = C.ChunkWriter(out, r.header)
    for i in range(r.count):
        ch = r.read_chunk(i)
        assert ch.spec.n_tokens == n and len(ch.stages) == S
        w.append_chunk(ch)
    assert out.getvalue() == raw


def test_corrupt_and_torn_records_are_isolated():
    raw, _ = _ref_file("s2")
    r = C.ChunkReader(io.BytesIO(raw))
    first = r._entries[0]
    bad = bytearray(raw)
    bad[first.offset + C.RECORD_HEADER_SIZE + 3] ^= 0xFF          # body byte of chunk 0
    r2 = C.ChunkReader(io.BytesIO(bytes(bad)))
    with pytest.raises(CorruptChunk):
        r2.read_chunk(0)
    r2.read_chunk(1)                                              # neighbour still readable
    torn = raw[:-7]                                               # last record cut short
    r3 = C.ChunkReader(io.BytesIO(torn))
    assert r3.count == 2
    r3.read_chunk(0)
    with pytest.raises(CorruptChunk):
        r3.read_chunk(1)
    with pytest.raises(OutOfRange):
        r3.read_chunk(2)


def test_header_validation():
    raw, _ = _ref_file("s1b4")
    with pytest.raises(BadMagic):
        C.QvgcHeader.from_bytes(b"XXXX" + raw[4:32])
    with pytest.raises(BadMagic):
        C.QvgcHeader.from_bytes(raw[:30] + b"\x01\x00")
    with pytest.raises(Truncated):
        C.QvgcHeader.from_bytes(raw[:10])
    h = C.QvgcHeader.from_bytes(raw)
    assert h.to_bytes() == raw[:32]
