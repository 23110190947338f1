"""QVGC container (Q/container.py mirror) host logic without a GPU: the file
header and the record index scan over files the REFERENCE wrote
(tests/golden/container_*.npz).  Record bodies (CRC, fields) are verified on
the device: tests/test_gpu_container.py."""
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
def test_reference_file_header_and_index(tag):
    raw, z = _ref_file(tag)
    r = C.ChunkReader(io.BytesIO(raw))
    bits, gs, S, K, seed, n = (int(v) for v in z["cfg"])
    assert (r.header.bits, r.header.group_size, r.header.stages, r.header.centroids, r.header.seed) == \
        (bits, gs, S, K, seed)
    assert r.count == 2
    rs = r.header.record_size(n)
    assert [e[0] for e in r._index] == [C.HEADER_SIZE, C.HEADER_SIZE + rs]
    assert all(e[1] == n and e[2] for e in r._index)
    assert C.HEADER_SIZE + 2 * rs == len(raw)


def test_torn_and_mislabelled_records_in_the_index():
    raw, _ = _ref_file("s2")
    r3 = C.ChunkReader(io.BytesIO(raw[:-7]))                      # last record cut short
    assert r3.count == 2 and r3._index[0][2] and not r3._index[1][2]
    with pytest.raises(CorruptChunk):
        r3._check(1)
    with pytest.raises(OutOfRange):
        r3._check(2)
    bad = bytearray(raw)
    bad[C.HEADER_SIZE] = 5                                         # chunk_index of record 0
    r4 = C.ChunkReader(io.BytesIO(bytes(bad)))
    assert r4.count == 2 and not r4._index[0][2] and r4._index[1][2]
    r5 = C.ChunkReader(io.BytesIO(raw[:C.HEADER_SIZE + 9]))       # torn record header
    assert r5.count == 1 and not r5._index[0][2]


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
