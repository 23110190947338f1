"""The synthetic-input restatement (paper_2602_02958_b200/datagen.py) against
the reference generator's own output (tests/golden/datagen.npz, written by
make_golden_datagen.py from Q/datagen.py): bit-identical float32 planes,
including drifted chunks addressed directly and full-size bench planes."""
import hashlib
import os

import numpy as np

from paper_2602_02958_b200 import datagen as G

GOLD = os.path.join(os.path.dirname(__file__), "golden", "datagen.npz")
SPECS = {  # mirrors make_golden_datagen.DIGESTS
    "sf_key_l0h0": (0, 4680, 0.0125, 10.0),
    "sf_val_l1h11": (2 * (1 * 12 + 11) + 1, 4680, 0.0125, 100.0),
    "sf_key_nodrift": (7, 4680, 0.0, 10.0),
    "longcat_val_h3": (7, 38400, 0.0, 100.0),
}


def test_small_stream_bit_identical():
    ref = np.load(GOLD)["small"]
    p = G.StreamParams(n_tokens=160, d=128, n_clusters=16, drift=0.05, outlier_scale=100.0)
    for c in (2, 0, 1):                         # any order: chunks are addressable
        got = G.stream_chunk(5, c, p)
        assert np.array_equal(got.view(np.uint32), ref[c].view(np.uint32)), c


def test_full_size_digests():
    z = np.load(GOLD)
    for name, dig in zip(z["digest_names"], z["digests"]):
        stream, c = str(name).split("/c")
        seed, n, drift, osc = SPECS[stream]
        p = G.StreamParams(n_tokens=n, drift=drift, outlier_scale=osc)
        got = G.stream_chunk(seed, int(c), p)
        assert hashlib.sha256(got.tobytes()).hexdigest() == str(dig), name


def test_parallel_cache_fill_matches_serial():
    planes = G.cache_layout(1, 2, [0, 1])
    par = G.kv_cache_bf16(planes, 2, 300, drift=0.0125, workers=2)
    for i, r in enumerate(planes):
        p = G.kv_params(300, r.value, 0.0125)
        one = G.round_bf16_bits(G.stream_chunk(G.kv_seed(r.layer, r.head, 2, r.value), r.chunk, p))
        assert np.array_equal(par[i], one), i
    # bf16 rounding is RNE (Q/lowprec.py round_to_bf16)
    from paper_2602_02958_b200.qvgcodec.lowprec import round_to_bf16
    x = G.stream_chunk(3, 0, G.kv_params(300, True))
    assert np.array_equal(G.bf16_bits_to_f32(G.round_bf16_bits(x)).view(np.uint32),
                          round_to_bf16(x).view(np.uint32))
