"""The CPU oracle (oracle/qvg_oracle.c) against fixtures written by the
reference itself (tests/golden/make_golden.py).  Pins the oracle."""
import numpy as np
import pytest

from conftest import golden_planes
from golden_io import load_kat, load_plane


def test_fp8_encode_matches_reference(oracle_lib):
    kat = load_kat()
    up = np.array([oracle_lib.e4m3_encode(x, True) for x in kat["fp8_x"]], np.uint8)
    ne = np.array([oracle_lib.e4m3_encode(x, False) for x in kat["fp8_x"]], np.uint8)
    assert np.array_equal(up, kat["fp8_up"])
    assert np.array_equal(ne, kat["fp8_nearest"])


def test_bf16_round_matches_reference(oracle_lib):
    kat = load_kat()
    assert np.array_equal(oracle_lib.round_bf16(kat["bf16_in"]).view(np.uint32),
                          kat["bf16_out"].view(np.uint32))


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("g", [8, 16, 64, 128])
def test_quantize_matrix_matches_reference(oracle_lib, bits, g):
    kat = load_kat()
    pre = f"qm_b{bits}_g{g}_"
    p, s = oracle_lib.quantize_matrix(kat[pre + "x"], bits, g)
    assert np.array_equal(p, kat[pre + "payload"])
    assert np.array_equal(s, kat[pre + "scales"])
    deq = oracle_lib.dequantize_matrix(p, s, 37, 128, bits, g)
    assert np.array_equal(deq.view(np.uint32), kat[pre + "deq"].view(np.uint32))


@pytest.mark.parametrize("name", golden_planes())
def test_prq_plane_matches_reference(oracle_lib, name):
    rec = load_plane(name)
    S, K = rec["stages"], rec["centroids"]
    draws = oracle_lib.pp_draws(0, rec["chunk_index"], S, K)
    warm = rec.get("warm")
    out = oracle_lib.prq_compress(rec["x"], rec["bits"], rec["group_size"], S, K,
                                  draws=draws, warm=warm)
    assert np.array_equal(out["iters"], rec["iters"]), "k-means iteration counts"
    assert np.array_equal(out["assignments"], rec["assignments"]), "assignments"
    assert np.array_equal(out["centroids_f64"].view(np.uint64), rec["cent_f64"].view(np.uint64))
    assert np.array_equal(out["centroids"].view(np.uint32), rec["centroids_bf16"].view(np.uint32))
    assert np.array_equal(out["payload"], rec["payload"]), "payload bytes"
    assert np.array_equal(out["scales"], rec["scales"]), "scale bytes"
    n, d = rec["x"].shape
    dec = oracle_lib.prq_decompress(out["payload"], out["scales"], out["centroids"],
                                    out["assignments"], n, d, rec["bits"], rec["group_size"])
    assert np.array_equal(dec.view(np.uint32), rec["decoded"].view(np.uint32))


@pytest.mark.parametrize("name", ["c1_key", "s4_pro", "k256", "ties", "n_lt_k"])
def test_kmeanspp_picks_match_reference(oracle_lib, name):
    rec = load_plane(name)
    if "pp_first_picks" not in rec:
        pytest.skip("warm-started")
    draws = oracle_lib.pp_draws(0, rec["chunk_index"], 1, rec["centroids"])[0]
    x = rec["x"].astype(np.float64)
    cent, chosen = oracle_lib.kmeans_pp(x, rec["centroids"], draws)
    ref_rows = x[rec["pp_first_picks"][0]]
    assert np.array_equal(cent, ref_rows)
