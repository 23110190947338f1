"""The CPU oracle (oracle/qvg_oracle.c) against fixtures written by the
reference itself (tests/golden/make_golden.py).  Pins the oracle."""
import os

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


def test_oracle_stage_curve_and_lloyd_vs_reference(oracle_lib):
    """curves.npz (make_golden_curves.py, the reference's stage_mse_curve and
    lloyd_step): the oracle's compress/decompress per stage prefix gives the
    same MSE values (np.mean over the same float64 differences), and its
    lloyd_step the same centroids, assignments (incl. the empty-cluster
    repair) and objective."""
    from paper_2602_02958_b200 import datagen as G

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "curves.npz"))
    xs = {}
    for name, seed, value in (("key", 10, False), ("value", 11, True)):
        p = G.StreamParams(n_tokens=1560, drift=0.0125, outlier_scale=100.0 if value else 10.0)
        x = G.bf16_bits_to_f32(G.round_bf16_bits(G.stream_chunk(seed, 3, p)))
        xs[name] = x
        for B in (16, 64):
            curve = []
            for S in range(5):
                draws = oracle_lib.pp_draws(0, 3, S, 64)
                r = oracle_lib.prq_compress(x, 2, B, S, 64, 10, 1e-4, draws=draws)
                rec = oracle_lib.prq_decompress(r["payload"], r["scales"], r["centroids"], r["assignments"],
                                                1560, 128, 2, B)
                curve.append(float(np.mean((x.astype(np.float64) - rec.astype(np.float64)) ** 2)))
            assert curve == list(z[f"{name}_curve_b{B}"]), (name, B)
    rows = xs["value"].astype(np.float64)[:700]
    init = rows[z["lloyd_pick"]].copy()
    init[z["lloyd_far"]] = 1e4
    cent, asg, obj = oracle_lib.lloyd_step(rows, init)
    assert np.array_equal(cent.view(np.uint64), z["lloyd_cent"].view(np.uint64))
    assert np.array_equal(asg, z["lloyd_asg"])
    assert obj == float(z["lloyd_obj"])
